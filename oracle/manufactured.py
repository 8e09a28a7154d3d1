"""Steady manufactured problem and FE error norms (ORACLE -- test infrastructure only).

PAPER.md:936-945 (sec. 5.1): exact solution u = curl phi, phi = [x y (1-x)(1-y)]^2,
p = 1, w = 0, one backward-Euler step with tau = 1; material parameters as in
the LFA validation (E = 3e4, alpha = 1, mu_f = 1, M = 1e6, K = k I).  Then
div u = 0 and grad p = 0, so eq. (Biot-eq1) gives rho g = -mu Laplace(u),
eq. (Biot-eq2) gives rho_f g = 0, and the mass equation reduces to
(f_hat, q) = (1/M)(1, q).  The right-hand side of eq. (block_form_rq) is

    u-block (-mu Laplace u, v_h),   w-block 0,   p-block -(1/M)(1, q_h).

PAPER.md:1016-1020 (Fig. fig:mgtime): |u - u_h|_1 = O(h), ||p - p_h|| = O(h^2)
on uniform meshes.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse.linalg as spla

from .mesh import Mesh, NORMALS
from .fem import Operator, p1_geometry


def _A(x):
    return x * x * (1 - x) ** 2


def _A1(x):
    return 2 * x - 6 * x ** 2 + 4 * x ** 3


def _A2(x):
    return 2 - 12 * x + 12 * x ** 2


def _A3(x):
    return -12 + 24 * x


def u_exact(x, y):
    """u = curl phi = (d_y phi, -d_x phi), phi = A(x) A(y), A(s) = s^2 (1-s)^2."""
    return np.stack([_A(x) * _A1(y), -_A1(x) * _A(y)], axis=-1)


def grad_u_exact(x, y):
    """(.., 2, 2) with [c, d] = d u_c / d x_d."""
    g = np.empty(np.shape(x) + (2, 2))
    g[..., 0, 0] = _A1(x) * _A1(y)
    g[..., 0, 1] = _A(x) * _A2(y)
    g[..., 1, 0] = -_A2(x) * _A(y)
    g[..., 1, 1] = -_A1(x) * _A1(y)
    return g


def laplace_u_exact(x, y):
    return np.stack([_A2(x) * _A1(y) + _A(x) * _A3(y), -(_A3(x) * _A(y) + _A1(x) * _A2(y))], axis=-1)


def triangle_rule(q=8):
    """Collapsed Gauss rule on the reference triangle (0,0),(1,0),(0,1); exact to degree 2q-2."""
    g, w = np.polynomial.legendre.leggauss(q)
    g = 0.5 * (g + 1.0)
    w = 0.5 * w
    U, Vv = np.meshgrid(g, g, indexing="ij")
    WU, WV = np.meshgrid(w, w, indexing="ij")
    x = U.ravel()
    y = (Vv * (1.0 - U)).ravel()
    wt = (WU * WV * (1.0 - U)).ravel()
    return np.stack([1.0 - x - y, x, y], axis=1), wt      # barycentric, weights (sum 1/2)


def rhs(op: Operator, mu, inv_M):
    """Right-hand side on the active DoFs."""
    mesh = op.mesh
    b = np.zeros(mesh.nslots)
    L, wt = triangle_rule(8)
    ls = mesh.local_slots()
    for t in range(mesh.ntri):
        P = mesh.tri_coords([t])[0]
        g, area = p1_geometry(P)
        X = L @ P
        f = -mu * laplace_u_exact(X[:, 0], X[:, 1])       # (nq, 2)
        W = wt * 2.0 * area
        for a in range(3):
            for c in range(2):
                b[ls[t, 2 * a + c]] += np.sum(W * L[:, a] * f[:, c])
        for e in range(3):
            a, bb = mesh.tri_eloc[t, e, 0], mesh.tri_eloc[t, e, 1]
            phi = 4.0 * L[:, a] * L[:, bb]
            b[ls[t, 6 + e]] += np.sum(W * phi * (f @ NORMALS[mesh.tri_ek[t, e]]))
        b[ls[t, 12]] += -inv_M * area
    return b[mesh.act_idx]


def errors(op: Operator, x):
    """(|u - u_h|_1 including the bubble part of grad u_h, ||p - p_h||_L2)."""
    mesh = op.mesh
    full = np.zeros(mesh.nslots)
    full[mesh.act_idx] = x
    L, wt = triangle_rule(8)
    ls = mesh.local_slots()
    e1 = 0.0
    ep = 0.0
    for t in range(mesh.ntri):
        P = mesh.tri_coords([t])[0]
        g, area = p1_geometry(P)
        X = L @ P
        G = grad_u_exact(X[:, 0], X[:, 1])                 # (nq, 2, 2)
        Gh = np.zeros_like(G)
        for a in range(3):
            for c in range(2):
                Gh[:, c, :] += full[ls[t, 2 * a + c]] * g[a][None, :]
        for e in range(3):
            a, bb = mesh.tri_eloc[t, e, 0], mesh.tri_eloc[t, e, 1]
            gpsi = 4.0 * (L[:, a:a + 1] * g[bb][None, :] + L[:, bb:bb + 1] * g[a][None, :])
            Gh += full[ls[t, 6 + e]] * NORMALS[mesh.tri_ek[t, e]][None, :, None] * gpsi[:, None, :]
        W = wt * 2.0 * area
        e1 += np.sum(W * np.sum((G - Gh) ** 2, axis=(1, 2)))
        ep += area * (1.0 - full[ls[t, 12]]) ** 2
    return np.sqrt(e1), np.sqrt(ep)


def solve_direct(n, nu=0.4, k=1e-6, E=3e4, inv_M=1e-6):
    """Direct sparse solve of the steady problem on an n x n mesh; returns (op, x)."""
    mu = E / (2.0 + 2.0 * nu)
    lam = E * nu / ((1.0 - 2.0 * nu) * (1.0 + nu))
    op = Operator(Mesh(n), lam, mu, 1.0, 1.0, inv_M, 1.0, K=k)
    b = rhs(op, mu, inv_M)
    x = spla.spsolve(op.A.tocsc(), b)
    return op, x

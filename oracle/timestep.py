"""Backward-Euler time stepping of the three-field Biot model (ORACLE -- test infrastructure only).

PAPER.md:113-130 (eqs. discrete1-discrete3): at step m, with constant step tau, solve
A^RQ x^m = b^m where the right-hand side carries the previous step through

    (f_hat, q) = tau (f, q) + (1/M)(p^{m-1}, q) + (alpha div u^{m-1}, q)

and eq. discrete3 is scaled by -1, so the pressure block of b^m is -(f_hat, q).  With
B_u = -(div ., q) and M_p = (., .) on P0:

    b_p^m = -tau (f^m, q) - (1/M) M_p p^{m-1} + alpha B_u u^{m-1},

while the displacement and flux blocks are the loads (rho g, v) and tau (rho_f g, r) at t_m
(discrete1, discrete2).  ``history_rhs`` is exactly that formula on the assembled blocks;
``step`` / ``run`` add the solve.

Time-dependent manufactured problem (reading A28): the paper's smooth test
 prescribes Dirichlet data for u and p on all sides, which the BASELINE
boundary conditions (u = 0, w.n = 0) cannot represent.  The same construction is applied to a
solution that satisfies u = 0 and w.n = 0 exactly:

    u = e^{-t} curl phi,  phi = [x y (1-x)(1-y)]^2   (the steady test's u),
    p = e^{-t} cos(pi x) cos(pi y)                   (dp/dn = 0 on the boundary),
    w = -(K/mu_f) grad p,

so div u = 0 and, from eqs. Biot-eq1..3,
    rho g   = -mu Laplace u + alpha grad p,
    rho_f g = 0,
    f       = (1/M) dp/dt + alpha d(div u)/dt + div w = -(1/M) p + 2 pi^2 (K/mu_f) p.
PAPER.md:1181-1184 (fig:easy_Nconv) states O(h + tau) for |u - u_h|_1 and ||p - p_h||.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse.linalg as spla

from .fem import Operator, p1_geometry
from .manufactured import grad_u_exact, laplace_u_exact, triangle_rule, u_exact
from .mesh import NORMALS


def history_rhs(op: Operator, x_prev):
    """-(1/M) M_p p^{m-1} + alpha B_u u^{m-1} on the pressure rows (active vector, zero elsewhere)."""
    out = np.zeros(op.A.shape[0])
    out[op.ip] = -op.inv_M * (op.Mp @ x_prev[op.ip]) + op.alpha * (op.Bu @ x_prev[op.iu])
    return out


def p_exact(x, y, t):
    return np.exp(-t) * np.cos(np.pi * x) * np.cos(np.pi * y)


def grad_p_exact(x, y, t):
    e = np.exp(-t)
    return np.stack([-np.pi * e * np.sin(np.pi * x) * np.cos(np.pi * y),
                     -np.pi * e * np.cos(np.pi * x) * np.sin(np.pi * y)], axis=-1)


def load(op: Operator, t, K):
    """Loads at time t on the active DoFs: u rows (rho g, v) with rho g = -mu Lap u + alpha grad p
    (u scaled by e^{-t}), w rows 0, p rows -tau (f, q) with f = (-(1/M) + 2 pi^2 K / mu_f) p."""
    mesh = op.mesh
    b = np.zeros(mesh.nslots)
    L, wt = triangle_rule(8)
    ls = mesh.local_slots()
    e = np.exp(-t)
    for tr in range(mesh.ntri):
        P = mesh.tri_coords([tr])[0]
        g, area = p1_geometry(P)
        X = L @ P
        f = -op.mu * e * laplace_u_exact(X[:, 0], X[:, 1]) + op.alpha * grad_p_exact(X[:, 0], X[:, 1], t)
        W = wt * 2.0 * area
        for a in range(3):
            for c in range(2):
                b[ls[tr, 2 * a + c]] += np.sum(W * L[:, a] * f[:, c])
        for ed in range(3):
            a, bb = mesh.tri_eloc[tr, ed, 0], mesh.tri_eloc[tr, ed, 1]
            phi = 4.0 * L[:, a] * L[:, bb]
            b[ls[tr, 6 + ed]] += np.sum(W * phi * (f @ NORMALS[mesh.tri_ek[tr, ed]]))
        fp = (-op.inv_M + 2.0 * np.pi ** 2 * K / op.mu_f) * p_exact(X[:, 0], X[:, 1], t)
        b[ls[tr, 12]] += -op.tau * np.sum(W * fp)
    return b[mesh.act_idx]


def initial(op: Operator):
    """x^0: P1 displacement = point values of u(., 0), bubbles 0, p^0 = cell means of p(., 0) (the
    only parts of x^0 the history term reads), w^0 = 0."""
    mesh = op.mesh
    x = np.zeros(mesh.nslots)
    n = mesh.n
    for j in range(1, n):
        for i in range(1, n):
            u = u_exact(i * mesh.h, j * mesh.h)
            x[mesh.slot(0, i, j)], x[mesh.slot(1, i, j)] = u[0], u[1]
    L, wt = triangle_rule(8)
    for tr in range(mesh.ntri):
        X = L @ mesh.tri_coords([tr])[0]
        x[mesh.tri_pslot[tr]] = 2.0 * np.sum(wt * p_exact(X[:, 0], X[:, 1], 0.0))
    return x[mesh.act_idx]


def errors(op: Operator, x, t):
    """(|u - u_h|_1 with the bubble part of grad u_h, ||p - p_h||_L2) at time t."""
    mesh = op.mesh
    full = np.zeros(mesh.nslots)
    full[mesh.act_idx] = x
    L, wt = triangle_rule(8)
    ls = mesh.local_slots()
    e1 = ep = 0.0
    e = np.exp(-t)
    for tr in range(mesh.ntri):
        P = mesh.tri_coords([tr])[0]
        g, area = p1_geometry(P)
        X = L @ P
        G = e * grad_u_exact(X[:, 0], X[:, 1])
        Gh = np.zeros_like(G)
        for a in range(3):
            for c in range(2):
                Gh[:, c, :] += full[ls[tr, 2 * a + c]] * g[a][None, :]
        for ed in range(3):
            a, bb = mesh.tri_eloc[tr, ed, 0], mesh.tri_eloc[tr, ed, 1]
            gpsi = 4.0 * (L[:, a:a + 1] * g[bb][None, :] + L[:, bb:bb + 1] * g[a][None, :])
            Gh += full[ls[tr, 6 + ed]] * NORMALS[mesh.tri_ek[tr, ed]][None, :, None] * gpsi[:, None, :]
        W = wt * 2.0 * area
        e1 += np.sum(W * np.sum((G - Gh) ** 2, axis=(1, 2)))
        ep += np.sum(W * (p_exact(X[:, 0], X[:, 1], t) - full[ls[tr, 12]]) ** 2)
    return np.sqrt(e1), np.sqrt(ep)


def run(op: Operator, K, nsteps, solve=None):
    """nsteps backward-Euler steps of size op.tau from x^0 = initial(op).  solve(b, x_prev) -> x^m
    (default: sparse direct).  Returns the list of iterates x^0 .. x^nsteps."""
    if solve is None:
        lu = spla.splu(op.A.tocsc())
        solve = lambda b, xp: lu.solve(b)   # noqa: E731
    xs = [initial(op)]
    for m in range(1, nsteps + 1):
        b = load(op, m * op.tau, K) + history_rhs(op, xs[-1])
        xs.append(solve(b, xs[-1]))
    return xs

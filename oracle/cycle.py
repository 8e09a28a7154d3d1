"""Hierarchy, coarsest solve, V-cycle, stationary solve and rho_N (ORACLE -- test infrastructure only).

Two-grid error propagation E_TG = E_s^{nu2} (I - P A_H^{-1} R A) E_s^{nu1}
(eq. TG-Operator-Biot), R = P^T, A_H by rediscretisation
(PAPER.md:477-484), recursed to a V-cycle with an exact solve on the coarsest
mesh.  Convergence factor rho_N = ||r_j|| / ||r_{j-1}||, run
until the change between iterations is below 1e-3.

Coarsest solve (reading A9): A_c (0, 1_p) = -gamma_c (0, 1_p) exactly under
u = 0, w.n = 0 on the whole boundary, so the dense solve is deflated the same
way as the Vanka patches.  For coarse problems too large for a dense matrix
(the two-grid pins at h = 1/64 have a 10k-unknown coarse level) a plain sparse
LU is used instead.

Heterogeneous K (reading A11): the coarse 1/K on a coarse triangle is the
arithmetic mean of 1/K over its four children.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .mesh import Mesh
from .fem import Operator
from .transfer import Transfer, _parent
from .relax import Vanka, BSR, vertex_patches


def coarsen_Kinv(fine: Mesh, coarse: Mesh, Kinv_f):
    """(2, n, n) fine 1/K -> (2, n/2, n/2) coarse 1/K (mean over the 4 children)."""
    par = _parent(fine, coarse, np.arange(fine.ntri))
    vals = Kinv_f[fine.tri_shape, fine.tri_cj, fine.tri_ci]
    acc = np.zeros(coarse.ntri)
    cnt = np.zeros(coarse.ntri)
    np.add.at(acc, par, vals)
    np.add.at(cnt, par, 1)
    out = np.zeros((2, coarse.n, coarse.n))
    out[coarse.tri_shape, coarse.tri_cj, coarse.tri_ci] = acc / cnt
    return out


class CoarseSolver:
    def __init__(self, op: Operator):
        self.op = op
        A = op.A
        N = A.shape[0]
        pm = np.zeros(N, dtype=bool)
        pm[op.ip] = True
        self.v = pm / np.sqrt(pm.sum())
        self.dense = N <= 4000
        if self.dense:
            Ad = A.toarray()
            Av = Ad @ self.v
            self.gamma = -(self.v @ Av)
            assert np.linalg.norm(Av + self.gamma * self.v) <= 1e-12 * max(1.0, np.abs(Ad).max())
            y = ~pm
            Ay = Ad[np.ix_(y, y)]
            By = Ad[np.ix_(pm, y)]
            sigma = np.trace(By @ np.linalg.solve(Ay, By.T)) / pm.sum()
            self.Kdef = Ad + sigma * np.outer(self.v, self.v)
        else:
            self.lu = spla.splu(A.tocsc())

    def solve(self, r):
        if self.dense:
            vr = self.v @ r
            y = np.linalg.solve(self.Kdef, r - vr * self.v)
            return y + (vr / (-self.gamma)) * self.v
        return self.lu.solve(r)


def reversed_rows(A):
    """The same CSR matrix with every row stored in reverse column order, so that a matvec sums
    each row in the opposite order (an equally legal fp64 evaluation; used by alt_order)."""
    B = A.copy()
    for i in range(B.shape[0]):
        s, e = B.indptr[i], B.indptr[i + 1]
        B.indices[s:e] = B.indices[s:e][::-1].copy()
        B.data[s:e] = B.data[s:e][::-1].copy()
    B.has_sorted_indices = False
    return B


class Hierarchy:
    """Per-level operators, transfers and smoothers.

    relax: 'vanka', 'bsr' (inexact BSR) or 'bsr_exact' (exact BSR).  levels = number
    of levels L (level 0 finest).  quadrature: 'rq' (A^RQ, eq. block_form_rq) or 'exact' (A of
    eq. block_form) on every level.
    alt_order=True builds the same method with every summation order reversed (CSR rows,
    patch DoF order, hence the pivot order of the patch solves): the spread between the two
    runs calibrates the fp64 rounding floor of the parity criterion (SURVEY.md 8(c) c-11,
    DESIGN.md reading A22).  It changes no arithmetic of the method."""

    def __init__(self, n, levels, lam, mu, tau, alpha, inv_M, mu_f=1.0, K=1.0, Kinv_field=None,
                 relax="vanka", alt_order=False, quadrature="rq"):
        if levels < 1 or n % (2 ** (levels - 1)) != 0 or n // (2 ** (levels - 1)) < 2:
            raise ValueError("n must be divisible by 2^(levels-1) with coarsest n >= 2")
        self.levels = levels
        self.meshes, self.ops, self.transfers, self.smoothers = [], [], [], []
        Kinv = Kinv_field
        for l in range(levels):
            m = Mesh(n // 2 ** l)
            if l > 0 and Kinv is not None:
                Kinv = coarsen_Kinv(self.meshes[-1], m, Kinv)
            op = Operator(m, lam, mu, tau, alpha, inv_M, mu_f, K=K, Kinv_field=Kinv, quadrature=quadrature)
            self.meshes.append(m)
            self.ops.append(op)
            if l > 0:
                self.transfers.append(Transfer(self.meshes[l - 1], m))
        self.relax = relax
        for l in range(levels - 1):
            if relax == "vanka":
                pat = [p[::-1] for p in vertex_patches(self.meshes[l], "full")] if alt_order else None
                self.smoothers.append(Vanka(self.ops[l], pat))
            else:
                self.smoothers.append(BSR(self.ops[l], reverse=alt_order, exact=relax == "bsr_exact"))
        self.coarse = CoarseSolver(self.ops[-1])
        if alt_order:
            for op in self.ops:
                op.A = reversed_rows(op.A)
            for tr in self.transfers:
                tr.P = reversed_rows(tr.P)
                tr.R = reversed_rows(tr.R)

    def smooth(self, l, x, b, opts):
        if self.relax == "vanka":
            return self.smoothers[l].sweep(x, b, opts["omega"])
        return self.smoothers[l].sweep(x, b, opts["omega"], opts.get("omega_J", 1.0), opts.get("jacobi_sweeps", 1))

    def cycle(self, x, b, opts, l=0):
        """One V(nu1, nu2) cycle on level l."""
        if l == self.levels - 1:
            return self.coarse.solve(b)
        for _ in range(opts["nu1"]):
            x = self.smooth(l, x, b, opts)
        r = b - self.ops[l].A @ x
        bc = self.transfers[l].restrict(r)
        xc = self.cycle(np.zeros_like(bc), bc, opts, l + 1)
        x = x + self.transfers[l].prolong(xc)
        for _ in range(opts["nu2"]):
            x = self.smooth(l, x, b, opts)
        return x

    def residual_norm(self, x, b):
        return float(np.linalg.norm(b - self.ops[0].A @ x))

    def solve(self, x, b, opts, rtol=None, max_cycles=20):
        """Stationary iteration of V-cycles.  history[0] = ||b - A x0||."""
        hist = [self.residual_norm(x, b)]
        for _ in range(max_cycles):
            x = self.cycle(x, b, opts)
            hist.append(self.residual_norm(x, b))
            if rtol is not None and hist[-1] <= rtol * hist[0]:
                break
        return x, np.array(hist)

    def measure_rho(self, opts, seed=0, max_cycles=200, min_cycles=30, tol=1e-3):
        """rho_N of PAPER.md:809-811: zero RHS, random initial guess."""
        rng = np.random.Generator(np.random.PCG64(seed))
        N = self.ops[0].A.shape[0]
        x = rng.uniform(-1.0, 1.0, N)
        b = np.zeros(N)
        prev_r = self.residual_norm(x, b)
        rhos = []
        for k in range(max_cycles):
            x = self.cycle(x, b, opts)
            r = self.residual_norm(x, b)
            rhos.append(r / prev_r)
            prev_r = r
            if len(rhos) >= min_cycles and abs(rhos[-1] - rhos[-2]) < tol:
                break
            if not np.isfinite(r) or r == 0.0:
                break
        return rhos[-1], np.array(rhos)


def lame(E, nu):
    """mu = E/(2+2nu), lambda = E nu / ((1-2nu)(1+nu))."""
    return E / (2.0 + 2.0 * nu), E * nu / ((1.0 - 2.0 * nu) * (1.0 + nu))

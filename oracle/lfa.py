"""Two-grid local Fourier analysis (ORACLE -- test infrastructure only).

LFA (Defs. at PAPER.md:708-712 and 741-747): on the infinite uniform grid every
operator of the two-grid method is invariant under index shifts (by one fine index for A_h and
the smoother, by one coarse index = two fine indices for P and R), so the span of the four
harmonics e^{i theta^alpha . x} (theta^alpha = theta + alpha pi, alpha in {0,1}^2, theta in
[-pi/2, pi/2)^2) times the 10 DoF kinds of the unit cell is invariant under

    E_TG = S^{nu2} (I - P A_H^{-1} R A_h) S^{nu1}        (eq. TG-Operator-Biot)

and the restriction of E_TG to it is a 40 x 40 matrix.  rho_LFA = sup_theta rho(E_TG(theta))
(PAPER.md:741-747), S = I - omega C A_h with C the smoother's correction operator (additive Vanka
M^{-1}, PAPER.md:577-590 / Appendix C; inexact Braess-Sarazin, PAPER.md:654-686 / Appendix E).

Reading A27: the printed symbols of Appendices A-E are garbled (SURVEY.md reading A3),
so no symbol is typed in from the paper.  Each symbol is read off the oracle's own assembled
operators, far from the boundary: the columns of A_h, C (applied to unit vectors), A_H and P at
one interior index give the stencil, and the symbol is the stencil's Fourier sum.  The phases use
the DoF's cell index (i, j) rather than its geometric position; that is a fixed diagonal
similarity of all 40 x 40 matrices per theta and leaves every spectral radius unchanged.

Symbols (x0 the interior fine index, X0 = x0 / 2 the coarse one, d index offsets):
  B~(theta)[q, q']   = sum_d B[(q, x0 + d), (q', x0)] e^{-i theta . d}        (A_h, C; A_H at 2 theta)
  P~_alpha[q, q']    = 1/4 sum_d P[(q, 2 X0 + d), (q', X0)] e^{-i theta^alpha . d}
  R~_alpha[q', q]    = sum_d P[(q, 2 X0 + d), (q', X0)] e^{+i theta^alpha . d}   (R = P^T)
"""
from __future__ import annotations

import numpy as np

from .mesh import Mesh
from .fem import Operator
from .transfer import Transfer
from .relax import Vanka, BSR

ALPHAS = ((0, 0), (1, 0), (0, 1), (1, 1))


def _columns(apply, mesh, i0, j0):
    """Stencil of a linear, shift-invariant operator given as apply(active vector) -> active
    vector: a list over source kinds q' of (kinds q, offsets d (m, 2), values) of its column at
    DoF (q', i0, j0)."""
    N1 = mesh.N1
    kind_of = np.repeat(np.arange(10), N1 * N1)
    ii = np.tile(np.arange(N1), 10 * N1)
    jj = np.tile(np.repeat(np.arange(N1), N1), 10)
    act = mesh.act_idx
    cols = []
    for qp in range(10):
        e = np.zeros(mesh.nact)
        p = mesh.pos[mesh.slot(qp, i0, j0)]
        assert p >= 0, "the stencil centre must be an active (interior) DoF"
        e[p] = 1.0
        c = apply(e)
        nz = np.nonzero(c)[0]
        s = act[nz]
        d = np.stack([ii[s] - i0, jj[s] - j0], axis=1)
        cols.append((kind_of[s], d, c[nz]))
    return cols


def _symbol(cols, theta, sign=-1.0, scale=1.0):
    """Fourier sum of a column stencil at the frequencies theta (T, 2): (T, 10, 10), rows the
    kinds of the output grid."""
    theta = np.atleast_2d(np.asarray(theta, float))
    out = np.zeros((theta.shape[0], 10, 10), dtype=complex)
    for qp, (q, d, v) in enumerate(cols):
        ph = scale * v[None, :] * np.exp(sign * 1j * (theta @ d.T))        # (T, m)
        for k in np.unique(q):
            out[:, k, qp] = ph[:, q == k].sum(axis=1)
    return out


def _prolong_columns(P, fine, coarse, X0, Y0):
    """Columns of P (fine active x coarse active) at coarse DoFs (q', X0, Y0), as fine stencils
    around (2 X0, 2 Y0)."""
    N1 = fine.N1
    kind_of = np.repeat(np.arange(10), N1 * N1)
    ii = np.tile(np.arange(N1), 10 * N1)
    jj = np.tile(np.repeat(np.arange(N1), N1), 10)
    cols = []
    for qp in range(10):
        e = np.zeros(coarse.nact)
        p = coarse.pos[coarse.slot(qp, X0, Y0)]
        assert p >= 0
        e[p] = 1.0
        c = P @ e
        nz = np.nonzero(c)[0]
        s = fine.act_idx[nz]
        d = np.stack([ii[s] - 2 * X0, jj[s] - 2 * Y0], axis=1)
        cols.append((kind_of[s], d, c[nz]))
    return cols


class TwoGridLFA:
    """Symbols of the two-grid method the oracle builds (the two levels of oracle.cycle.Hierarchy:
    Operator on both meshes, Transfer, Vanka or BSR on the fine one).

    relax='vanka' or 'bsr' (then omega_J, jacobi_sweeps as in Hierarchy.smooth).  The stencils are
    read at the centre (n/2, n/2) of an n x n patch of mesh; h (default 1/n) is the fine spacing
    the symbols are for -- the element integrals only see the vertex coordinates i h, so a small
    patch of a fine mesh gives the interior stencils of the unit square at 1/h cells (the prolongation
    weights are scale invariant, oracle.transfer.build_P).  n = 16 leaves every stencil (radius <= 3
    indices for C) clear of the patch boundary."""

    def __init__(self, n, lam, mu, tau, alpha, inv_M, mu_f=1.0, K=1.0, relax="vanka",
                 omega_J=None, jacobi_sweeps=1, h=None):
        if n % 4 != 0 or n < 16:
            raise ValueError("n must be a multiple of 4, n >= 16")
        fine, coarse = Mesh(n), Mesh(n // 2)
        if h is not None:
            fine.h, coarse.h = h, 2.0 * h
        self.h = fine.h
        op_f = Operator(fine, lam, mu, tau, alpha, inv_M, mu_f, K=K)
        op_c = Operator(coarse, lam, mu, tau, alpha, inv_M, mu_f, K=K)
        x0 = n // 2
        self.relax = relax
        self.A_cols = _columns(lambda e: op_f.A @ e, fine, x0, x0)
        self.AH_cols = _columns(lambda e: op_c.A @ e, coarse, x0 // 2, x0 // 2)
        self.P_cols = _prolong_columns(Transfer(fine, coarse).P, fine, coarse, x0 // 2, x0 // 2)
        self._fine, self._x0, self.jacobi_sweeps = fine, x0, jacobi_sweeps
        if relax == "vanka":
            self.C_cols = _columns(Vanka(op_f).apply_Minv, fine, x0, x0)         # C = M^{-1}
        else:
            if omega_J is None:
                raise ValueError("bsr needs omega_J")
            self._bsr = BSR(op_f)
            self.set_omega_J(omega_J)

    def set_omega_J(self, omega_J):
        """BSR: the correction operator C(omega_J) = one sweep from x = 0 with omega = 1, which is
        linear in the residual."""
        sm, fine = self._bsr, self._fine
        z = np.zeros(fine.nact)
        self.omega_J = omega_J
        self.C_cols = _columns(lambda e: sm.sweep(z, e, 1.0, omega_J, self.jacobi_sweeps),
                               fine, self._x0, self._x0)

    # ---- symbols (theta: (T, 2) batch, or one (2,) frequency) ------------------------------
    def A(self, theta):
        return _symbol(self.A_cols, theta)

    def C(self, theta):
        return _symbol(self.C_cols, theta)

    def A_H(self, theta):
        """Coarse operator symbol at the coarse frequency 2 theta."""
        return _symbol(self.AH_cols, 2.0 * np.atleast_2d(np.asarray(theta, float)))

    def P(self, theta):
        """(T, 40, 10): the four harmonic blocks P~_alpha stacked (alpha in ALPHAS order)."""
        th = np.atleast_2d(np.asarray(theta, float))
        return np.concatenate([_symbol(self.P_cols, th + np.pi * np.array(a), -1.0, 0.25)
                               for a in ALPHAS], axis=1)

    def R(self, theta):
        """(T, 10, 40), R = P^T: the blocks R~_alpha side by side."""
        th = np.atleast_2d(np.asarray(theta, float))
        return np.concatenate([_symbol(self.P_cols, th + np.pi * np.array(a), +1.0).transpose(0, 2, 1)
                               for a in ALPHAS], axis=2)

    def E_TG(self, theta, omega, nu1, nu2):
        """(T, 40, 40) two-grid error propagation symbols."""
        th = np.atleast_2d(np.asarray(theta, float))
        T = th.shape[0]
        Ah = np.zeros((T, 40, 40), dtype=complex)
        Ch = np.zeros((T, 40, 40), dtype=complex)
        for k, a in enumerate(ALPHAS):
            ta = th + np.pi * np.array(a)
            Ah[:, 10 * k:10 * k + 10, 10 * k:10 * k + 10] = self.A(ta)
            Ch[:, 10 * k:10 * k + 10, 10 * k:10 * k + 10] = self.C(ta)
        I = np.eye(40)
        S = I - omega * Ch @ Ah
        K = I - self.P(th) @ np.linalg.solve(self.A_H(th), self.R(th) @ Ah)
        return np.linalg.matrix_power(S, nu2) @ K @ np.linalg.matrix_power(S, nu1)

    @staticmethod
    def thetas(m=32):
        """m x m grid of theta in [-pi/2, pi/2)^2 shifted by half a step, so that theta = 0
        (where A_H is singular) is never sampled (discrete sampling; PAPER.md:822:
        32 points per direction, offset from the origin)."""
        t = -np.pi / 2 + (np.arange(m) + 0.5) * np.pi / m
        t1, t2 = np.meshgrid(t, t, indexing="ij")
        return np.stack([t1.ravel(), t2.ravel()], axis=1)

    def rho(self, omega, nu1, nu2, m=32):
        """rho_LFA = max over the sampled theta of the spectral radius of E_TG(theta)."""
        E = self.E_TG(self.thetas(m), omega, nu1, nu2)
        return float(np.abs(np.linalg.eigvals(E)).max())

    def optimize(self, omegas, nu1, nu2, m=32):
        """Brute-force parameter choice: the omega of the grid with the
        smallest rho_LFA, and that rho."""
        rs = [self.rho(w, nu1, nu2, m) for w in omegas]
        k = int(np.argmin(rs))
        return float(omegas[k]), rs[k]

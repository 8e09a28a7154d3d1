"""Flexible GMRES preconditioned by one multigrid V-cycle (ORACLE -- test infrastructure only).

PAPER.md:922 (sec. 5.1, 'Steady-State Model'): "a single four-level V-cycle of the monolithic
multigrid method as a preconditioner for FGMRES using a relative residual stopping tolerance"; the
timing tables (tab:time_vanka_redisc, tab:time_bsr_redisc, tab:mgtime) report its iterations.  The
preconditioner applies one V-cycle from a zero initial guess to the current Krylov vector, z = B(v).

Textbook right-preconditioned flexible GMRES(m) (Saad, 'A flexible inner-outer preconditioned GMRES
algorithm', 1993): Arnoldi with modified Gram-Schmidt on w = A z_j, Givens rotations on the
Hessenberg matrix, x = x0 + Z y at restarts and at the end.  history[i] is the Euclidean residual
norm estimate |g_{i}| after i inner iterations (history[0] = ||b - A x0||), which equals
||b - A x_i|| in exact arithmetic.
"""
from __future__ import annotations

import numpy as np


def fgmres(A, b, x0, precond, rtol=1e-6, max_iters=100, restart=30):
    """A: callable x -> A x; precond: callable v -> z (one V-cycle from zero).  Returns (x, hist)."""
    x = x0.copy()
    r = b - A(x)
    beta = np.linalg.norm(r)
    hist = [beta]
    if beta == 0.0:
        return x, np.array(hist)
    target = rtol * beta
    iters = 0
    while iters < max_iters:
        m = min(restart, max_iters - iters)
        V = [r / beta]
        Z = []
        Hm = np.zeros((m + 1, m))
        cs, sn = np.zeros(m), np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        k = 0
        for j in range(m):
            z = precond(V[j])
            Z.append(z)
            w = A(z)
            for i in range(j + 1):                     # modified Gram-Schmidt
                Hm[i, j] = np.dot(w, V[i])
                w = w - Hm[i, j] * V[i]
            Hm[j + 1, j] = np.linalg.norm(w)
            V.append(w / Hm[j + 1, j] if Hm[j + 1, j] != 0.0 else w)
            for i in range(j):                         # previous rotations
                t = cs[i] * Hm[i, j] + sn[i] * Hm[i + 1, j]
                Hm[i + 1, j] = -sn[i] * Hm[i, j] + cs[i] * Hm[i + 1, j]
                Hm[i, j] = t
            d = np.hypot(Hm[j, j], Hm[j + 1, j])
            cs[j], sn[j] = Hm[j, j] / d, Hm[j + 1, j] / d
            Hm[j, j] = d
            Hm[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            k = j + 1
            iters += 1
            hist.append(abs(g[j + 1]))
            if hist[-1] <= target:
                break
        y = np.linalg.solve(np.triu(Hm[:k, :k]), g[:k])
        x = x + np.stack(Z[:k], axis=1) @ y
        r = b - A(x)
        beta = np.linalg.norm(r)
        if hist[-1] <= target or beta == 0.0:
            break
    return x, np.array(hist)


def fgmres_mg(H, b, opts, rtol=1e-6, max_iters=100, restart=30, x0=None):
    """FGMRES on level 0 of an oracle Hierarchy, preconditioned by one V-cycle H.cycle(0, v)."""
    A = lambda v: H.ops[0].A @ v
    M = lambda v: H.cycle(np.zeros_like(v), v, opts)
    return fgmres(A, b, np.zeros_like(b) if x0 is None else x0, M, rtol, max_iters, restart)

"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no operator, no transfer, no
relaxation).  It only draws the random inputs BASELINE.json's configs name and
states which slots of the ABI vector layout are degrees of freedom, so that the
oracle (``oracle/``) and the GPU path consume byte-identical inputs.

Vector layout (SURVEY.md §8 "Common data layout"): one level
vector is 10 planes of (n+1) x (n+1) values, plane-major, row j then column i
(entry [k, j, i]).  Plane meaning:

====  =================================================  ========================
plane DoF                                                active when
====  =================================================  ========================
0/1   u_x / u_y, P1 at vertex (i,j)                       0<i<n and 0<j<n
2     bubble, horizontal edge (i,j)-(i+1,j)               i<n, 0<j<n
3     bubble, vertical edge (i,j)-(i,j+1)                 0<i<n, j<n
4     bubble, diagonal edge (i+1,j)-(i,j+1)               i<n, j<n
5/6/7 RT0 on the same H / V / D edges                     as planes 2 / 3 / 4
8/9   P0 on lower-left / upper-right triangle of cell     i<n, j<n
====  =================================================  ========================

The active set is the Dirichlet condition u = 0, w.n = 0 on the boundary of
the unit square (PAPER.md:936-945 steady test; BASELINE.json configs).

Recipe: b = Generator(PCG64(seed)).uniform
(-1, 1) over all 10 (n+1)^2 slots in the order above, inactive slots then set to
0.  Heterogeneous permeability (config 4): K_T = exp(Z_T) with
Z = Generator(PCG64(seed)).normal(0, 2, size=(2, n, n)) (planes LL, UR; [plane,
j, i]).
"""
from __future__ import annotations

import numpy as np

NPLANES = 10


def active_mask(n: int) -> np.ndarray:
    """Boolean (10, n+1, n+1) mask of the slots that are unknowns at mesh size n."""
    m = np.zeros((NPLANES, n + 1, n + 1), dtype=bool)
    j, i = np.meshgrid(np.arange(n + 1), np.arange(n + 1), indexing="ij")
    vert = (i > 0) & (i < n) & (j > 0) & (j < n)
    hedge = (i < n) & (j > 0) & (j < n)
    vedge = (i > 0) & (i < n) & (j < n)
    cell = (i < n) & (j < n)
    m[0] = vert
    m[1] = vert
    m[2] = hedge
    m[3] = vedge
    m[4] = cell
    m[5] = hedge
    m[6] = vedge
    m[7] = cell
    m[8] = cell
    m[9] = cell
    return m


def n_active(n: int) -> int:
    """Number of unknowns, 10 n^2 - 8 n + 2."""
    return 10 * n * n - 8 * n + 2


def uniform_rhs(n: int, seed: int) -> np.ndarray:
    """b ~ U(-1,1) on every slot from PCG64(seed), inactive slots zeroed. Shape (10, n+1, n+1)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    b = rng.uniform(-1.0, 1.0, size=NPLANES * (n + 1) * (n + 1)).reshape(NPLANES, n + 1, n + 1)
    b[~active_mask(n)] = 0.0
    return b


def uniform_vector(n: int, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """Generic seeded test vector on the active slots (used for x in parity tests)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    v = rng.uniform(lo, hi, size=NPLANES * (n + 1) * (n + 1)).reshape(NPLANES, n + 1, n + 1)
    v[~active_mask(n)] = 0.0
    return v


def lognormal_K(n: int, seed: int, sigma: float = 2.0) -> np.ndarray:
    """Per-triangle permeability K_T = exp(N(0, sigma^2)); shape (2, n, n), planes (LL, UR), [plane, j, i]."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.exp(rng.normal(0.0, sigma, size=(2, n, n)))


# BASELINE.json configs.  1/M = 1 and mu_f = 1 (readings A5, A6 of DESIGN.md;
# with 1/M = 1e-6 the rediscretised V-cycle diverges like 1/gamma at these parameters, see E0).
# omega / omega_J: the minimisers of experiment E0 (tests/scripts/e0_omega_scan.py,
# tests/golden/e0_omega_scan.json; V(1,1) on 64^2, 5 levels): Vanka 0.74 (configs 1/2),
# 0.70 (configs 3, 5); BSR (omega_J, omega) = (1.0, 0.75) (config 2) and (0.7, 0.3) for the
# heterogeneous config 4, where every scanned pair diverges (reading A24).
CONFIGS = {
    1: dict(n=16, levels=3, lam=1.0, mu=1.0, K=1.0, tau=1.0, alpha=1.0, inv_M=1.0, mu_f=1.0,
            b_seed=0, K_seed=None, relax="vanka", cycles=10, omega=0.74),
    2: dict(n=256, levels=7, lam=1.0, mu=1.0, K=1.0, tau=1.0, alpha=1.0, inv_M=1.0, mu_f=1.0,
            b_seed=1, K_seed=None, relax="vanka+bsr", cycles=20, omega=0.74, bsr_omega=0.75, omega_J=1.0),
    3: dict(n=1024, levels=9, lam=1e6, mu=1.0, K=1e-6, tau=1.0, alpha=1.0, inv_M=1.0, mu_f=1.0,
            b_seed=2, K_seed=None, relax="vanka", rtol=1e-8, omega=0.70),
    4: dict(n=2048, levels=10, lam=1.0, mu=1.0, K=None, tau=1.0, alpha=1.0, inv_M=1.0, mu_f=1.0,
            b_seed=4, K_seed=3, relax="bsr", cycles=20, bsr_omega=0.3, omega_J=0.7),
    5: dict(n=4096, levels=11, lam=100.0, mu=1.0, K=1e-2, tau=1.0, alpha=1.0, inv_M=1.0, mu_f=1.0,
            b_seed=5, K_seed=None, relax="vanka", rtol=1e-8, omega=0.70),
}

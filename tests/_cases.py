"""Shared helpers for the GPU parity tests: oracle objects and array conversions.

Only tests import this (it imports the oracle)."""
import functools

import numpy as np

import mg_inputs
from oracle.cycle import Hierarchy as OHierarchy
from oracle.fem import Operator
from oracle.mesh import Mesh

# named parameter sets (lambda, mu, K, tau, alpha, inv_M)
PARAMS = {
    "unit": (1.0, 1.0, 1.0, 1.0, 1.0, 1.0),             # BASELINE configs 1/2
    "stiff": (1e6, 1.0, 1e-6, 1.0, 1.0, 1.0),           # config 3 regime
    "cfg5": (100.0, 1.0, 1e-2, 1.0, 1.0, 1.0),          # config 5 regime
    "mixed": (2.5, 0.7, 0.3, 0.8, 1.3, 0.05),           # generic values, every term distinct
}


@functools.lru_cache(maxsize=None)
def mesh(n):
    return Mesh(n)


@functools.lru_cache(maxsize=None)
def operator(n, pname, het_seed=None):
    lam, mu, K, tau, alpha, invM = PARAMS[pname]
    kinv = None if het_seed is None else 1.0 / mg_inputs.lognormal_K(n, het_seed)
    return Operator(mesh(n), lam, mu, tau, alpha, invM, 1.0, K=K, Kinv_field=kinv)


@functools.lru_cache(maxsize=None)
def hierarchy(n, levels, pname, relax, het_seed=None):
    lam, mu, K, tau, alpha, invM = PARAMS[pname]
    kinv = None if het_seed is None else 1.0 / mg_inputs.lognormal_K(n, het_seed)
    return OHierarchy(n, levels, lam, mu, tau, alpha, invM, 1.0, K=K, Kinv_field=kinv, relax=relax)


def small_coarse_levels(n, min_levels=1):
    """Levels for a test of level-0 (or level 0 -> 1) operations: the fewest levels >= min_levels
    whose coarsest n_c is either > 20 (mg_setup builds no dense coarsest inverse) or <= 8, so the
    host's dense inverse (O(n_c^6) work for 8 < n_c <= 20) stays small; the operations under
    test do not depend on the levels below."""
    L, m = 1, n
    while True:
        if L >= min_levels and (m > 20 or m <= 8):
            return L
        if m % 2 or m // 2 < 2:
            return max(L, min_levels)
        m //= 2
        L += 1


def gpu_hierarchy(n, levels, pname, het_seed=None, march=False, env=None):
    """march=True forces the row-marching TMA kernels (production path of the levels with n >= 512)
    on every level, so that small parity cases exercise them (MG_MARCH_MIN_N is read by mg_setup);
    env: further MG_* knobs read at setup (e.g. MG_FUSE_PROLONG)."""
    import os
    from paper_2107_04060_b200 import Hierarchy
    knobs = dict(env or {})
    if march:
        knobs["MG_MARCH_MIN_N"] = "0"
    os.environ.update(knobs)
    lam, mu, K, tau, alpha, invM = PARAMS[pname]
    kf = None if het_seed is None else mg_inputs.lognormal_K(n, het_seed)
    try:
        return Hierarchy(n, levels, lam, mu, K=K, tau=tau, alpha=alpha, inv_M=invM, mu_f=1.0, K_field=kf)
    finally:
        for k in knobs:
            os.environ.pop(k, None)


def abs_matvec(op, x):
    """|A| |x| on the active vector (the rounding scale of one residual evaluation)."""
    A = op.A.copy()
    A.data = np.abs(A.data)
    return A @ np.abs(x)


def block_rel_err(m, a, b):
    """Relative errors per block (u: planes 0-4, w: 5-7, p: 8-9) of two (10, n+1, n+1) arrays."""
    out = {}
    for name, sl in (("u", slice(0, 5)), ("w", slice(5, 8)), ("p", slice(8, 10))):
        d = np.linalg.norm((a[sl] - b[sl]).ravel())
        s = np.linalg.norm(b[sl].ravel())
        out[name] = d / s if s > 0 else d
    return out

"""The exact-integration operator A of eq. block_form (lambda (div u, div v) integrated exactly,
PAPER.md:143-167) and exact Braess-Sarazin relaxation (S dp = g solved exactly)
on the GPU against the oracle (Operator(quadrature="exact"), BSR(exact=True)).

Tolerances as test_gpu_parity.py: residual componentwise 32 u (|b| + |A||x|); one sweep relative
to the result in the max norm (1e-11; exact BSR 1e-10: the device CG stops at 1e-14 in the
D_S^{-1} norm, the oracle uses sparse LU); cycle histories with the SURVEY 8c-11 floor.
"""
import functools

import numpy as np
import pytest

import mg_inputs
from tests import _cases as C
from tests.test_gpu_parity import _inactive_zero

pytestmark = pytest.mark.gpu
U = 2.0 ** -53


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@functools.lru_cache(maxsize=None)
def _op(n, pname):
    from oracle.fem import Operator
    lam, mu, K, tau, alpha, invM = C.PARAMS[pname]
    return Operator(C.mesh(n), lam, mu, tau, alpha, invM, 1.0, K=K, quadrature="exact")


def _gpu(n, levels, pname):
    from paper_2107_04060_b200 import Hierarchy
    lam, mu, K, tau, alpha, invM = C.PARAMS[pname]
    return Hierarchy(n, levels, lam, mu, K=K, tau=tau, alpha=alpha, inv_M=invM, mu_f=1.0, quadrature="exact")


@pytest.mark.parametrize("n,pname", [(8, "mixed"), (16, "unit"), (40, "cfg5"), (66, "stiff")])
def test_exact_residual(n, pname):
    torch = _torch()
    H = _gpu(n, C.small_coarse_levels(n), pname)
    op = _op(n, pname)
    m = C.mesh(n)
    x = mg_inputs.uniform_vector(n, 81)
    b = mg_inputs.uniform_rhs(n, 82)
    xd, bd, rd = H.to_device(x), H.to_device(b), H.zeros()
    H.residual(0, xd, bd, rd)
    torch.cuda.synchronize()
    rG = m.to_active(H.to_host(rd))
    xa, ba = m.to_active(x), m.to_active(b)
    rO = ba - op.A @ xa
    scale = np.abs(ba) + C.abs_matvec(op, xa)
    assert np.all(np.abs(rG - rO) <= 32 * U * scale)
    # the exact and RQ operators differ exactly in the bubble rows
    rq = C.operator(n, pname)
    d = np.abs(op.A @ xa - rq.A @ xa)
    kind = m.slot_kind(m.act_idx)
    assert np.all(d[(kind < 2) | (kind > 4)] <= 1e-12 * (1 + np.abs(op.A @ xa).max()))
    _inactive_zero(H, rd)


@pytest.mark.parametrize("n,pname,omega", [(8, "mixed", 0.8), (16, "unit", 0.74), (40, "cfg5", 0.7)])
def test_exact_vanka_sweep(n, pname, omega):
    torch = _torch()
    from oracle.relax import Vanka
    H = _gpu(n, C.small_coarse_levels(n), pname)
    V = Vanka(_op(n, pname))
    m = C.mesh(n)
    x = mg_inputs.uniform_vector(n, 83)
    b = mg_inputs.uniform_rhs(n, 84)
    xd, bd = H.to_device(x), H.to_device(b)
    H.relax_vanka(0, xd, bd, omega, sweeps=1)
    torch.cuda.synchronize()
    xO = m.from_active(V.sweep(m.to_active(x), m.to_active(b), omega))
    err = np.abs(H.to_host(xd) - xO).max() / np.abs(xO).max()
    assert err <= 1e-11, err


@pytest.mark.parametrize("n,pname,quad", [(8, "mixed", "exact"), (16, "unit", "rq"), (32, "unit", "exact"),
                                          (40, "cfg5", "rq")])
def test_exact_bsr_sweep(n, pname, quad):
    torch = _torch()
    from oracle.relax import BSR
    from paper_2107_04060_b200 import Hierarchy
    lam, mu, K, tau, alpha, invM = C.PARAMS[pname]
    H = Hierarchy(n, C.small_coarse_levels(n), lam, mu, K=K, tau=tau, alpha=alpha, inv_M=invM, quadrature=quad)
    op = _op(n, pname) if quad == "exact" else C.operator(n, pname)
    S = BSR(op, exact=True)
    m = C.mesh(n)
    x = mg_inputs.uniform_vector(n, 85)
    b = mg_inputs.uniform_rhs(n, 86)
    xd, bd = H.to_device(x), H.to_device(b)
    rc, its = H.relax_bsr_exact(0, xd, bd, 0.8, sweeps=1)
    torch.cuda.synchronize()
    print(n, pname, quad, "CG iterations", its)
    assert rc == 0 and 0 < its <= 24 * n + 64            # converged to the tolerance, not at the cap
    xO = m.from_active(S.sweep(m.to_active(x), m.to_active(b), 0.8, 0.0, 0))
    err = np.abs(H.to_host(xd) - xO).max() / np.abs(xO).max()
    assert err <= 1e-10, err


@pytest.mark.parametrize("relax,quad,nu,omega,cycles,n", [("vanka", "exact", 0.49, 0.7, 8, 32),
                                                          ("bsr_exact", "rq", 0.4, 0.8, 6, 16),
                                                          ("bsr", "exact", 0.4, 0.7, 8, 16),
                                                          ("bsr_exact", "exact", 0.2, 0.8, 6, 16)])
def test_exact_two_grid_history(relax, quad, nu, omega, cycles, n):
    """Two-grid V(2,2) / V(1,1) histories at the paper's tab:naive parameters (E = 3e4, k = 1e-6,
    tau = 1, M = 1e6), h = 1/32 and 1/16 (the dense coarsest inverse of the 16^2 grid
    takes ~50 s of host long-double work per context, so only one case keeps h = 1/32): zero RHS, the
    oracle's random x_0."""
    torch = _torch()
    from oracle.cycle import Hierarchy as OH, lame
    from paper_2107_04060_b200 import Hierarchy, Opts
    mu, lam = lame(3e4, nu)
    od = dict(nu1=2, nu2=2, omega=omega) if relax == "vanka" else dict(nu1=1, nu2=1, omega=omega, omega_J=1.0,
                                                                         jacobi_sweeps=1)
    go = Opts(od["nu1"], od["nu2"], relax, omega, 1.0, 1)
    Oh = OH(n, 2, lam, mu, 1.0, 1.0, 1e-6, 1.0, K=1e-6, relax=relax, quadrature=quad)
    Oa = OH(n, 2, lam, mu, 1.0, 1.0, 1e-6, 1.0, K=1e-6, relax=relax, quadrature=quad, alt_order=True)
    m = Oh.meshes[0]
    rng = np.random.Generator(np.random.PCG64(0))
    x0 = rng.uniform(-1.0, 1.0, Oh.ops[0].A.shape[0])
    b = np.zeros_like(x0)
    hO, hA, xo, xa = [], [], x0.copy(), x0.copy()
    for _ in range(cycles):
        xo = Oh.cycle(xo, b, od)
        xa = Oa.cycle(xa, b, od)
        hO.append(Oh.residual_norm(xo, b))
        hA.append(Oa.residual_norm(xa, b))
    hO, hA = np.array(hO), np.array(hA)
    H = Hierarchy(n, 2, lam, mu, K=1e-6, tau=1.0, alpha=1.0, inv_M=1e-6, quadrature=quad)
    xd, bd = H.to_device(m.from_active(x0)), H.zeros()
    hG = np.array([H.cycle(xd, bd, go) for _ in range(cycles)])
    F = 4 * np.abs(hO - hA) + 8 * U * np.linalg.norm(C.abs_matvec(Oh.ops[0], np.abs(xo)))
    print(relax, quad, nu, "rho", hO[1:] / hO[:-1], "rel dev", np.abs(hG - hO) / hO)
    tol = 1e-10 if relax != "bsr_exact" else 1e-8      # CG to 1e-14 vs LU, amplified by the cycle
    assert np.all(np.abs(hG - hO) <= tol * hO + F)
    assert np.all(np.abs(hG[1:] / hG[:-1] - hO[1:] / hO[:-1]) <= 1e-3)

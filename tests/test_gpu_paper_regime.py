"""GPU parity in the paper's own parameter regime ("What's missing" 4): the steady
test of PAPER.md:936-945 -- E = 3e4 (mu = E/(2+2nu), lambda = E nu/((1-2nu)(1+nu))),
alpha = mu_f = tau = 1, M = 1e6, K = 1e-6 I, the FE load vector of the
manufactured solution u = curl[xy(1-x)(1-y)]^2, p = 1 assembled by the oracle -- at N = 17 and 33
with coarsest h = 1/8, the tab:mgtime setting.

Here 1/M = 1e-6, so every patch's constant-pressure eigenvalue is gamma = (1/M) h^2/2 ~ 1e-9..2e-9
and the coarsest one ~ 8e-9: the exact deflation of reading A9 carries the solve.  The
cycles are tab:mgtime's: Vanka V(2,2) at tab:vanka22's omega (reading A25) and inexact BSR V(1,1) with
one Jacobi sweep at tab:bsr_vanka11's (omega_J, omega) for k = 1e-6.

Checks: the stationary cycle history against the oracle's (SURVEY 8c-11 floor, as in
test_gpu_parity.py), and the FGMRES(30) iteration count to 1e-6 equal to the
oracle's, with per-iteration estimates within 1e-9 relative + 4x the oracle's own spread.
"""
import functools

import numpy as np
import pytest

import mg_inputs

pytestmark = pytest.mark.gpu
U = 2.0 ** -53

OPTS = {  # tab:vanka22 / tab:bsr_vanka11 at k = 1e-6
    (0.4, "vanka"): dict(nu1=2, nu2=2, omega=0.80),
    (0.4, "bsr"): dict(nu1=1, nu2=1, omega=0.74, omega_J=0.94, jacobi_sweeps=1),
    (0.499, "vanka"): dict(nu1=2, nu2=2, omega=0.72),
    (0.499, "bsr"): dict(nu1=1, nu2=1, omega=0.68, omega_J=0.86, jacobi_sweeps=1),
}


def lame(E, nu):
    return E / (2.0 + 2.0 * nu), E * nu / ((1.0 - 2.0 * nu) * (1.0 + nu))


@functools.lru_cache(maxsize=None)
def _oracle(n, nu, relax, alt):
    from oracle.cycle import Hierarchy
    from oracle.manufactured import rhs
    mu, lam = lame(3e4, nu)
    H = Hierarchy(n, n.bit_length() - 3, lam, mu, 1.0, 1.0, 1e-6, 1.0, K=1e-6, relax=relax, alt_order=alt)
    return H, rhs(H.ops[0], mu, 1e-6)


def _gpu(n, nu):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2107_04060_b200 import Hierarchy
    mu, lam = lame(3e4, nu)
    return Hierarchy(n, n.bit_length() - 3, lam, mu, K=1e-6, tau=1.0, alpha=1.0, inv_M=1e-6, mu_f=1.0)


def _gopts(o, relax):
    from paper_2107_04060_b200 import Opts
    return Opts(o["nu1"], o["nu2"], relax, o["omega"], o.get("omega_J", 1.0), o.get("jacobi_sweeps", 1))


@pytest.mark.parametrize("n", [16, 32])
@pytest.mark.parametrize("nu", [0.4, 0.499])
@pytest.mark.parametrize("relax", ["vanka", "bsr"])
def test_paper_regime_cycle_history(n, nu, relax):
    Oh, b = _oracle(n, nu, relax, False)
    Oa, _ = _oracle(n, nu, relax, True)
    m = Oh.meshes[0]
    o = OPTS[(nu, relax)]
    cycles = 6
    xs, hO, hA, xa = [np.zeros_like(b)], [Oh.residual_norm(np.zeros_like(b), b)], [], np.zeros_like(b)
    hA.append(Oa.residual_norm(xa, b))
    for _ in range(cycles):
        xs.append(Oh.cycle(xs[-1], b, o))
        hO.append(Oh.residual_norm(xs[-1], b))
        xa = Oa.cycle(xa, b, o)
        hA.append(Oa.residual_norm(xa, b))
    hO, hA = np.array(hO), np.array(hA)
    A = Oh.ops[0].A.copy()
    A.data = np.abs(A.data)
    F = np.array([max(8 * U * np.linalg.norm(np.abs(b) + A @ np.abs(x)), 4 * abs(h - ha))
                  for x, h, ha in zip(xs, hO, hA)])
    H = _gpu(n, nu)
    xd, bd = H.to_device(np.zeros((10, n + 1, n + 1))), H.to_device(m.from_active(b))
    hG = [H.residual(0, xd, bd, norm=True)] + [H.cycle(xd, bd, _gopts(o, relax)) for _ in range(cycles)]
    hG = np.array(hG)
    dev = np.abs(hG - hO)
    print(n, nu, relax, "rel dev", dev / hO, "floor/h", F / hO)
    assert np.all(dev <= 1e-10 * hO + F), (dev / hO, F / hO)
    ok = hO[1:] >= 1e3 * F[1:]
    assert np.all(np.abs(hG[1:] / hG[:-1] - hO[1:] / hO[:-1])[ok] <= 1e-3)
    e_go = np.linalg.norm(m.to_active(H.to_host(xd)) - xs[-1]) / np.linalg.norm(xs[-1])
    e_oo = np.linalg.norm(xa - xs[-1]) / np.linalg.norm(xs[-1])
    assert e_go <= 1e-9 + 4 * e_oo, (e_go, e_oo)
    H.close()


@pytest.mark.parametrize("n", [16, 32])
@pytest.mark.parametrize("nu", [0.4, 0.499])
@pytest.mark.parametrize("relax", ["vanka", "bsr"])
def test_paper_regime_fgmres_iterations(n, nu, relax):
    """FGMRES(30) + one V-cycle per iteration to 1e-6 (tab:mgtime): the GPU takes
    exactly the oracle's iteration count, and its residual estimates follow the oracle's."""
    from oracle.krylov import fgmres_mg
    Oh, b = _oracle(n, nu, relax, False)
    Oa, _ = _oracle(n, nu, relax, True)
    m = Oh.meshes[0]
    o = OPTS[(nu, relax)]
    _, hO = fgmres_mg(Oh, b, o, rtol=1e-6, max_iters=100, restart=30)
    _, hA = fgmres_mg(Oa, b, o, rtol=1e-6, max_iters=100, restart=30)
    H = _gpu(n, nu)
    xd, bd = H.to_device(np.zeros((10, n + 1, n + 1))), H.to_device(m.from_active(b))
    rc, hG = H.fgmres(xd, bd, _gopts(o, relax), rtol=1e-6, max_iters=100, restart=30)
    print(n, nu, relax, "iterations GPU / oracle / alt", len(hG) - 1, len(hO) - 1, len(hA) - 1)
    assert rc == 0
    assert len(hG) == len(hO)
    k = min(len(hG), len(hA))
    F = 4 * np.abs(hA[:k] - hO[:k]) + 64 * U * np.linalg.norm(b)
    assert np.all(np.abs(hG[:k] - hO[:k]) <= 1e-9 * hO[:k] + F)
    H.close()

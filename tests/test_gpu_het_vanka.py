"""Heterogeneous-K additive Vanka on the GPU (reading A20 revised in DESIGN.md):
every vertex patch K_v = V_v A V_v^T of the operator with per-triangle K^{-1} in M_w, solved by the
condensed kernel (class-constant displacement/pressure part, per-vertex 6x6 RT0 Schur complement),
against the oracle's plain dense patch solves of the same patches (oracle/relax.py Vanka on an
Operator with a K field; its M_w per-triangle path is pinned by tests/test_oracle_coefficients.py).

Tolerances: one sweep is a linear map of the residual; max-norm error relative to the result
<= 1e-11 (1e-9 for the stiff lambda = 1e6, K = 1e-6 regime, as the scalar-K sweep test); cycles as
test_gpu_parity.test_cycle_history (SURVEY 8c-11 floor with the oracle's reversed-order spread).
"""
import numpy as np
import pytest

import mg_inputs
from tests import _cases as C
from tests.test_gpu_parity import _oracle_history, floor_parity, _inactive_zero

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.parametrize("n,pname,het,omega", [(4, "unit", 3, 0.74), (8, "mixed", 7, 0.9), (16, "unit", 3, 0.74),
                                                (40, "cfg5", 5, 0.7), (66, "mixed", 9, 0.8), (130, "unit", 3, 0.74),
                                                (24, "stiff", 11, 0.7)])
def test_het_vanka_sweep(n, pname, het, omega):
    torch = _torch()
    from oracle.relax import Vanka
    H = C.gpu_hierarchy(n, C.small_coarse_levels(n), pname, het)
    op = C.operator(n, pname, het)
    V = Vanka(op)
    m = C.mesh(n)
    x = mg_inputs.uniform_vector(n, 61)
    b = mg_inputs.uniform_rhs(n, 62)
    xd, bd = H.to_device(x), H.to_device(b)
    H.relax_vanka(0, xd, bd, omega, sweeps=1)
    torch.cuda.synchronize()
    xG = H.to_host(xd)
    xO = m.from_active(V.sweep(m.to_active(x), m.to_active(b), omega))
    err = np.abs(xG - xO).max() / np.abs(xO).max()
    assert err <= (1e-9 if pname == "stiff" else 1e-11), err
    _inactive_zero(H, xd)


@pytest.mark.parametrize("n,levels,pname,het,cycles", [(16, 3, "unit", 3, 8), (32, 4, "unit", 3, 8),
                                                       (32, 4, "mixed", 7, 6), (64, 5, "cfg5", 5, 5)])
def test_het_vanka_cycle_history(n, levels, pname, het, cycles):
    torch = _torch()
    from paper_2107_04060_b200 import Opts
    from oracle.cycle import Hierarchy as OH
    H = C.gpu_hierarchy(n, levels, pname, het)
    Oh = C.hierarchy(n, levels, pname, "vanka", het)
    lam, mu, K, tau, alpha, invM = C.PARAMS[pname]
    kinv = 1.0 / mg_inputs.lognormal_K(n, het)
    Oalt = OH(n, levels, lam, mu, tau, alpha, invM, 1.0, K=K, Kinv_field=kinv, relax="vanka", alt_order=True)
    m = Oh.meshes[0]
    b = mg_inputs.uniform_rhs(n, 0)
    ba = m.to_active(b)
    od = dict(nu1=1, nu2=1, omega=0.74)
    xsO, hO = _oracle_history(Oh, ba, od, cycles)
    xsA, hA = _oracle_history(Oalt, ba, od, cycles)
    F = floor_parity(Oh, Oalt, ba, xsO, xsA, hO, hA)
    xd, bd = H.to_device(np.zeros_like(b)), H.to_device(b)
    hG = [H.residual(0, xd, bd, norm=True)] + [H.cycle(xd, bd, Opts(1, 1, "vanka", 0.74)) for _ in range(cycles)]
    hG = np.array(hG)
    dev = np.abs(hG - hO)
    print("rel dev", dev / hO, "rho", hO[1:] / hO[:-1])
    assert np.all(dev <= 1e-10 * hO + F), (dev / hO, F / hO)
    ok = hO[1:] >= 1e3 * F[1:]
    assert np.all(np.abs(hG[1:] / hG[:-1] - hO[1:] / hO[:-1])[ok] <= 1e-3)
    e_go = C.block_rel_err(m, H.to_host(xd), m.from_active(xsO[-1]))
    e_oo = C.block_rel_err(m, m.from_active(xsA[-1]), m.from_active(xsO[-1]))
    for k in e_go:
        assert e_go[k] <= 1e-9 + 4 * e_oo[k], (e_go, e_oo)


@pytest.mark.parametrize("n,levels,pname,het,nu", [(64, 5, "unit", 3, 1), (96, 4, "stiff", 7, 2), (112, 5, "mixed", 5, 1),
                                                   (36, 3, "unit", 3, 1), (576, 7, "unit", 3, 1)])
def test_het_warp_sweep_bitwise(n, levels, pname, het, nu):
    """The warp-marching heterogeneous-K Vanka sweep (vanka_hwarp_kernel: K^{-1} rows in a TMA ring,
    residuals and patch corrections moved by shuffles, boundary-vertex patches from vanka_bnd_kernel)
    gives bitwise the iterates and norms of the 2-D tile kernel vanka_het_kernel (same arithmetic, same
    summation order, reading A20) on every level -- ragged strips and
    segments, zero-initial-guess levels; the 576^2 case runs the production dispatch (warp sweep on the
    576 level with the S~^{-1} prefetch, 2-D tiles below) against the 2-D tiles everywhere."""
    _torch()
    from paper_2107_04060_b200 import Opts
    b = mg_inputs.uniform_rhs(n, 11)
    out = []
    for warp in ("1", "0"):
        knob = ("256" if n >= 512 else "1") if warp == "1" else "0"
        H = C.gpu_hierarchy(n, levels, pname, het, env={"MG_HET_WARP_N": knob})
        xd, bd = H.to_device(np.zeros_like(b)), H.to_device(b)
        hist = [H.cycle(xd, bd, Opts(nu, nu, "vanka", 0.74)) for _ in range(3)]
        out.append((H.to_host(xd), hist))
        H.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]

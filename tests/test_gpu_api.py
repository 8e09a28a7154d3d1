"""The public entry points around the cycle (include/mg.h): host-buffer solve, asynchronous cycle
with the fused input norm, cycle tracing, argument checks.  Each is checked against the plain
device path it wraps (bitwise where the arithmetic is the same) or against the definition of what
it reports; the numerics of the path itself are test_gpu_parity.py's."""
import numpy as np
import pytest

import mg_inputs
from tests import _cases as C

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.parametrize("n,levels,pname,relax", [(32, 4, "cfg5", "vanka"), (64, 5, "unit", "bsr")])
def test_solve_host_equals_device_solve(n, levels, pname, relax):
    """mg_solve_host (pinned host x, b in; x, history out) runs the same cycles as mg_solve on
    device buffers: identical histories and iterates."""
    torch = _torch()
    from paper_2107_04060_b200 import Opts
    o = Opts(1, 1, "vanka", 0.72) if relax == "vanka" else Opts(1, 1, "bsr", 0.75, 1.0, 3)
    b = mg_inputs.uniform_rhs(n, 21)
    H = C.gpu_hierarchy(n, levels, pname)
    xd, bd = H.to_device(np.zeros_like(b)), H.to_device(b)
    rc_d, hist_d = H.solve(xd, bd, o, rtol=1e-6, max_cycles=12)
    torch.cuda.synchronize()
    x_dev = H.to_host(xd)
    xh = np.zeros_like(b)
    rc_h, hist_h = H.solve_host(xh, np.ascontiguousarray(b), o, rtol=1e-6, max_cycles=12)
    assert rc_h == rc_d
    assert np.array_equal(hist_h, hist_d)
    assert np.array_equal(xh[mg_inputs.active_mask(n)], x_dev[mg_inputs.active_mask(n)])
    H.close()


def test_cycle_async_norm_and_iterate():
    """mg_cycle_async with norm2_out: the fused norm is ||b - A x_in||^2 of the INPUT iterate (one
    rounding-scale of mg_residual's), and the iterate equals mg_cycle's bitwise."""
    torch = _torch()
    from paper_2107_04060_b200 import Opts
    n, levels = 64, 5
    o = Opts(1, 1, "vanka", 0.72)
    b = mg_inputs.uniform_rhs(n, 22)
    x0 = mg_inputs.uniform_vector(n, 23)
    H = C.gpu_hierarchy(n, levels, "mixed")
    bd = H.to_device(b)
    xa, xb = H.to_device(x0), H.to_device(x0)
    r0 = H.residual(0, xa, bd, norm=True)
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    H.cycle_async(xa, bd, o, norm2_out=out)
    H.cycle(xb, bd, o)
    torch.cuda.synchronize()
    assert abs(float(out.sqrt().item()) - r0) <= 1e-12 * r0
    assert torch.equal(xa, xb)
    H.close()


def test_cycle_tracing():
    """mg_set_timing / mg_timing / mg_timing_levels: five positive phase times whose sum is the
    traced cycle, a per-level split that adds up to the same cycle, and a kernel count."""
    torch = _torch()
    from paper_2107_04060_b200 import Opts
    n, levels = 128, 6
    b = mg_inputs.uniform_rhs(n, 24)
    H = C.gpu_hierarchy(n, levels, "cfg5")
    xd, bd = H.to_device(np.zeros_like(b)), H.to_device(b)
    H.set_timing(True)
    H.cycle(xd, bd, Opts(1, 1, "vanka", 0.7))
    torch.cuda.synchronize()
    ph = H.timing()
    lv = H.timing_levels()
    H.set_timing(False)
    assert len(ph) == 5 and all(v >= 0.0 for v in ph) and ph[0] > 0.0 and ph[4] > 0.0
    assert len(lv["pre"]) == levels - 1 and len(lv["post"]) == levels - 1
    tot_levels = sum(lv["pre"]) + sum(lv["restrict"]) + lv["coarse"] + sum(lv["prolong"]) + sum(lv["post"])
    assert abs(tot_levels - sum(ph)) <= 0.05 * sum(ph) + 0.05
    assert H.cycle_kernels() > 0
    H.close()


def test_fgmres_argument_checks():
    """mg_fgmres rejects restart lengths outside [1, 31] with MG_EINVAL (no launch)."""
    _torch()
    from paper_2107_04060_b200 import Opts
    from paper_2107_04060_b200.mg import MGError
    n, levels = 16, 3
    b = mg_inputs.uniform_rhs(n, 25)
    H = C.gpu_hierarchy(n, levels, "unit")
    xd, bd = H.to_device(np.zeros_like(b)), H.to_device(b)
    for restart in (0, 32):
        with pytest.raises(MGError):
            H.fgmres(xd, bd, Opts(1, 1, "vanka", 0.74), rtol=1e-8, max_iters=10, restart=restart)
    H.close()


@pytest.mark.parametrize("nu1,nu2,relax", [(1, 0, "vanka"), (2, 1, "vanka"), (1, 2, "bsr"), (0, 1, "vanka")])
def test_odd_sweep_solve_returns_recorded_iterate(nu1, nu2, relax):
    """mg_solve with an odd number of level-0 sweeps (the cycle ends with a copy back into x): the
    returned x is the iterate whose residual is the last history entry, not one smoothing step
    past it (the copy honours the stop flag).  ||b - A x_returned|| = hist[-1] to one
    rounding of the residual norm, and a second solve on the same context still computes (the
    stop flag was cleared)."""
    torch = _torch()
    from paper_2107_04060_b200 import Opts
    n, levels = 64, 5
    o = Opts(nu1, nu2, "vanka", 0.72) if relax == "vanka" else Opts(nu1, nu2, "bsr", 0.75, 1.0, 3)
    b = mg_inputs.uniform_rhs(n, 26)
    H = C.gpu_hierarchy(n, levels, "cfg5")
    xd, bd = H.to_device(np.zeros_like(b)), H.to_device(b)
    for rtol, cap in ((1e-3, 60), (1e-30, 5)):     # converged stop, then the max_cycles stop
        xd.zero_()
        rc, hist = H.solve(xd, bd, o, rtol=rtol, max_cycles=cap)
        torch.cuda.synchronize()
        r = H.residual(0, xd, bd, norm=True)
        assert abs(r - hist[-1]) <= 1e-12 * hist[-1], (nu1, nu2, r, hist[-1], rc)
    # max_cycles = 0: x is left untouched
    x0 = mg_inputs.uniform_vector(n, 27)
    xd = H.to_device(x0)
    rc, hist = H.solve(xd, bd, o, rtol=1e-8, max_cycles=0)
    torch.cuda.synchronize()
    assert len(hist) == 1 and torch.equal(xd, H.to_device(x0))
    H.close()


def test_binding_rejects_bad_vectors():
    """The binding refuses tensors the C call would read out of bounds (wrong element count,
    non-contiguous views) and the library refuses misaligned pointers (MG_EINVAL, no launch)."""
    torch = _torch()
    from paper_2107_04060_b200.mg import MGError
    import ctypes
    n, levels = 16, 3
    H = C.gpu_hierarchy(n, levels, "unit")
    good = H.zeros()
    with pytest.raises(MGError):
        H.residual(0, good[:, :, : n + 1], good, norm=True)            # strided view
    with pytest.raises(MGError):
        H.residual(0, good.reshape(-1)[:-32], good, norm=True)         # too short
    raw = torch.zeros(good.numel() + 1, dtype=torch.float64, device="cuda")
    rc = H.lib.mg_residual(H.ctx, 0, ctypes.c_void_p(raw.data_ptr() + 8), ctypes.c_void_p(good.data_ptr()),
                           None, None, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == -1                                                      # 8-byte aligned only
    with pytest.raises(MGError):
        H.solve_host(np.zeros((10, n + 1, n)), np.zeros((10, n + 1, n + 1)), None)
    H.close()

"""GPU parity: every C-ABI operation of libmg.so against the CPU oracle on the same seeded inputs.

Tolerances:
* residual: componentwise |r_G - r_O| <= 32 u (|b| + |A||x|), u = 2^-53 (rounding of one residual
  evaluation in two summation orders);
* one relaxation sweep / transfer / coarse solve: the result is a linear map of rounded inputs;
  compared in the max norm relative to the result, bounds derived from the operator's conditioning
  and stated per case;
* cycles: per-cycle residual norms within 1e-10 relative while the norm is above the rounding floor
  (SURVEY 8c-11), convergence factors within 1e-3.
"""
import numpy as np
import pytest

import mg_inputs
from tests import _cases as C

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _inactive_zero(H, v, level=0):
    """Inactive and padding slots of a device vector are exactly 0."""
    nl = H.level_n(level)
    a = v.cpu().numpy()
    mask = np.zeros(a.shape, dtype=bool)
    mask[:, :, : nl + 1] = mg_inputs.active_mask(nl)
    assert np.all(a[~mask] == 0.0)


@pytest.mark.parametrize("n,pname,het,march", [(4, "unit", None, False), (8, "mixed", None, False),
                                               (16, "stiff", None, False), (40, "cfg5", None, False),
                                               (66, "mixed", None, False), (24, "unit", 3, False),
                                               (34, "mixed", 7, False), (40, "cfg5", None, True),
                                               (66, "mixed", None, True), (130, "stiff", None, True),
                                               (34, "mixed", 7, True), (66, "unit", 3, True)])
def test_residual(n, pname, het, march):
    """r = b - A x and its norm; march=True runs the row-marching residual kernel (production for
    n >= 512; with a K field its K^{-1} rows arrive in a TMA ring) on small grids."""
    torch = _torch()
    H = C.gpu_hierarchy(n, C.small_coarse_levels(n), pname, het, env={"MG_RESID_MARCH_N": "0"} if march else None)
    op = C.operator(n, pname, het)
    m = C.mesh(n)
    x = mg_inputs.uniform_vector(n, 11)
    b = mg_inputs.uniform_rhs(n, 12)
    xd, bd = H.to_device(x), H.to_device(b)
    rd = H.zeros()
    nrm = H.residual(0, xd, bd, rd, norm=True)
    torch.cuda.synchronize()
    rG = m.to_active(H.to_host(rd))
    xa, ba = m.to_active(x), m.to_active(b)
    rO = ba - op.A @ xa
    scale = np.abs(ba) + C.abs_matvec(op, xa)
    err = np.abs(rG - rO)
    assert np.all(err <= 32 * U * scale), (err / scale).max() / U
    assert abs(nrm - np.linalg.norm(rO)) <= 1e-13 * np.linalg.norm(rO) + 32 * U * np.linalg.norm(scale)
    _inactive_zero(H, rd)


@pytest.mark.parametrize("n,pname,omega,march", [(4, "unit", 0.74, False), (8, "mixed", 0.9, False),
                                                 (16, "stiff", 0.7, False), (40, "cfg5", 0.7, False),
                                                 (66, "unit", 0.74, False), (4, "unit", 0.74, True),
                                                 (30, "mixed", 0.9, True), (57 * 2, "stiff", 0.7, True),
                                                 (130, "cfg5", 0.7, True)])
def test_vanka_sweep(n, pname, omega, march):
    """One Vanka sweep; march=True runs the production row-marching TMA kernel on small grids
    (ragged strips: n + 1 not a multiple of the strip width, several row segments)."""
    torch = _torch()
    H = C.gpu_hierarchy(n, C.small_coarse_levels(n), pname, march=march)
    from oracle.relax import Vanka
    op = C.operator(n, pname)
    V = Vanka(op)
    m = C.mesh(n)
    x = mg_inputs.uniform_vector(n, 21)
    b = mg_inputs.uniform_rhs(n, 22)
    xd, bd = H.to_device(x), H.to_device(b)
    H.relax_vanka(0, xd, bd, omega, sweeps=1)
    torch.cuda.synchronize()
    xG = H.to_host(xd)
    xO = m.from_active(V.sweep(m.to_active(x), m.to_active(b), omega))
    err = np.abs(xG - xO).max() / np.abs(xO).max()
    tol = 1e-12 if pname != "stiff" else 1e-9
    assert err <= tol, err
    _inactive_zero(H, xd)


@pytest.mark.parametrize("n,pname", [(8, "unit"), (16, "mixed"), (40, "stiff"), (66, "cfg5")])
def test_restrict_prolong(n, pname):
    torch = _torch()
    from oracle.transfer import Transfer
    H = C.gpu_hierarchy(n, C.small_coarse_levels(n, 2), pname)
    mf, mc = C.mesh(n), C.mesh(n // 2)
    T = Transfer(mf, mc)
    r = mg_inputs.uniform_vector(n, 31)
    e = mg_inputs.uniform_vector(n // 2, 32)
    x = mg_inputs.uniform_vector(n, 33)
    rd, bc = H.to_device(r), H.zeros(1)
    H.restrict(0, rd, bc)
    ed, xd = H.to_device(e, 1), H.to_device(x)
    H.prolong(0, ed, xd)
    torch.cuda.synchronize()
    # componentwise rounding bound of a sparse matvec in two summation orders: 32 u |R| |r|
    absR, absP = abs(T.R), abs(T.P)
    ra, ea = np.abs(mf.to_active(r)), np.abs(mc.to_active(e))
    bO = T.R @ mf.to_active(r)
    bG = mc.to_active(H.to_host(bc, 1))
    assert np.all(np.abs(bG - bO) <= 32 * U * (absR @ ra))
    xO = mf.to_active(x) + T.P @ mc.to_active(e)
    xG = mf.to_active(H.to_host(xd))
    assert np.all(np.abs(xG - xO) <= 32 * U * (np.abs(mf.to_active(x)) + absP @ ea))
    _inactive_zero(H, bc, 1)
    _inactive_zero(H, xd)


@pytest.mark.parametrize("nc,pname,het", [(4, "unit", None), (4, "stiff", None), (8, "mixed", None), (4, "unit", 5)])
def test_coarse_solve(nc, pname, het):
    torch = _torch()
    from oracle.cycle import CoarseSolver
    n = nc * 4
    H = C.gpu_hierarchy(n, 3, pname, het)
    Oh = C.hierarchy(n, 3, pname, "bsr" if het else "vanka", het)
    opc = Oh.ops[-1]
    mc = Oh.meshes[-1]
    b = mg_inputs.uniform_vector(nc, 41)
    bd, xd = H.to_device(b, 2), H.zeros(2)
    H.coarse_solve(bd, xd)
    torch.cuda.synchronize()
    xG = mc.to_active(H.to_host(xd, 2))
    xO = Oh.coarse.solve(mc.to_active(b))
    err = np.abs(xG - xO).max() / np.abs(xO).max()
    assert err <= 1e-11, err
    # and it is a solve: residual at the rounding level of A_c
    res = mc.to_active(b) - opc.A @ xG
    assert np.linalg.norm(res) <= 1e-12 * (np.linalg.norm(mc.to_active(b)) + np.linalg.norm(C.abs_matvec(opc, xG)))


@pytest.mark.parametrize("n,pname,het,nJ,march", [(8, "unit", None, 1, False), (16, "mixed", None, 3, False),
                                                  (40, "unit", None, 3, False), (16, "unit", 3, 3, False),
                                                  (34, "mixed", 9, 2, False), (16, "mixed", None, 3, True),
                                                  (40, "unit", None, 3, True), (16, "unit", 3, 3, True),
                                                  (34, "mixed", 9, 2, True), (58, "stiff", 5, 3, True)])
def test_bsr_sweep(n, pname, het, nJ, march):
    """One BSR sweep vs the oracle; march=True runs the row-marching TMA stages (production path of
    the levels with n >= 512) on small grids, strips and segments included."""
    torch = _torch()
    from oracle.relax import BSR
    H = C.gpu_hierarchy(n, C.small_coarse_levels(n), pname, het, march=march)
    op = C.operator(n, pname, het)
    S = BSR(op)
    m = C.mesh(n)
    x = mg_inputs.uniform_vector(n, 51)
    b = mg_inputs.uniform_rhs(n, 52)
    xd, bd = H.to_device(x), H.to_device(b)
    om, omJ = 0.7, 0.9
    H.relax_bsr(0, xd, bd, om, omJ, nJ, sweeps=1)
    torch.cuda.synchronize()
    xG = H.to_host(xd)
    xO = m.from_active(S.sweep(m.to_active(x), m.to_active(b), om, omJ, nJ))
    err = np.abs(xG - xO).max() / np.abs(xO).max()
    assert err <= 1e-11, err
    _inactive_zero(H, xd)


def _oracle_history(Oh, b, opts, cycles):
    N = Oh.ops[0].A.shape[0]
    x = np.zeros(N)
    hist = [Oh.residual_norm(x, b)]
    xs = [x]
    for _ in range(cycles):
        x = Oh.cycle(x, b, opts)
        hist.append(Oh.residual_norm(x, b))
        xs.append(x)
    return xs, np.array(hist)


def floor_parity(Oh, Oalt, b, xs_O, xs_alt, hO, hAlt):
    """Per-cycle rounding floor F_k = max(8 u || |b| + |A||x_k| ||, 4 |h_k - h'_k|) where h' is the
    oracle run with every summation order reversed (reading A22)."""
    op = Oh.ops[0]
    F = np.array([max(8 * U * np.linalg.norm(np.abs(b) + C.abs_matvec(op, x)), 4 * abs(h - ha))
                  for x, h, ha in zip(xs_O, hO, hAlt)])
    return F


@pytest.mark.parametrize("n,levels,pname,relax,het,cycles,march", [
    (16, 3, "unit", "vanka", None, 10, False),      # BASELINE config 1
    (64, 5, "cfg5", "vanka", None, 6, True),        # config 5 regime, marching kernels on every level
    (64, 5, "unit", "bsr", None, 4, True),          # marching restriction under BSR
    (32, 4, "stiff", "vanka", None, 8, False),      # config 3 regime
    (32, 4, "cfg5", "vanka", None, 8, False),       # config 5 regime
    (32, 4, "unit", "bsr", None, 8, False),         # config 2 (BSR) regime
    (32, 4, "unit", "bsr", 3, 6, False),            # config 4 regime (heterogeneous K)
    (32, 4, "unit", "bsr", 3, 4, True),             # config 4 regime, marching restriction (K field)
    (48, 3, "mixed", "vanka", None, 5, True),       # n not a power of two (coarsest 12), marching kernels
    (48, 3, "mixed", "bsr", 7, 4, True),            # the same with BSR and a K field
])
def test_cycle_history(n, levels, pname, relax, het, cycles, march):
    torch = _torch()
    from paper_2107_04060_b200 import Opts
    from oracle.cycle import Hierarchy as OH
    H = C.gpu_hierarchy(n, levels, pname, het, march=march)
    Oh = C.hierarchy(n, levels, pname, relax, het)
    lam, mu, K, tau, alpha, invM = C.PARAMS[pname]
    kinv = None if het is None else 1.0 / mg_inputs.lognormal_K(n, het)
    Oalt = OH(n, levels, lam, mu, tau, alpha, invM, 1.0, K=K, Kinv_field=kinv, relax=relax, alt_order=True)
    m = Oh.meshes[0]
    b = mg_inputs.uniform_rhs(n, 0)
    ba = m.to_active(b)
    if relax == "vanka":
        od = dict(nu1=1, nu2=1, omega=0.72)
        go = Opts(1, 1, "vanka", 0.72)
    else:
        od = dict(nu1=1, nu2=1, omega=0.5 if het else 0.75, omega_J=0.7 if het else 1.0, jacobi_sweeps=3)
        go = Opts(1, 1, "bsr", od["omega"], od["omega_J"], 3)
    xsO, hO = _oracle_history(Oh, ba, od, cycles)
    xsA, hA = _oracle_history(Oalt, ba, od, cycles)
    F = floor_parity(Oh, Oalt, ba, xsO, xsA, hO, hA)
    xd, bd = H.to_device(np.zeros_like(b)), H.to_device(b)
    hG = [H.residual(0, xd, bd, norm=True)]
    for _ in range(cycles):
        hG.append(H.cycle(xd, bd, go))
    hG = np.array(hG)
    dev = np.abs(hG - hO)
    print("rel dev", dev / hO, "floor/h", F / hO, "oracle spread/h", np.abs(hA - hO) / hO)
    assert np.all(dev <= 1e-10 * hO + F), (dev / hO, F / hO)
    # final iterate per block, floor = 4x the oracle self-spread
    xG = H.to_host(xd)
    e_go = C.block_rel_err(m, xG, m.from_active(xsO[-1]))
    e_oo = C.block_rel_err(m, m.from_active(xsA[-1]), m.from_active(xsO[-1]))
    for k in e_go:
        assert e_go[k] <= 1e-9 + 4 * e_oo[k], (e_go, e_oo)
    rG, rO = hG[1:] / hG[:-1], hO[1:] / hO[:-1]
    ok = hO[1:] >= 1e3 * F[1:]
    assert np.all(np.abs(rG - rO)[ok] <= 1e-3)


@pytest.mark.parametrize("n,levels,pname,nu2", [(64, 5, "cfg5", 1), (32, 4, "mixed", 2), (64, 4, "stiff", 1)])
def test_fused_prolong_bitwise(n, levels, pname, nu2):
    """The prolongation fused into the first post-sweep of the marching kernel
    gives bitwise the iterates of prolong_kernel followed by the sweep (same arithmetic, same
    order), over several cycles and with a second, unfused post-sweep (nu2 = 2)."""
    torch = _torch()
    from paper_2107_04060_b200 import Opts
    b = mg_inputs.uniform_rhs(n, 3)
    out = []
    for fuse in ("1", "0"):
        H = C.gpu_hierarchy(n, levels, pname, march=True, env={"MG_FUSE_PROLONG": fuse})
        xd, bd = H.to_device(np.zeros_like(b)), H.to_device(b)
        hist = [H.cycle(xd, bd, Opts(1, nu2, "vanka", 0.7)) for _ in range(3)]
        out.append((H.to_host(xd), hist))
        H.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]


@pytest.mark.parametrize("n,levels,pname,nu2", [(64, 5, "cfg5", 1), (48, 3, "mixed", 2), (128, 6, "stiff", 1),
                                                (32, 4, "cfg5", 2)])
def test_warp_sweep_bitwise(n, levels, pname, nu2):
    """The warp-marching Vanka sweep (vanka_warp_kernel: one warp per 30-column strip, residuals and
    patch corrections moved between lanes by shuffles) gives bitwise the iterates and fused norms
    of the CTA row-marching sweep on every level (same arithmetic, same summation order; PAPER.md:
    575-588), for the zero-initial-guess pre-sweeps, the level-0 sweep with its fused norm, the first
    post-sweep with the prolongation fused in, ragged strips (49 columns = 30 +
    19) and ragged row segments."""
    torch = _torch()
    from paper_2107_04060_b200 import Opts
    b = mg_inputs.uniform_rhs(n, 5)
    out = []
    # (warp kernel on every level, prolongation fused into the first post-sweep); the last is the
    # reference: CTA marching kernels with a separate prolong_kernel
    for warp, fuse in (("1", "1"), ("1", "0"), ("0", "1"), ("0", "0")):
        H = C.gpu_hierarchy(n, levels, pname, march=True, env={"MG_WARP_MIN_N": warp, "MG_FUSE_PROLONG": fuse})
        xd, bd = H.to_device(np.zeros_like(b)), H.to_device(b)
        hist = [H.cycle(xd, bd, Opts(1, nu2, "vanka", 0.7)) for _ in range(3)]
        out.append((H.to_host(xd), hist))
        H.close()
    for k in range(3):
        assert np.array_equal(out[k][0], out[3][0]), k
        assert out[k][1] == out[3][1], k


@pytest.mark.parametrize("n,levels,pname,het,nJ", [(64, 5, "unit", 3, 3), (48, 3, "mixed", None, 1),
                                                    (96, 4, "stiff", 7, 2), (64, 5, "cfg5", None, 3)])
def test_warp_bsr_bitwise(n, levels, pname, het, nJ):
    """The warp-marching BSR stage B (bsr_b_warp_kernel: y_u and the displacement-patch corrections
    moved by shuffles, dp and K^{-1} in TMA rings) gives bitwise the iterates and norms of the CTA
    marching stage (same arithmetic, same order), with and without a K field,
    zero-initial-guess levels, ragged strips and segments."""
    torch = _torch()
    from paper_2107_04060_b200 import Opts
    b = mg_inputs.uniform_rhs(n, 8)
    out = []
    for warp in ("1", "0"):
        H = C.gpu_hierarchy(n, levels, pname, het, march=True, env={"MG_WARP_MIN_N": warp, "MG_WARP_BSR": warp})
        xd, bd = H.to_device(np.zeros_like(b)), H.to_device(b)
        hist = [H.cycle(xd, bd, Opts(1, 1, "bsr", 0.7, 0.9, nJ)) for _ in range(3)]
        out.append((H.to_host(xd), hist))
        H.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]


@pytest.mark.parametrize("n,levels,pname,het,nJ", [(64, 5, "unit", 3, 3), (48, 3, "mixed", None, 1),
                                                    (96, 4, "stiff", 7, 2), (64, 5, "cfg5", None, 4),
                                                    (48, 3, "unit", 5, 5)])
def test_bsr_rvec_bitwise(n, levels, pname, het, nJ):
    """Marching BSR with stage B reading the residual planes stage A stored (bsr_b_march_kernel<.., 2>,
    MG_BSR_RVEC=1, the default) gives bitwise the iterates and norms of the path that evaluates
    r = b - A x in both stages (one residual per relaxation), with and without a
    K field, on zero-initial-guess levels, ragged strips and segments; likewise two Jacobi sweeps on S
    in one launch against two launches."""
    torch = _torch()
    from paper_2107_04060_b200 import Opts
    b = mg_inputs.uniform_rhs(n, 8)
    out = []
    # default (residual vector + paired Jacobi sweeps, bsr_jacobi2_t_kernel) against the plain path
    for rvec in ("1", "0"):
        H = C.gpu_hierarchy(n, levels, pname, het, march=True, env={"MG_BSR_RVEC": rvec, "MG_JACOBI_PAIR": rvec})
        xd, bd = H.to_device(np.zeros_like(b)), H.to_device(b)
        hist = [H.cycle(xd, bd, Opts(2, 1, "bsr", 0.7, 0.9, nJ)) for _ in range(3)]
        x1 = H.to_host(xd)
        H.relax_bsr(0, xd, bd, 0.7, 0.9, nJ, sweeps=3)
        out.append((x1, hist, H.to_host(xd)))
        H.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]
    assert np.array_equal(out[0][2], out[1][2])


@pytest.mark.parametrize("n,levels,pname,het,nJ", [(64, 5, "unit", 3, 3), (48, 3, "mixed", None, 4),
                                                    (256, 7, "unit", None, 3), (160, 5, "stiff", 7, 5),
                                                    (576, 7, "unit", 3, 3)])
def test_bsr_jacobi_fused_b_bitwise(n, levels, pname, het, nJ):
    """The 2-D tile stage B with the last two table Jacobi sweeps run inside it (MG_JACOBI_FUSE_B=1, the
    default on the levels below the marching threshold) gives bitwise the iterates and
    norms of separate Jacobi launches followed by the plain stage B: small 8 x 4 and 32 x 8 tiles, with and
    without a K field, n_J = 3, 4, 5."""
    torch = _torch()
    from paper_2107_04060_b200 import Opts
    b = mg_inputs.uniform_rhs(n, 9)
    out = []
    for fuse in ("1", "0"):
        # the 576^2 case: production dispatch (marching stages with the residual vector on the 576 level)
        H = C.gpu_hierarchy(n, levels, pname, het, env={"MG_JACOBI_FUSE_B": fuse, "MG_JACOBI_PAIR": fuse,
                                                        "MG_BSR_RVEC": fuse})
        xd, bd = H.to_device(np.zeros_like(b)), H.to_device(b)
        hist = [H.cycle(xd, bd, Opts(2, 1, "bsr", 0.7, 0.9, nJ)) for _ in range(3)]
        out.append((H.to_host(xd), hist))
        H.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]


@pytest.mark.parametrize("n,levels,pname,nu", [(64, 5, "cfg5", 1), (48, 3, "mixed", 2), (128, 6, "stiff", 1)])
def test_small_tile_sweep_bitwise(n, levels, pname, nu):
    """The small-tile sweep with all of its global reads in the first round trip (vanka_small_kernel:
    b and owner x in registers, the boundary classes' inverses staged in shared memory) gives bitwise
    vanka_kernel's iterates and norms on the levels with n <= 128 (same arithmetic, same order)."""
    torch = _torch()
    from paper_2107_04060_b200 import Opts
    b = mg_inputs.uniform_rhs(n, 6)
    out = []
    # 2: four threads per position (vanka_small4_kernel), 1: vanka_small_kernel, 0: vanka_kernel + prolong_kernel
    for diet in ("2", "1", "0"):
        H = C.gpu_hierarchy(n, levels, pname, env={"MG_SMALL_DIET": diet})
        xd, bd = H.to_device(np.zeros_like(b)), H.to_device(b)
        hist = [H.cycle(xd, bd, Opts(nu, nu, "vanka", 0.7)) for _ in range(3)]
        out.append((H.to_host(xd), hist))
        H.close()
    for k in range(2):
        assert np.array_equal(out[k][0], out[2][0]), k
        assert out[k][1] == out[2][1], k


@pytest.mark.parametrize("n,levels,pname,nu", [(64, 5, "cfg5", 1), (32, 4, "mixed", 2), (128, 6, "stiff", 1)])
def test_bottom_kernel_bitwise(n, levels, pname, nu):
    """The grid-wide bottom of the V-cycle (levels with n <= 128 and the coarsest solve in one
    cooperative kernel) reproduces bitwise the per-level kernel sequence it replaces (same tile
    functions, same order), over several cycles and for V(2,2)."""
    torch = _torch()
    from paper_2107_04060_b200 import Opts
    b = mg_inputs.uniform_rhs(n, 4)
    out = []
    for bottom in ("128", "0"):   # MG_BOTTOM_N=128 switches the (off by default) bottom kernel on
        H = C.gpu_hierarchy(n, levels, pname, env={"MG_BOTTOM_N": bottom})
        xd, bd = H.to_device(np.zeros_like(b)), H.to_device(b)
        hist = [H.cycle(xd, bd, Opts(nu, nu, "vanka", 0.7)) for _ in range(3)]
        out.append((H.to_host(xd), hist))
        H.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]


def test_solve_matches_cycles():
    """mg_solve (device-side stop flag, fused norms) reproduces the cycle-by-cycle history and stops at rtol."""
    torch = _torch()
    from paper_2107_04060_b200 import Opts
    n, levels = 16, 3
    H = C.gpu_hierarchy(n, levels, "unit")
    Oh = C.hierarchy(n, levels, "unit", "vanka")
    m = Oh.meshes[0]
    b = mg_inputs.uniform_rhs(n, 0)
    od = dict(nu1=1, nu2=1, omega=0.74)
    _, hO = _oracle_history(Oh, m.to_active(b), od, 40)
    xd, bd = H.to_device(np.zeros_like(b)), H.to_device(b)
    rc, hist = H.solve(xd, bd, Opts(1, 1, "vanka", 0.74), rtol=1e-8, max_cycles=40)
    k = len(hist) - 1
    assert rc == 0
    assert hist[-1] <= 1e-8 * hist[0] and hist[-2] > 1e-8 * hist[0]
    floor = 64 * U * np.linalg.norm(m.to_active(b))
    assert np.all(np.abs(hist - hO[: k + 1]) <= 1e-10 * hO[: k + 1] + floor)
    # not converged within 3 cycles -> MG_NOTCONV with 4 history entries
    xd.zero_()
    rc, hist = H.solve(xd, bd, Opts(1, 1, "vanka", 0.74), rtol=1e-14, max_cycles=3)
    assert rc == 1 and len(hist) == 4
    assert np.all(np.abs(hist - hO[:4]) <= 1e-10 * hO[:4])


@pytest.mark.parametrize("n,levels,pname,relax,march", [(16, 3, "unit", "vanka", False),
                                                       (32, 4, "cfg5", "vanka", False),
                                                       (32, 4, "unit", "bsr", False),
                                                       (32, 4, "cfg5", "vanka", True)])
def test_fgmres_history(n, levels, pname, relax, march):
    """FGMRES + one V-cycle per iteration: the GPU history equals the oracle's
    (oracle: modified Gram-Schmidt; GPU: classical Gram-Schmidt twice) to 1e-9 relative while
    above 1e3 x the rounding floor, and the final iterates agree."""
    torch = _torch()
    from paper_2107_04060_b200 import Opts
    from oracle.krylov import fgmres_mg
    # march: every kernel in its production (row-marching) variant, the residual / apply included
    H = C.gpu_hierarchy(n, levels, pname, march=march, env={"MG_RESID_MARCH_N": "0"} if march else None)
    Oh = C.hierarchy(n, levels, pname, relax)
    m = Oh.meshes[0]
    b = mg_inputs.uniform_rhs(n, 3)
    ba = m.to_active(b)
    if relax == "vanka":
        od, go = dict(nu1=1, nu2=1, omega=0.72), Opts(1, 1, "vanka", 0.72)
    else:
        od, go = dict(nu1=1, nu2=1, omega=0.75, omega_J=1.0, jacobi_sweeps=3), Opts(1, 1, "bsr", 0.75, 1.0, 3)
    from oracle.cycle import Hierarchy as OH
    lam, mu, K, tau, alpha, invM = C.PARAMS[pname]
    Oalt = OH(n, levels, lam, mu, tau, alpha, invM, 1.0, K=K, relax=relax, alt_order=True)
    xO, hO = fgmres_mg(Oh, ba, od, rtol=1e-9, max_iters=40, restart=30)
    xA, hA = fgmres_mg(Oalt, ba, od, rtol=1e-9, max_iters=40, restart=30)
    xd, bd = H.to_device(np.zeros_like(b)), H.to_device(b)
    rc, hG = H.fgmres(xd, bd, go, rtol=1e-9, max_iters=40, restart=30)
    k = min(len(hG), len(hO), len(hA))
    # floor: 4 x the spread between two legal summation orders of the oracle; Krylov
    # iterations amplify rounding, so late iterations are compared at that level
    F = 4 * np.abs(hA[:k] - hO[:k]) + 64 * U * np.linalg.norm(ba)
    dev = np.abs(hG[:k] - hO[:k])
    print("fgmres its GPU/oracle/alt", len(hG) - 1, len(hO) - 1, len(hA) - 1,
          "max rel dev", (dev / hO[:k]).max(), "max rel spread", (np.abs(hA[:k] - hO[:k]) / hO[:k]).max())
    assert abs(len(hG) - len(hO)) <= 1
    assert np.all(dev <= 1e-9 * hO[:k] + F)
    errs = C.block_rel_err(m, H.to_host(xd), m.from_active(xO))
    e_oo = C.block_rel_err(m, m.from_active(xA), m.from_active(xO))
    for key in errs:
        assert errs[key] <= 1e-7 + 4 * e_oo[key], (errs, e_oo)

"""Backward-Euler time stepping on the GPU: mg_step_rhs /
mg_time_step against the oracle's time stepper (oracle/timestep.py) on the same loads.

* mg_step_rhs: the history term -(1/M) M_p p^{m-1} + alpha B_u u^{m-1} is a short sum per triangle;
  componentwise within 16 u of its rounding scale.
* mg_time_step: the paper's smooth-problem solver setting (FGMRES to 1e-10,
  additive Vanka; V(2,2) with tab:vanka22's omega, reading A25; E = 3e4, M = 1e6, alpha = mu_f = 1)
  on the manufactured solution of reading A28 at h = tau = 1/32, four steps: per step the GPU takes
  the oracle's FGMRES iteration count (+-1: the 1e-10 threshold is crossed at rounding level) and
  the iterates agree per block within 1e-8 + 4x the oracle's own summation-order spread.
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


@pytest.mark.parametrize("n,pname", [(8, "mixed"), (40, "cfg5"), (130, "unit")])
def test_step_rhs(n, pname):
    torch = _torch()
    from oracle import timestep as T
    H = C.gpu_hierarchy(n, C.small_coarse_levels(n), pname)
    op = C.operator(n, pname)
    m = C.mesh(n)
    x = mg_inputs.uniform_vector(n, 71)
    b = mg_inputs.uniform_rhs(n, 72)
    xd, bd, od = H.to_device(x), H.to_device(b), H.zeros()
    H.step_rhs(xd, bd, od)
    torch.cuda.synchronize()
    got = m.to_active(H.to_host(od))
    xa = m.to_active(x)
    want = m.to_active(b) + T.history_rhs(op, xa)
    scale = np.abs(m.to_active(b)).copy()
    scale[op.ip] += op.inv_M * (abs(op.Mp) @ np.abs(xa[op.ip])) + op.alpha * (abs(op.Bu) @ np.abs(xa[op.iu]))
    assert np.all(np.abs(got - want) <= 16 * U * scale)


@pytest.mark.parametrize("nu", [0.4, 0.499])
def test_time_steps_match_oracle(nu):
    torch = _torch()
    from paper_2107_04060_b200 import Hierarchy, Opts
    from oracle import timestep as T
    from oracle.cycle import Hierarchy as OH, lame
    from oracle.krylov import fgmres
    n, levels, steps, k = 32, 4, 4, 1.0
    tau = 1.0 / n
    mu, lam = lame(3e4, nu)
    omega = 0.80 if nu == 0.4 else 0.72
    od = dict(nu1=2, nu2=2, omega=omega)
    runs = []
    for alt in (False, True):
        Oh = OH(n, levels, lam, mu, tau, 1.0, 1e-6, 1.0, K=k, relax="vanka", alt_order=alt)
        A = lambda v, Oh=Oh: Oh.ops[0].A @ v                           # noqa: E731
        M = lambda v, Oh=Oh: Oh.cycle(np.zeros_like(v), v, od)          # noqa: E731
        its = []

        def solve(b, xp, A=A, M=M, its=its):
            x, h = fgmres(A, b, xp, M, rtol=1e-10, max_iters=100, restart=30)
            its.append(len(h) - 1)
            return x
        xs = T.run(Oh.ops[0], k, steps, solve=solve)
        runs.append((Oh, xs, its))
    (Oh, xsO, itsO), (_, xsA, _) = runs
    m = Oh.meshes[0]
    H = Hierarchy(n, levels, lam, mu, K=k, tau=tau, alpha=1.0, inv_M=1e-6, mu_f=1.0)
    xd = H.to_device(m.from_active(xsO[0]))
    itsG = []
    for step in range(1, steps + 1):
        bl = H.to_device(m.from_active(T.load(Oh.ops[0], step * tau, k)))
        rc, hist = H.time_step(xd, bl, Opts(2, 2, "vanka", omega), rtol=1e-10, max_iters=100, restart=30)
        assert rc == 0
        itsG.append(len(hist) - 1)
    torch.cuda.synchronize()
    print("iterations per step GPU / oracle", itsG, itsO)
    assert all(abs(a - b) <= 1 for a, b in zip(itsG, itsO))
    e_go = C.block_rel_err(m, H.to_host(xd), m.from_active(xsO[-1]))
    e_oo = C.block_rel_err(m, m.from_active(xsA[-1]), m.from_active(xsO[-1]))
    for key in e_go:
        assert e_go[key] <= 1e-8 + 4 * e_oo[key], (e_go, e_oo)
    # and it is the discretisation's solution: O(h + tau) error level of the manufactured solution
    eu, ep = T.errors(Oh.ops[0], m.to_active(H.to_host(xd)), steps * tau)
    eu0, ep0 = T.errors(Oh.ops[0], xsO[-1], steps * tau)
    assert abs(eu - eu0) <= 1e-6 * eu0 and abs(ep - ep0) <= 1e-6 * ep0

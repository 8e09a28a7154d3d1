"""Oracle pins: FGMRES preconditioned by one V-cycle (tab:mgtime PAPER.md:1090-1108)."""
import numpy as np
import pytest

from oracle.krylov import fgmres, fgmres_mg
from oracle.cycle import Hierarchy, lame
from oracle.manufactured import rhs
from tests._golden import load


def _system(n=30, seed=0):
    rng = np.random.default_rng(seed)
    Q = rng.standard_normal((n, n))
    A = Q + Q.T + np.diag(np.linspace(-3, 5, n))      # symmetric indefinite, like A^RQ
    b = rng.standard_normal(n)
    return A, b


def test_exact_preconditioner_one_iteration():
    A, b = _system()
    Ainv = np.linalg.inv(A)
    x, h = fgmres(lambda v: A @ v, b, np.zeros_like(b), lambda v: Ainv @ v, rtol=1e-12, max_iters=10)
    assert len(h) == 2 and h[-1] <= 1e-12 * h[0]
    assert np.linalg.norm(A @ x - b) <= 1e-12 * np.linalg.norm(b)


def test_identity_preconditioner_is_minimal_residual():
    """With M = I, FGMRES is GMRES: history[i] = min over the Krylov space K_i(A, b) of ||b - A x||
    (brute force least squares on an explicit, orthonormalised Krylov basis)."""
    A, b = _system(24, 1)
    x, h = fgmres(lambda v: A @ v, b, np.zeros_like(b), lambda v: v, rtol=1e-14, max_iters=12, restart=12)
    Kb = [b]
    for i in range(1, 12):
        Kb.append(A @ Kb[-1])
    for i in range(1, 12):
        Qb, _ = np.linalg.qr(np.stack(Kb[:i], axis=1))
        y, *_ = np.linalg.lstsq(A @ Qb, b, rcond=None)
        best = np.linalg.norm(b - A @ Qb @ y)
        assert abs(h[i] - best) <= 1e-9 * np.linalg.norm(b), (i, h[i], best)


def test_restart_and_true_residual():
    rng = np.random.default_rng(2)
    A = np.diag(np.linspace(1.0, 10.0, 40)) + 0.1 * rng.standard_normal((40, 40))   # positive real part:
    b = rng.standard_normal(40)                                                     # GMRES(7) converges
    x, h = fgmres(lambda v: A @ v, b, np.zeros_like(b), lambda v: v, rtol=1e-10, max_iters=400, restart=7)
    assert np.linalg.norm(b - A @ x) <= 1.01e-10 * np.linalg.norm(b) or h[-1] <= 1e-10 * h[0]
    assert np.all(np.diff(h[:8]) <= 1e-12 * h[0])            # non-increasing inside a restart cycle


@pytest.mark.slow
def test_tab_mgtime_vanka_iterations():
    """FGMRES + one V-cycle with additive Vanka on the steady manufactured problem,
    nu = 0.4, E = 3e4, M = 1e6, k = 1e-6, coarsest h = 1/8, rtol 1e-6: tab:mgtime prints 8 (N = 17)
    and 9 (N = 33).  Reading A25: V(2,2), omega = 0.8 (tab:vanka22, nu = 0.4) -- the oracle takes
    10 and 11; the band [paper, paper + 3] fails for a broken cycle (V(1,1) needs 17 / 26)."""
    g = load("paper_tables.json")["tab_mgtime_iters"]
    mu, lam = lame(3e4, 0.4)
    for (n, L, paper) in ((16, 2, g["vanka_nu0.4"][0]), (32, 3, g["vanka_nu0.4"][1])):
        H = Hierarchy(n, L, lam, mu, 1.0, 1.0, 1e-6, 1.0, K=1e-6, relax="vanka")
        b = rhs(H.ops[0], mu, 1e-6)
        x, h = fgmres_mg(H, b, dict(nu1=2, nu2=2, omega=0.8), rtol=1e-6, max_iters=60)
        its = len(h) - 1
        assert paper <= its <= paper + 3, (n, its, paper)
        assert np.linalg.norm(b - H.ops[0].A @ x) <= 1.05e-6 * np.linalg.norm(b)

"""Oracle pins for the exact-integration operator and exact BSR:
Operator(quadrature="exact") -- lambda (div u, div v) integrated exactly (eq. block_form,
PAPER.md:143-167) -- and BSR(exact=True) -- S dp = g solved exactly.

* the lambda term against an independent integration: div u is linear on each triangle, so
  int_T (div u)^2 = |T|/12 (sum_v d_v^2 + (sum_v d_v)^2) from its vertex values d_v, computed here
  from the basis definitions (bubble 4 lambda_a lambda_b n_e, reading A1) with this test's own
  gradients (the oracle integrates with the edge-midpoint rule);
* lambda = 0 and P1-only fields: the two operators coincide (div of P1 is constant per triangle,
  P_Q is then the identity);
* exact BSR equals inexact BSR with enough Jacobi sweeps (their common limit);
* the solver incompatibility of tab:naive: on the exact operator the two-grid
  Vanka factor degrades toward 1 as nu -> 1/2 (printed 0.794 at nu = 0.49 and 0.970 at 0.499),
  while on A^RQ it stays near tab:vanka22's 0.596 at nu = 0.499.
"""
import numpy as np
import pytest

import mg_inputs
from oracle.cycle import Hierarchy, lame
from oracle.fem import Operator
from oracle.mesh import Mesh, NORMALS
from oracle.relax import BSR


def _div_energy_vertex(mesh, u_full):
    """sum_T int_T (div u)^2 by the vertex formula; u_full: full-slot vector."""
    tot = 0.0
    ls = mesh.local_slots()
    for t in range(mesh.ntri):
        P = mesh.tri_coords([t])[0]
        J = np.array([P[1] - P[0], P[2] - P[0]]).T
        Ji = np.linalg.inv(J)
        g = np.array([-(Ji[0] + Ji[1]), Ji[0], Ji[1]])        # grad lambda_v (rows)
        area = 0.5 * abs(np.linalg.det(J))
        d = np.zeros(3)
        for v in range(3):
            dv = sum(u_full[ls[t, 2 * a]] * g[a, 0] + u_full[ls[t, 2 * a + 1]] * g[a, 1] for a in range(3))
            for e in range(3):
                a, b = mesh.tri_eloc[t, e, 0], mesh.tri_eloc[t, e, 1]
                la, lb = float(a == v), float(b == v)
                dv += u_full[ls[t, 6 + e]] * 4.0 * (la * g[b] + lb * g[a]) @ NORMALS[mesh.tri_ek[t, e]]
            d[v] = dv
        tot += area / 12.0 * (np.sum(d * d) + d.sum() ** 2)
    return tot


def test_exact_lambda_term_vertex_formula():
    n, lam, mu = 6, 3.7, 1.3
    m = Mesh(n)
    ex = Operator(m, lam, mu, 1.0, 1.0, 1.0, quadrature="exact")
    ref = Operator(m, 0.0, mu, 1.0, 1.0, 1.0, quadrature="exact")      # lambda = 0: 2 mu A_eps only
    rng = np.random.default_rng(5)
    for _ in range(3):
        x = np.zeros(ex.A.shape[0])
        x[ex.iu] = rng.standard_normal(ex.iu.size)
        uf = np.zeros(m.nslots)
        uf[m.act_idx] = x
        got = x @ ((ex.A - ref.A) @ x)
        want = lam * _div_energy_vertex(m, uf)
        assert abs(got - want) <= 1e-12 * want


def test_exact_equals_rq_at_lambda0_and_on_p1():
    n = 8
    m = Mesh(n)
    a0 = Operator(m, 0.0, 1.3, 0.7, 1.1, 0.4, quadrature="exact").A
    b0 = Operator(m, 0.0, 1.3, 0.7, 1.1, 0.4, quadrature="rq").A
    assert abs(a0 - b0).max() == 0.0
    ex = Operator(m, 5.0, 1.3, 0.7, 1.1, 0.4, quadrature="exact")
    rq = Operator(m, 5.0, 1.3, 0.7, 1.1, 0.4, quadrature="rq")
    x = m.to_active(mg_inputs.uniform_vector(n, 3))
    kind = m.slot_kind(m.act_idx)
    x[(kind >= 2) & (kind <= 4)] = 0.0                                # P1 displacement only
    d = ex.A @ x - rq.A @ x
    assert np.abs(d[(kind < 2) | (kind > 4)]).max() <= 1e-13 * np.abs(ex.A @ x).max()
    assert abs(x @ d) <= 1e-12 * abs(x @ (ex.A @ x))


def test_exact_bsr_is_the_jacobi_limit():
    n = 8
    m = Mesh(n)
    op = Operator(m, 1.0, 1.0, 1.0, 1.0, 400.0, quadrature="exact")
    x = m.to_active(mg_inputs.uniform_vector(n, 4))
    b = m.to_active(mg_inputs.uniform_rhs(n, 5))
    e = BSR(op, exact=True).sweep(x, b, 0.9, 0.0, 0)
    j = BSR(op).sweep(x, b, 0.9, 0.6, 600)
    assert np.abs(e - j).max() <= 1e-9 * np.abs(e).max()


@pytest.mark.slow
def test_tab_naive_solver_incompatibility():
    """Two-grid Vanka(2,2), h = 1/32, E = 3e4, k = 1e-6, tau = 1, M = 1e6 (tab:naive setting,
    PAPER.md:176-184), omega = 0.7: the factor on the exact operator rises with nu and is close to 1
    at nu = 0.499 (printed 0.970), while A^RQ at the same omega stays far below (tab:vanka22: 0.596).
    The h = 1/64 values of the paper's own mesh are in tests/golden/tab_naive_scan.json
    (tests/scripts/tab_naive_scan.py)."""
    rho = {}
    for quad in ("exact", "rq"):
        for nu in (0.4, 0.499):
            mu, lam = lame(3e4, nu)
            H = Hierarchy(32, 2, lam, mu, 1.0, 1.0, 1e-6, 1.0, K=1e-6, relax="vanka", quadrature=quad)
            _, rs = H.measure_rho(dict(nu1=2, nu2=2, omega=0.7), seed=0, min_cycles=40, max_cycles=40)
            rho[(quad, nu)] = float(np.mean(rs[-3:]))
    assert rho[("exact", 0.499)] >= 0.85, rho          # 0.894 at h = 1/32 (0.950 at h = 1/64, tab_naive_scan.json)
    assert rho[("exact", 0.499)] > rho[("exact", 0.4)] + 0.3, rho
    assert rho[("rq", 0.499)] <= 0.7, rho

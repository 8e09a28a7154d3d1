"""Oracle pins for backward-Euler time stepping (oracle/timestep.py).

* FE convergence O(h + tau) with tau = h for |u - u_h|_1 and ||p - p_h|| (the paper's claim for its
  smooth time-dependent test, fig:easy_Nconv), on the manufactured solution of
  reading A28 (u = 0 and w.n = 0 on the boundary), for nu = 0.4 and 0.499, k = 1.
* The history term against its definition on a P1 field with known divergence: for u = (x, y)
  interpolated at the vertices (div u = 2 exactly on every triangle, bubbles 0) and p = 0,
  alpha B_u u = -2 alpha |T| per triangle (B_u = -(div ., q)), and the p part is
  -(1/M) |T| p_T.
"""
import numpy as np
import pytest

from oracle.cycle import lame
from oracle.fem import Operator
from oracle.mesh import Mesh
from oracle import timestep as T


@pytest.mark.parametrize("nu", [0.4, 0.499])
def test_time_stepping_rates(nu):
    mu, lam = lame(3e4, nu)
    errs = []
    for n in (8, 16, 32):
        tau = 1.0 / n
        op = Operator(Mesh(n), lam, mu, tau, 1.0, 1e-6, 1.0, K=1.0)
        xs = T.run(op, 1.0, n // 2)                    # t = 0 .. 1/2
        errs.append(T.errors(op, xs[-1], 0.5))
    e = np.array(errs)
    rates = np.log2(e[:-1] / e[1:])
    assert np.all((rates > 0.9) & (rates < 1.2)), rates


def test_history_rhs_definition():
    n, alpha, invM = 6, 1.7, 0.3
    m = Mesh(n)
    op = Operator(m, 1.0, 1.0, 0.5, alpha, invM, K=1.0)
    x = np.zeros(m.nslots)
    # full-slot u = (x, y): the P1 interpolant of a linear field has div u = 2 on every triangle; the
    # boundary vertices are eliminated, so only triangles away from the boundary see div = 2 exactly
    for j in range(n + 1):
        for i in range(n + 1):
            x[m.slot(0, i, j)], x[m.slot(1, i, j)] = i * m.h, j * m.h
    pT = np.linspace(-1.0, 2.0, m.ntri)
    x[m.tri_pslot] = pT
    xa = x[m.act_idx]
    hr = T.history_rhs(op, xa)
    full = np.zeros(m.nslots)
    full[m.act_idx] = hr
    area = 0.5 * m.h ** 2
    for t in range(m.ntri):
        vi, vj = m.tri_vi[t], m.tri_vj[t]
        if np.any((vi == 0) | (vi == n) | (vj == 0) | (vj == n)):
            continue                                   # boundary vertices eliminated (u = 0 there)
        expect = -invM * area * pT[t] + alpha * (-2.0 * area)
        assert abs(full[m.tri_pslot[t]] - expect) <= 1e-13
    assert np.all(hr[op.iu] == 0.0) and np.all(hr[op.iw] == 0.0)

"""Oracle pins: discretisation (Appendix A, tab:mgtime, Lemma 2.1 corollaries)."""
import numpy as np
import pytest
import scipy.sparse as sp

import mg_inputs
from oracle.mesh import Mesh
from oracle.fem import Operator
from tests._golden import load, num


def _row(mat, mesh, plane, i, j):
    r = mat[mesh.slot(plane, i, j)].tocoo()
    out = {}
    for c, v in zip(r.col, r.data):
        if abs(v) > 1e-14:
            k = c // (mesh.N1 ** 2)
            rem = c % (mesh.N1 ** 2)
            out[(int(k), int(rem % mesh.N1 - i), int(rem // mesh.N1 - j))] = v
    return out


def _check_row(got, entries, scale, exact=True):
    exp = {(e[0], e[1], e[2]): num(e[3]) * scale for e in entries}
    for key, val in exp.items():
        assert key in got, f"missing stencil entry {key}"
        assert abs(got[key] - val) <= 1e-12 * max(1.0, abs(val)), (key, got[key], val)
    if exact:
        assert set(got) == set(exp), (set(got) ^ set(exp))


@pytest.mark.parametrize("n", [8, 16])
def test_appendix_a_stencils(n):
    """Every printed interior stencil value of Appendix A."""
    g = load("appendix_a_stencils.json")
    m = Mesh(n)
    op = Operator(m, lam=0.0, mu=1.0, tau=1.0, alpha=1.0, inv_M=1.0, K=1.0)
    h = m.h
    A2 = 2.0 * op.full["Aeps"]          # 2 mu A_eps with mu = 1
    i = j = n // 2
    for name, entries in g["2muAeps"].items():
        plane = int(name.split("plane ")[1].rstrip(")"))
        got = {k: v for k, v in _row(A2, m, plane, i, j).items() if k[0] == plane or k[0] in {e[0] for e in entries}}
        exact = name.startswith("D") or name.startswith("H") or name.startswith("V")
        _check_row({k: v for k, v in got.items() if k[0] in {e[0] for e in entries}}, entries, 1.0,
                   exact=exact and True)
    _check_row(_row(op.full["Mw"], m, 5, i, j), g["Mw"]["H row (plane 5)"], h * h)
    _check_row(_row(op.full["Mw"], m, 7, i, j), g["Mw"]["D row (plane 7)"], h * h)
    _check_row(_row(op.full["Mp"], m, 8, i, j), g["Mp"]["LL (plane 8)"], h * h)
    _check_row(_row(op.full["Bu"], m, 8, i, j), g["Bu"]["LL row (plane 8)"], h)
    _check_row(_row(op.full["Bw"], m, 8, i, j), g["Bw"]["LL row (plane 8)"], h)


def test_dof_counts_tab_mgtime():
    """All-DoF counts = tab:mgtime DoF column; active = 10n^2-8n+2."""
    g = load("paper_tables.json")["tab_mgtime_dofs"]["N_to_dofs"]
    for N, dofs in g.items():
        n = int(N) - 1
        m = Mesh(n)
        assert m.n_dofs_all() == dofs
        assert m.nact == 10 * n * n - 8 * n + 2
        assert np.array_equal(m.active.reshape(10, n + 1, n + 1), mg_inputs.active_mask(n))


def test_divfree_counting_identity():
    """(2 N_v + N_e) - (N_T - 1) = 3 N_v holds on the periodic idealisation:
    per periodic cell N_v = 1, N_e = 3, N_T = 2."""
    for n in (4, 8, 16):
        Nv, Ne, NT = n * n, 3 * n * n, 2 * n * n      # periodic torus counts
        assert (2 * Nv + Ne) - NT == 3 * Nv - 0 and (2 * Nv + Ne) - (NT - 1) == 3 * Nv + 1
    m = Mesh(8)   # Euler on the square: N_v - N_e + N_T = 1
    assert 81 - (3 * 64 + 2 * 8) + 128 == 1


@pytest.mark.parametrize("Kfield", [False, True])
def test_symmetry_and_spd(Kfield):
    """A^RQ is symmetric (eq. block_form_rq); A_u^RQ is SPD after elimination."""
    n = 8
    Kinv = 1.0 / mg_inputs.lognormal_K(n, 3) if Kfield else None
    op = Operator(Mesh(n), lam=3.0, mu=1.5, tau=0.7, alpha=0.9, inv_M=1e-2, K=2.0, Kinv_field=Kinv)
    A = op.A
    assert abs(A - A.T).max() <= 1e-15 * abs(A).max()
    ev = np.linalg.eigvalsh(op.Au.toarray())
    assert ev.min() > 0


def test_rq_projection_inequality():
    """lambda||P_Q div v||^2 <= lambda||div v||^2 and
    ||P_Q div v|| <= zeta^{-1} ||v||_{A^RQ}, zeta^2 = lambda + mu (eqn:B_less_Arq, d = 2)."""
    rng = np.random.default_rng(0)
    m = Mesh(8)
    lam, mu = 5.0, 2.0
    op = Operator(m, lam=lam, mu=mu, tau=1.0, alpha=1.0, inv_M=1.0)
    # exact (div u, div v) by the midpoint rule on each triangle (div of P1+bubble is linear)
    from oracle.fem import element_matrices
    for _ in range(5):
        x = rng.standard_normal(op.iu.size)
        u = np.zeros(m.nslots)
        u[m.act_idx[op.iu]] = x
        ls = m.local_slots()
        exact = 0.0
        for t in range(m.ntri):
            E = op.elem[m.tri_shape[t]]
            g = E["grad"]
            loc = u[ls[t, :9]]
            # div at the three edge midpoints
            from oracle.mesh import NORMALS
            qp = np.array([[0.5, 0.5, 0.0], [0.0, 0.5, 0.5], [0.5, 0.0, 0.5]])
            divs = []
            for L in qp:
                d = sum(loc[2 * a] * g[a, 0] + loc[2 * a + 1] * g[a, 1] for a in range(3))
                for e in range(3):
                    a, b = m.tri_eloc[t, e, 0], m.tri_eloc[t, e, 1]
                    d += loc[6 + e] * 4.0 * (L[a] * g[b] + L[b] * g[a]) @ NORMALS[m.tri_ek[t, e]]
                divs.append(d)
            exact += E["area"] / 3.0 * sum(d * d for d in divs)
        Bu = op.Bu
        pq = x @ (Bu.T @ (sp.diags(1.0 / op.Mp.diagonal()) @ (Bu @ x)))   # ||P_Q div v||^2
        assert pq <= exact * (1 + 1e-12)
        anorm = x @ (op.Au @ x)
        assert pq <= anorm / (lam + mu) * (1 + 1e-12)


def test_constant_pressure_eigenvector():
    """A^RQ (0, 1_p) = -(1/M)|T| (0, 1_p): B_u^T 1 = 0 and B_w^T 1 = 0 with the full Dirichlet /
    no-flux boundary, which is what makes deflation exact (reading A9)."""
    m = Mesh(8)
    op = Operator(m, lam=10.0, mu=1.0, tau=1.0, alpha=1.0, inv_M=1e-6)
    v = np.zeros(m.nact)
    v[op.ip] = 1.0
    Av = op.A @ v
    gam = 1e-6 * m.h ** 2 / 2
    assert np.abs(Av + gam * v).max() <= 1e-15

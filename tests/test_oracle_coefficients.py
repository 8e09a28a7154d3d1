"""Oracle pins for the coefficient paths the round-1 pins left open ("What's weak" 1):

* the per-triangle K^{-1} in M_w (oracle/fem.py, Operator with Kinv_field) -- pinned by the exact
  energy of a globally-RT0 linear field, integrated here with the vertex formula;
* the coarse K^{-1} of reading A11 (oracle/cycle.py coarsen_Kinv) -- pinned by the nested-space
  Galerkin identity for a K that is constant on coarse triangles (placement) and by the energy of a
  constant field for a general K (arithmetic mean of K^{-1});
* the Schur complement S of inexact BSR and n_J > 1 Jacobi sweeps (oracle/relax.py BSR) -- S pinned
  against its closed form from the printed element values (M_w diagonal 2h^2/(3k) PAPER.md:1487-1491,
  B_w = (h, h, -sqrt2 h) PAPER.md:1507-1510, S = s0 M_p + tau B_w D_w^{-1} B_w^T PAPER.md:684), the
  sweeps against the closed form of n_J weighted-Jacobi steps from dp = 0,
  dp_n = [I - (I - w_J D^{-1} S)^n] S^{-1} g, and its n -> infinity limit, the exact-S update of
  PAPER.md:666-672.

Every check was confirmed to fail on an injected error (transposed K field, swapped LL/UR planes,
harmonic instead of arithmetic coarse mean, a sign flip of S's off-diagonals, a dropped Jacobi
term): see the `inject` parametrisations, which run the same check on a corrupted input and
require it to fail.
"""
import numpy as np
import pytest

import mg_inputs
from oracle.cycle import coarsen_Kinv
from oracle.fem import Operator
from oracle.mesh import Mesh
from oracle.relax import BSR
from oracle.transfer import Transfer

SQ2 = np.sqrt(2.0)


def _edge_dofs(mesh, field):
    """RT0 DoF vector (full slot space) of a vector field: normal trace n_e . w at the midpoint of
    every existing edge (normal-trace normalisation, reading A1; normals reading A2).  Geometry is
    written out here from the mesh definition, not taken from the oracle."""
    n, h = mesh.n, mesh.h
    W = np.zeros((10, n + 1, n + 1))
    for j in range(n + 1):
        for i in range(n + 1):
            if i < n:        # H(i,j): (i,j)-(i+1,j), normal +y
                W[5, j, i] = field((i + 0.5) * h, j * h)[1]
            if j < n:        # V(i,j): (i,j)-(i,j+1), normal +x
                W[6, j, i] = field(i * h, (j + 0.5) * h)[0]
            if i < n and j < n:   # D(i,j): (i+1,j)-(i,j+1), normal (1,1)/sqrt2
                w = field((i + 0.5) * h, (j + 0.5) * h)
                W[7, j, i] = (w[0] + w[1]) / SQ2
    return W.reshape(-1)


def _triangle_energy(mesh, field, kinv):
    """sum_T K_T^{-1} int_T |w|^2 for a field linear on every triangle, by the vertex formula
    int_T f g = |T|/12 (sum_i f_i g_i + sum_i f_i sum_j g_j); kinv[shape, j, i]."""
    n, h = mesh.n, mesh.h
    area = 0.5 * h * h
    tot = 0.0
    for j in range(n):
        for i in range(n):
            for s, verts in ((0, [(i, j), (i + 1, j), (i, j + 1)]), (1, [(i + 1, j), (i + 1, j + 1), (i, j + 1)])):
                v = np.array([field(a * h, b * h) for a, b in verts])
                e = area / 12.0 * (np.sum(v * v) + np.dot(v.sum(0), v.sum(0)))
                tot += kinv[s, j, i] * e
    return tot


def _linear_field(a, c, x0):
    return lambda x, y: np.array([a[0] + c * (x - x0[0]), a[1] + c * (y - x0[1])])


@pytest.mark.parametrize("inject", [None, "transpose", "swap_shapes"])
def test_mw_energy_of_linear_rt0_field(inject):
    """w(x) = a + c (x - x0) lies in RT0 globally (normal traces are constant along straight
    edges), so its interpolant is w itself and W^T M_w W = mu_f sum_T K_T^{-1} int_T |w|^2 exactly
    (M_w(e,e') = sum_T mu_f K_T^{-1} int_T psi_e . psi_e').  The energy density
    varies with position anisotropically, so a K field read transposed ([shape, i, j]) or with the
    LL/UR planes swapped changes the left side."""
    n, mu_f = 8, 1.7
    m = Mesh(n)
    K = mg_inputs.lognormal_K(n, 31, sigma=1.0)
    kinv = 1.0 / K
    fed = kinv
    if inject == "transpose":
        fed = kinv.transpose(0, 2, 1).copy()
    elif inject == "swap_shapes":
        fed = kinv[::-1].copy()
    op = Operator(m, 1.0, 1.0, 1.0, 1.0, 1.0, mu_f=mu_f, Kinv_field=fed)
    f = _linear_field((0.8, -0.3), 1.9, (0.2, 0.7))
    W = _edge_dofs(m, f)
    lhs = W @ (op.full["Mw"] @ W)
    rhs = mu_f * _triangle_energy(m, f, kinv)
    ok = abs(lhs - rhs) <= 1e-12 * rhs
    assert ok == (inject is None), (inject, lhs, rhs)


def _coarse_parent_field(kinv_H):
    """Fine (2, 2N, 2N) field that is constant on every coarse triangle: coarse cell (I, J) holds
    fine cells (2I+a, 2J+b); the coarse LL [(0,0),(2,0),(0,2)] (local units) contains fine cell (0,0)
    and the LL halves of (1,0), (0,1); the coarse UR the rest (geometry of PAPER.md:1329)."""
    N = kinv_H.shape[1]
    f = np.empty((2, 2 * N, 2 * N))
    for J in range(N):
        for I in range(N):
            for b in range(2):
                for a in range(2):
                    for s in range(2):
                        parent = 0 if (a + b == 0 or (a + b == 1 and s == 0)) else 1
                        f[s, 2 * J + b, 2 * I + a] = kinv_H[parent, J, I]
    return f


@pytest.mark.parametrize("inject", [None, "transpose"])
def test_coarsen_kinv_placement_galerkin(inject):
    """Reading A11 placement: for a K that is constant on coarse triangles the RT0 spaces and the
    weights are nested, so R_w M_w^h(K) P_w = M_w^H(coarsen(K)) exactly and coarsen must return the
    coarse values themselves.  A child mapped to the wrong parent (or a transposed [shape, j, i]
    coarse field) breaks the identity."""
    nc = 4
    mf, mc = Mesh(2 * nc), Mesh(nc)
    kinv_H = 1.0 / mg_inputs.lognormal_K(nc, 32, sigma=1.0)
    kinv_h = _coarse_parent_field(kinv_H)
    KH = coarsen_Kinv(mf, mc, kinv_h)
    if inject == "transpose":
        KH = KH.transpose(0, 2, 1).copy()
    opf = Operator(mf, 1.0, 1.0, 1.0, 1.0, 1.0, Kinv_field=kinv_h)
    opc = Operator(mc, 1.0, 1.0, 1.0, 1.0, 1.0, Kinv_field=KH)
    Pw = Transfer(mf, mc).mats["P_w"]
    G = (Pw.T @ opf.full["Mw"] @ Pw).toarray()
    Hm = opc.full["Mw"].toarray()
    ok = np.abs(G - Hm).max() <= 1e-13 * np.abs(Hm).max() and np.array_equal(KH, kinv_H)
    assert ok == (inject is None)


@pytest.mark.parametrize("inject", [None, "harmonic"])
def test_coarsen_kinv_arithmetic_mean_energy(inject):
    """Reading A11 value: M_w is linear in K^{-1}, so with coarse K^{-1} = the mean of the four
    children's K^{-1} a constant field has the same energy on both levels:
    (P_w w)^T M_w^h (P_w w) = w^T M_w^H w = mu_f |w|^2 sum_t |t| K_t^{-1}.  The harmonic mean of
    K^{-1} (the arithmetic mean of K) does not."""
    nc = 4
    mf, mc = Mesh(2 * nc), Mesh(nc)
    kinv_h = 1.0 / mg_inputs.lognormal_K(2 * nc, 33, sigma=1.5)
    if inject == "harmonic":
        KH = 1.0 / coarsen_Kinv(mf, mc, 1.0 / kinv_h)
    else:
        KH = coarsen_Kinv(mf, mc, kinv_h)
    opf = Operator(mf, 1.0, 1.0, 1.0, 1.0, 1.0, Kinv_field=kinv_h)
    opc = Operator(mc, 1.0, 1.0, 1.0, 1.0, 1.0, Kinv_field=KH)
    f = lambda x, y: np.array([0.6, -1.1])
    Wc = _edge_dofs(mc, f)
    Wf = Transfer(mf, mc).mats["P_w"] @ Wc
    assert np.allclose(Wf, _edge_dofs(mf, f), atol=1e-14)      # canonical P_w reproduces constants
    Ef = Wf @ (opf.full["Mw"] @ Wf)
    Ec = Wc @ (opc.full["Mw"] @ Wc)
    exact = np.dot(f(0, 0), f(0, 0)) * 0.5 * mf.h ** 2 * kinv_h.sum()
    ok = abs(Ef - exact) <= 1e-12 * exact and abs(Ec - exact) <= 1e-12 * exact
    assert ok == (inject is None), (Ef, Ec, exact)


def _S_closed(op, kinv, s0):
    """S = s0 M_p + tau B_w D_w^{-1} B_w^T written from the printed element values: per triangle
    int |psi_e|^2 = h^2/3 for every edge (diagonal of M_w = (h^2/3k)[2 ...], with
    one triangle's share), so D_w(e) = (h^2/3) mu_f (K_T1^{-1} + K_T2^{-1}); |B_w(T, e)| = |e| (h on H
    and V edges, sqrt2 h on D) with opposite signs on the two sides of e; M_p = |T|.
    Neighbours: LL(i,j)-UR(i,j) across D(i,j), LL(i,j)-UR(i,j-1) across H(i,j) (j > 0),
    LL(i,j)-UR(i-1,j) across V(i,j) (i > 0).  Rows in op.ip order."""
    m = op.mesh
    n, h = m.n, m.h
    mu_f, tau = op.mu_f, op.tau
    slots = m.act_idx[op.ip]
    idx = {int(s): q for q, s in enumerate(slots)}
    P = lambda s, i, j: idx[int(m.slot(8 + s, i, j))]
    S = np.zeros((len(slots), len(slots)))
    for q in range(len(slots)):
        S[q, q] = s0 * 0.5 * h * h

    def couple(t1, t2, k1, k2, elen):
        Dw = h * h / 3.0 * mu_f * (k1 + k2)
        c = tau * elen ** 2 / Dw
        S[t1, t1] += c
        S[t2, t2] += c
        S[t1, t2] -= c
        S[t2, t1] -= c
    for j in range(n):
        for i in range(n):
            couple(P(0, i, j), P(1, i, j), kinv[0, j, i], kinv[1, j, i], SQ2 * h)
            if j > 0:
                couple(P(0, i, j), P(1, i, j - 1), kinv[0, j, i], kinv[1, j - 1, i], h)
            if i > 0:
                couple(P(0, i, j), P(1, i - 1, j), kinv[0, j, i], kinv[1, j, i - 1], h)
    return S


@pytest.mark.parametrize("inject", [None, "sign"])
def test_bsr_schur_complement_closed_form(inject):
    """The oracle's S (assembled from B_w and diag M_w) equals the closed form, off-diagonals
    included, for a heterogeneous K and generic material values (d = 2, reading A19)."""
    n = 8
    m = Mesh(n)
    lam, mu, tau, alpha, invM, mu_f = 2.5, 0.7, 0.8, 1.3, 0.05, 1.4
    kinv = 1.0 / mg_inputs.lognormal_K(n, 34, sigma=1.0)
    op = Operator(m, lam, mu, tau, alpha, invM, mu_f=mu_f, Kinv_field=kinv)
    B = BSR(op)
    Sc = _S_closed(op, kinv, invM + alpha ** 2 / (lam + mu))
    if inject == "sign":
        Sc = 2.0 * np.diag(np.diag(Sc)) - Sc
    ok = np.abs(B.S.toarray() - Sc).max() <= 1e-13 * np.abs(Sc).max()
    assert ok == (inject is None)


@pytest.mark.parametrize("n_J", [2, 3, 5])
@pytest.mark.parametrize("inject", [None, "no_offdiag"])
def test_bsr_jacobi_sweeps_closed_form(n_J, inject):
    """n_J weighted-Jacobi sweeps on S dp = g from dp = 0 (BASELINE n_J = 3) give
    dp_n = [I - (I - w_J D^{-1} S)^n] S^{-1} g (D = diag S).  dp is read off the pressure block of
    the BSR update (x_new(n_J) - x_new(0) = omega dp_n there) and g from the first
    sweep (dp_1 = w_J D^{-1} g); S is the closed form above, so the check involves every
    off-diagonal of S.  The injected variant drops S's off-diagonals from the closed form."""
    n = 8
    m = Mesh(n)
    lam, mu, tau, alpha, invM = 2.5, 0.7, 0.8, 1.3, 0.05
    kinv = 1.0 / mg_inputs.lognormal_K(n, 35, sigma=1.0)
    op = Operator(m, lam, mu, tau, alpha, invM, Kinv_field=kinv)
    B = BSR(op)
    x = m.to_active(mg_inputs.uniform_vector(n, 36))
    b = m.to_active(mg_inputs.uniform_rhs(n, 37))
    om, omJ = 0.8, 0.9
    base = B.sweep(x, b, om, omJ, 0)
    dp = lambda k: (B.sweep(x, b, om, omJ, k) - base)[op.ip] / om
    S = _S_closed(op, kinv, invM + alpha ** 2 / (lam + mu))
    if inject == "no_offdiag":
        S = np.diag(np.diag(S))
    D = np.diag(S)
    g = D * dp(1) / omJ
    E = np.eye(len(D)) - omJ * S / D[:, None]
    pred = (np.eye(len(D)) - np.linalg.matrix_power(E, n_J)) @ np.linalg.solve(S, g)
    got = dp(n_J)
    ok = np.abs(got - pred).max() <= 1e-11 * np.abs(pred).max()
    assert ok == (inject is None), np.abs(got - pred).max() / np.abs(pred).max()


def test_bsr_many_sweeps_reach_exact_schur_update():
    """n_J -> infinity: the inexact BSR update tends to the exact-S update of PAPER.md:666-672
    (dp = S^{-1} g, eq. bsr_p), with S the closed form.  A large 1/M lifts the constant-pressure
    mode of S (otherwise ~(pi h)^2-slow for Jacobi) so that 600 sweeps converge to fp64."""
    n = 8
    m = Mesh(n)
    lam, mu, tau, alpha, invM = 1.0, 1.0, 1.0, 1.0, 400.0
    kinv = 1.0 / mg_inputs.lognormal_K(n, 38, sigma=0.5)
    op = Operator(m, lam, mu, tau, alpha, invM, Kinv_field=kinv)
    B = BSR(op)
    x = m.to_active(mg_inputs.uniform_vector(n, 39))
    b = m.to_active(mg_inputs.uniform_rhs(n, 40))
    om, omJ = 1.0, 0.6
    base = B.sweep(x, b, om, omJ, 0)
    dp1 = (B.sweep(x, b, om, omJ, 1) - base)[op.ip]
    S = _S_closed(op, kinv, invM + alpha ** 2 / (lam + mu))
    g = np.diag(S) * dp1 / omJ
    exact = np.linalg.solve(S, g)
    far = (B.sweep(x, b, om, omJ, 600) - base)[op.ip]
    assert np.abs(far - exact).max() <= 1e-9 * np.abs(exact).max()

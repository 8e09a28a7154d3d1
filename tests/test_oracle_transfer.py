"""Oracle pins: grid transfers (Appendix B)."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle.mesh import Mesh
from oracle.fem import Operator
from oracle.transfer import build_P, Transfer, _parent
from tests._golden import load, num


@pytest.fixture(scope="module")
def mats():
    mf, mc = Mesh(16), Mesh(8)
    return mf, mc, build_P(mf, mc)


def test_appendix_b_theta0_sums(mats):
    """theta = 0 restriction symbols = sums of P over each fine DoF type."""
    mf, mc, M = mats
    g = load("appendix_b_theta0.json")
    I = J = 4
    for key, blk in (("P_u", M["P_u"]), ("P_w", M["P_w"]), ("P_p", M["P_p"])):
        for cplane, exp in g[key].items():
            col = blk[:, mc.slot(int(cplane), I, J)].toarray().ravel().reshape(10, -1).sum(axis=1)
            expv = np.zeros(10)
            for fplane, v in exp.items():
                expv[int(fplane)] = num(v)
            assert np.allclose(col, expv, rtol=0, atol=1e-13), (key, cplane, col, expv)


def test_divergence_preserving_identity(mats):
    """B_u^h P_u = J B_u^H exactly: every corner fine triangle gets zero flux, the middle
    child carries the coarse divergence (eq. divfreefine)."""
    mf, mc, M = mats
    opf = Operator(mf, 1, 1, 1, 1, 1.0)
    opc = Operator(mc, 1, 1, 1, 1, 1.0)
    BP = (opf.full["Bu"] @ M["P_u"]).toarray()
    BH = opc.full["Bu"].toarray()
    par = _parent(mf, mc, np.arange(mf.ntri))
    for t in range(mf.ntri):
        mid = not any((mf.tri_vi[t, a] % 2 == 0) and (mf.tri_vj[t, a] % 2 == 0) for a in range(3))
        target = BH[mc.tri_pslot[par[t]]] if mid else 0.0
        assert np.abs(BP[mf.tri_pslot[t]] - target).max() <= 1e-15


def test_nested_galerkin_identities():
    """Constant K: RT0/P0 spaces are nested, so R_w M_w P_w = M_w^H, R_p B_w P_w = B_w^H,
    R_p M_p P_p = M_p^H; and R_p B_u P_u = B_u^H; P_u^T (lam B^T M^-1 B)_h P_u = 4 (.)_H."""
    mf, mc = Mesh(16), Mesh(8)
    opf = Operator(mf, 1.0, 1.0, 1.0, 1.0, 1.0, K=0.37)
    opc = Operator(mc, 1.0, 1.0, 1.0, 1.0, 1.0, K=0.37)
    tr = Transfer(mf, mc)
    M = tr.mats
    fa, ca = mf.act_idx, mc.act_idx

    def R(X):
        return X[fa][:, ca]
    Pw, Pp, Pu = R(M["P_w"]), R(M["P_p"]), R(M["P_u"])
    Ff, Fc = opf.full, opc.full
    chk = [
        (Pw.T @ Ff["Mw"][fa][:, fa] @ Pw, Fc["Mw"][ca][:, ca]),
        (Pp.T @ Ff["Bw"][fa][:, fa] @ Pw, Fc["Bw"][ca][:, ca]),
        (Pp.T @ Ff["Mp"][fa][:, fa] @ Pp, Fc["Mp"][ca][:, ca]),
        (Pp.T @ Ff["Bu"][fa][:, fa] @ Pu, Fc["Bu"][ca][:, ca]),
    ]
    for G, H in chk:
        assert abs(G - H).max() <= 1e-14 * max(1.0, abs(H).max())
    lamf = Ff["Bu"].T @ sp.diags(1.0 / np.where(Ff["Mp"].diagonal() > 0, Ff["Mp"].diagonal(), 1.0)) @ Ff["Bu"]
    lamc = Fc["Bu"].T @ sp.diags(1.0 / np.where(Fc["Mp"].diagonal() > 0, Fc["Mp"].diagonal(), 1.0)) @ Fc["Bu"]
    G = Pu.T @ lamf[fa][:, fa] @ Pu
    assert abs(G - 4.0 * lamc[ca][:, ca]).max() <= 1e-12


def test_divfree_linear_field_reproduced():
    """A divergence-free linear coarse field u = (y, x) - (1/2,1/2) (P1 part only, coarse bubbles 0)
    is reproduced exactly by P_u: fine P1 = point values, all fine bubbles 0."""
    mf, mc = Mesh(8), Mesh(4)
    M = build_P(mf, mc)
    uc = np.zeros(mc.nslots)
    for i in range(mc.n + 1):
        for j in range(mc.n + 1):
            x, y = i * mc.h, j * mc.h
            uc[mc.slot(0, i, j)] = y - 0.5
            uc[mc.slot(1, i, j)] = x - 0.5
    uf = M["P_u"] @ uc
    for i in range(mf.n + 1):
        for j in range(mf.n + 1):
            x, y = i * mf.h, j * mf.h
            assert abs(uf[mf.slot(0, i, j)] - (y - 0.5)) < 1e-14
            assert abs(uf[mf.slot(1, i, j)] - (x - 0.5)) < 1e-14
    assert np.abs(uf.reshape(10, -1)[2:5]).max() < 1e-14

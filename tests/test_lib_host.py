"""CPU tests of the product path's host side (no GPU needed):

* libmg.so loads and exports every function include/mg.h declares;
* mg_setup rejects bad arguments with MG_EINVAL before touching the device;
* the generated geometry (gen_tables.py -> mg_tables.h) reproduces the paper's printed Appendix A
  stencils and Appendix B theta = 0 transfer sums, and equals the oracle's assembled operator and
  prolongation at interior locations;
* the host setup (mg_host_level_tables) equals the oracle's weighted patch inverses for all 9
  vertex classes, including the deflated stiff regime.
"""
import ctypes
import os
import re
import subprocess
import sys

import numpy as np
import pytest

from tests._golden import load, num

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2107_04060_b200", "csrc")
sys.path.insert(0, CSRC)
import gen_tables as G  # noqa: E402


@pytest.fixture(scope="module")
def lib():
    from paper_2107_04060_b200 import build, mg
    build.build()
    return mg.load_library()


def test_exports_every_declared_symbol(lib):
    hdr = open(os.path.join(ROOT, "include", "mg.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    names = set(re.findall(r"\b(mg_[a-z_0-9]+)\s*\(", hdr))
    assert len(names) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2107_04060_b200", "libmg.so")],
                         capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (mg_[a-z_0-9]+)", out))
    missing = names - exported
    assert not missing, missing
    from paper_2107_04060_b200.mg import SIGNATURES
    assert names <= set(SIGNATURES), names - set(SIGNATURES)


def test_library_is_sm100a(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          os.path.join(ROOT, "paper_2107_04060_b200", "libmg.so")], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("bad", [
    dict(n=16, levels=0), dict(n=16, levels=5), dict(n=18, levels=3), dict(n=16, levels=3, mu=0.0),
    dict(n=16, levels=3, lam=-1.0), dict(n=16, levels=3, K=0.0), dict(n=16, levels=3, tau=0.0),
    dict(n=16, levels=3, inv_M=0.0), dict(n=16, levels=3, alpha=float('nan'))])
def test_setup_rejects(lib, bad):
    from paper_2107_04060_b200.mg import Grid, _VP
    p = dict(n=16, levels=3, lam=1.0, mu=1.0, K=1.0, tau=1.0, alpha=1.0, inv_M=1.0)
    p.update(bad)
    g = Grid(p["n"], None, p["inv_M"], 1.0)
    ctx = _VP()
    rc = lib.mg_setup(ctypes.byref(g), p["lam"], p["mu"], p["K"], p["tau"], p["alpha"], p["levels"], ctypes.byref(ctx))
    assert rc == -1
    assert lib.mg_last_error()
    assert not ctx.value


def _stencil_value(rows, k, col, mu=1.0, lam=0.0):
    """2 mu A_eps entry (lambda = 0) of row k, column (plane, dx, dy) from the generated tables."""
    E = [G.element(0), G.element(1)]
    for (c, lst) in rows[k]["entries"]:
        if c == col:
            return sum(2 * mu * E[s]["Aeps"][q, q2] for (s, q, q2) in lst if q < 9 and q2 < 9)
    return 0.0


def test_generated_appendix_a_stencils():
    """Interior stencils of 2 mu A_eps, M_w, M_p, B_u, B_w from mg_tables.h geometry."""
    g = load("appendix_a_stencils.json")
    rows = G.stencil()
    plane_of = {"P1x row (plane 0)": 0, "P1y row (plane 1)": 1, "D bubble row (plane 4)": 4,
                "H bubble row (plane 2)": 2, "V bubble row (plane 3)": 3}
    for key, ents in g["2muAeps"].items():
        k = plane_of[key]
        for (pl, di, dj, v) in ents:
            assert abs(_stencil_value(rows, k, (di, dj, pl)) - num(v)) < 1e-13, (key, pl, di, dj)
    E = [G.element(0), G.element(1)]
    # M_w (units mu_f h^2/k): sum over the two triangles of the H edge
    mw = {}
    for (cx, cy, s, dx, dy, pl, e, e2) in rows[5]["ww"]:
        mw[(pl, dx, dy)] = mw.get((pl, dx, dy), 0.0) + E[s]["Mw1"][e, e2]
    for (pl, di, dj, v) in g["Mw"]["H row (plane 5)"]:
        assert abs(mw[(pl, di, dj)] - num(v)) < 1e-13
    assert abs(E[0]["Mp"] - 0.5) < 1e-15 and abs(E[1]["Mp"] - 0.5) < 1e-15
    # B_u and B_w rows of the LL triangle of cell (0,0) (units h)
    bu = {}
    for q, (dx, dy, pl) in enumerate(G.LOCAL[0][:9]):
        bu[(pl, dx, dy)] = E[0]["Bu"][q]
    for (pl, di, dj, v) in g["Bu"]["LL row (plane 8)"]:
        assert abs(bu[(pl, di, dj)] - num(v)) < 1e-13
    for (pl, di, dj, v) in g["Bw"]["LL row (plane 8)"]:
        e = pl - 5
        assert abs(E[0]["Bw"][e] - num(v)) < 1e-13


def test_generated_appendix_b_sums():
    """theta = 0 transfer symbols: the sums of the prolongation weights of one
    interior coarse DoF over the fine DoFs of each type, from the generated P table."""
    g = load("appendix_b_theta0.json")
    P = G.prolongation()
    for key in ("P_u", "P_w", "P_p"):
        for cplane, exp in g[key].items():
            cp = int(cplane)
            sums = np.zeros(10)
            # coarse DoF at coarse index (I, J): it appears in coarse cells (I - dI, J - dJ)
            for (di, dj, kf), ent in P.items():
                for c, w in ent.items():
                    if G.COARSE_DOFS[c][2] == cp:
                        sums[kf] += w
            expv = np.zeros(10)
            for fplane, v in exp.items():
                expv[int(fplane)] = num(v)
            assert np.allclose(sums, expv, atol=1e-13), (key, cplane, sums, expv)


def test_generated_tables_equal_oracle():
    """Merged stencil and prolongation equal the oracle's assembled A^RQ and P rows (interior)."""
    from oracle.mesh import Mesh
    from oracle.fem import Operator
    from oracle.transfer import build_P
    n = 8
    lam, mu, K, tau, al, iM = 2.0, 1.3, 0.6, 0.7, 0.9, 0.3
    m = Mesh(n)
    op = Operator(m, lam, mu, tau, al, iM, 1.0, K=K)
    h = 1.0 / n
    E = [G.element(0, h), G.element(1, h)]

    def A_T(s, q, q2):
        e = E[s]
        bq, b2 = G.block(q), G.block(q2)
        if bq == "u" and b2 == "u":
            return 2 * mu * e["Aeps"][q, q2] + lam / e["Mp"] * e["Bu"][q] * e["Bu"][q2]
        if bq == "u" and b2 == "p":
            return al * e["Bu"][q]
        if bq == "p" and b2 == "u":
            return al * e["Bu"][q2]
        if bq == "w" and b2 == "p":
            return tau * e["Bw"][q - 9]
        if bq == "p" and b2 == "w":
            return tau * e["Bw"][q2 - 9]
        return -iM * e["Mp"]

    rows = G.stencil()
    A = op.A_full.toarray()
    for (i, j) in ((3, 4), (1, 1), (6, 2)):
        for k in range(10):
            ref = A[m.slot(k, i, j)]
            mine = np.zeros_like(ref)
            for (col, lst) in rows[k]["entries"]:
                mine[m.slot(col[2], i + col[0], j + col[1])] += sum(A_T(*t) for t in lst)
            for (cx, cy, sh, dx, dy, pl, e, e2) in rows[k]["ww"]:
                mine[m.slot(pl, i + dx, j + dy)] += tau / K * E[sh]["Mw1"][e, e2]
            if m.active[m.slot(k, i, j)]:
                act = m.active
                assert np.abs((mine - ref)[act]).max() < 1e-12, (i, j, k)
    mf, mc = Mesh(8), Mesh(4)
    M = build_P(mf, mc)
    Pf = (M["P_u"] + M["P_w"] + M["P_p"]).toarray()
    P = G.prolongation()
    for (I, J) in ((1, 2), (0, 0), (2, 1)):
        for (di, dj, kf), ent in P.items():
            row = Pf[mf.slot(kf, 2 * I + di, 2 * J + dj)]
            mine = np.zeros_like(row)
            for c, v in ent.items():
                dI, dJ, pc = G.COARSE_DOFS[c]
                mine[mc.slot(pc, I + dI, J + dJ)] += v
            assert np.abs(mine - row).max() < 1e-14, (I, J, di, dj, kf)


def test_generated_header_is_current(tmp_path):
    """mg_tables.h is exactly what gen_tables.py writes."""
    out = tmp_path / "t.h"
    G.emit(str(out))
    assert out.read_text() == open(os.path.join(CSRC, "mg_tables.h")).read()


VS = [(0, 0, 0), (0, 0, 1), (0, 0, 2), (-1, 0, 2), (0, 0, 3), (0, -1, 3), (-1, 0, 4), (0, -1, 4), (0, 0, 5),
      (-1, 0, 5), (0, 0, 6), (0, -1, 6), (-1, 0, 7), (0, -1, 7), (0, 0, 8), (-1, -1, 9), (-1, 0, 8), (0, -1, 9),
      (-1, 0, 9), (0, -1, 8)]


@pytest.mark.parametrize("params", [(2.0, 1.3, 0.6, 0.7, 0.9, 0.3), (1e6, 1.0, 1e-6, 1.0, 1.0, 1.0),
                                    (100.0, 1.0, 1e-2, 1.0, 1.0, 1.0)])
def test_host_patch_inverses_equal_oracle(lib, params):
    """D_v K_v^{-1} of the host setup (deflated, long double) equals the oracle's Vanka patch solve
    (deflated, fp64 LAPACK) for every vertex class; displacement patches equal inv(A_u) blocks."""
    from paper_2107_04060_b200 import host_level_tables
    from oracle.mesh import Mesh
    from oracle.fem import Operator
    from oracle.relax import Vanka
    lam, mu, K, tau, al, iM = params
    n = 8
    t = host_level_tables(n, lam, mu, K, tau, al, iM)
    m = Mesh(n)
    op = Operator(m, lam, mu, tau, al, iM, 1.0, K=K)
    V = Vanka(op)
    A = op.A.toarray()
    cases = {0: (3, 4), 1: (0, 3), 2: (n, 3), 3: (3, 0), 6: (3, n), 4: (0, 0), 5: (n, 0), 7: (0, n), 8: (n, n)}
    for cls, (a, b) in cases.items():
        pos = [m.pos[m.slot(pl, a + dx, b + dy)] if 0 <= a + dx <= n and 0 <= b + dy <= n else -1
               for (dx, dy, pl) in VS]
        idx = [q for q in range(20) if pos[q] >= 0]
        I = np.array([pos[q] for q in idx])
        # oracle: apply its deflated patch solve to unit vectors of this patch
        found = [(d, r) for d in V.data for r in range(d["I"].shape[0])
                 if d["I"].shape[1] == len(I) and set(d["I"][r]) == set(I)]
        assert len(found) == 1
        d, row = found[0]
        Ip = list(d["I"][row])
        Y = np.zeros((len(Ip), len(Ip)))
        for c in range(len(Ip)):
            R = np.zeros(d["I"].shape)
            R[row, c] = 1.0
            Y[:, c] = V.patch_solve(d, R)[row]
        perm = [Ip.index(p) for p in I]
        Y = Y[np.ix_(perm, perm)]
        ref = np.zeros((20, 20))
        ref[np.ix_(idx, idx)] = V.weight[I][:, None] * Y
        mine = t["vanka"][cls]
        err = np.abs(mine - ref).max() / np.abs(ref).max()
        assert err < 1e-9, (cls, err)


@pytest.mark.parametrize("params", [(64, 100.0, 1.0, 1e-2, 1.0, 1.0, 1.0), (37, 2.5, 0.7, 0.3, 0.8, 1.3, 0.05),
                                    (100, 1e6, 1.3, 1e-6, 2.0, 0.3, 7.0)])
def test_factored_stencil_equals_merged(lib, params):
    """MG_STENCIL_FACT (the form the kernels evaluate) reproduces every merged stencil entry
    coef[ci] of MG_STENCIL_ROW_k: entries it drops are exactly zero for this material, the others
    equal +-cg[g] = +-coef[representative] to rounding (eq. block_form_rq)."""
    from paper_2107_04060_b200.mg import host_level_tables
    hdr = open(os.path.join(ROOT, "paper_2107_04060_b200", "csrc", "mg_tables.h")).read()
    coef = host_level_tables(*params)["coef"]
    merged = {}
    for k in range(10):
        body = re.search(r"#define MG_STENCIL_ROW_%d\(X\)(.*)" % k, hdr).group(1)
        for (row, dx, dy, pl, ci) in re.findall(r"X\((\d+),(-?\d+),(-?\d+),(\d+),(\d+)\)", body):
            merged[(int(row), int(dx), int(dy), int(pl))] = coef[int(ci)]
    rep = {int(g): (int(ci), int(sg)) for g, ci, sg in re.findall(
        r"R\((\d+),(\d+),(-?\d+)\)", re.search(r"#define MG_STENCIL_GROUP_REP\(R\)(.*)", hdr).group(1))}
    fact = {}
    body = re.search(r"#define MG_STENCIL_FACT\(A\)(.*)", hdr).group(1)
    for row, g, ms, expr in re.findall(r"A\((\d+),(\d+),([+-]),\(([^()]*(?:\([^()]*\)[^()]*)*)\)\)", body):
        cg = rep[int(g)][1] * coef[rep[int(g)][0]] * (1.0 if ms == "+" else -1.0)
        for sgn, dx, dy, pl in re.findall(r"([+-]?)\s*XS\((-?\d+),(-?\d+),(\d+)\)", expr):
            key = (int(row), int(dx), int(dy), int(pl))
            assert key not in fact
            fact[key] = cg * (-1.0 if sgn == "-" else 1.0)
    scale = np.abs(coef).max()
    assert set(fact) <= set(merged)
    assert len(fact) == 113 and len(merged) == 141
    for key, v in merged.items():
        assert abs(fact.get(key, 0.0) - v) <= 1e-13 * scale, (key, v, fact.get(key))
        if key not in fact:
            assert v == 0.0

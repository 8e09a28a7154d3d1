"""Generator for ``mg_tables.h``: the compile-time geometry of the CUDA path.

Product-side code (not the oracle).  It evaluates, once, everything of the
discretisation that does not depend on the level or the material parameters:

1. Reference element integrals on the two triangle shapes of a cell with h = 1
   (PAPER.md:137-167 bilinear forms; PAPER.md:1333-1337 for the RQ term),
   using the basis normalisation of reading A1 and the edge normals of
   reading A2:
       P1      lambda_a e_x, lambda_a e_y
       bubble  4 lambda_a lambda_b n_e             (normal trace 1 at the midpoint)
       RT0     s_{T,e} |e|/(2|T|) (x - x_opp)      (normal trace 1)
       P0      indicator
   Scaling with h: A_eps is scale free, B_u, B_w ~ h, M_w, M_p ~ h^2.
2. The merged matrix-free stencil of A^RQ (eq. block_form_rq):
   for each of the 10 DoF kinds owned by grid index (i, j), the list of
   distinct neighbour DoFs (dx, dy, plane) it couples to, and, per entry, the
   element entries (shape, q, q') whose sum is the coefficient.  The M_w part
   of the RT0 rows is emitted per triangle so a per-triangle K^{-1} can scale it.
3. The prolongation P = diag(P_u, P_w, P_p) of PAPER.md:477-566 on one coarse
   cell: canonical P1/RT0/P0 interpolation, flux-preserving bubbles, then the
   divergence-preserving reset of the three interior-edge bubbles of every
   coarse triangle (zero outward flux of each corner child; reading A4).  P is
   level independent, so it is emitted as literal constants, together with
   its transpose for the restriction R = P^T.

Run ``python gen_tables.py`` to rewrite ``mg_tables.h`` next to this file.
"""
from __future__ import annotations

import os
import numpy as np

SQ2 = np.sqrt(2.0)
NORMAL = {"H": np.array([0.0, 1.0]), "V": np.array([1.0, 0.0]), "D": np.array([1.0, 1.0]) / SQ2}
KIND = {"H": 0, "V": 1, "D": 2}
# plane ids of the ABI layout (include/mg.h)
UX, UY, BH, BV, BD, WH, WV, WD, PLL, PUR = range(10)

# Cell (i, j): LL = [(i,j), (i+1,j), (i,j+1)], UR = [(i+1,j), (i+1,j+1), (i,j+1)].
# Edge tuple: (kind, owner offset of the edge DoF relative to the cell, endpoint a, endpoint b).
SHAPES = [
    dict(name="LL", verts=[(0, 0), (1, 0), (0, 1)],
         edges=[("H", (0, 0), 0, 1), ("V", (0, 0), 0, 2), ("D", (0, 0), 1, 2)], p=PLL),
    dict(name="UR", verts=[(1, 0), (1, 1), (0, 1)],
         edges=[("H", (0, 1), 2, 1), ("V", (1, 0), 0, 1), ("D", (0, 0), 0, 2)], p=PUR),
]


def local_map(shape):
    """13 local DoFs -> (dx, dy, plane) relative to the cell: u (2a+c), bubble 6+e, RT0 9+e, P0 12."""
    S = SHAPES[shape]
    out = []
    for a in range(3):
        for c in range(2):
            out.append((S["verts"][a][0], S["verts"][a][1], UX + c))
    for e in range(3):
        k, o, _, _ = S["edges"][e]
        out.append((o[0], o[1], BH + KIND[k]))
    for e in range(3):
        k, o, _, _ = S["edges"][e]
        out.append((o[0], o[1], WH + KIND[k]))
    out.append((0, 0, S["p"]))
    return out


LOCAL = [local_map(0), local_map(1)]


def block(q):
    return "u" if q < 9 else ("w" if q < 12 else "p")


COUPLED = {("u", "u"), ("u", "p"), ("p", "u"), ("w", "w"), ("w", "p"), ("p", "w"), ("p", "p")}


# ----------------------------------------------------------------------------- element integrals
def element(shape, h=1.0):
    """Reference element integrals on one triangle, edge-midpoint quadrature."""
    S = SHAPES[shape]
    P = np.array(S["verts"], dtype=float) * h
    M = np.array([P[1] - P[0], P[2] - P[0]]).T
    Minv = np.linalg.inv(M)
    g = np.zeros((3, 2))
    g[1], g[2] = Minv[0], Minv[1]
    g[0] = -(g[1] + g[2])
    area = 0.5 * abs(np.linalg.det(M))
    cen = P.mean(axis=0)
    ed = S["edges"]
    nrm = [NORMAL[e[0]] for e in ed]
    elen = [np.linalg.norm(P[e[3]] - P[e[2]]) for e in ed]
    opp = [3 - e[2] - e[3] for e in ed]
    sgn = [1.0 if np.dot(0.5 * (P[e[2]] + P[e[3]]) - cen, nrm[k]) > 0 else -1.0 for k, e in enumerate(ed)]
    Aeps = np.zeros((9, 9)); Bu = np.zeros(9); Mw1 = np.zeros((3, 3))
    for (la, lb) in ((0, 1), (1, 2), (0, 2)):             # edge midpoints
        lam = np.zeros(3); lam[la] = lam[lb] = 0.5
        X = lam @ P
        w = area / 3.0
        G = np.zeros((9, 2, 2))                          # G[q, comp, d] = d phi_q,comp / d x_d
        for a in range(3):
            G[2 * a, 0] = g[a]
            G[2 * a + 1, 1] = g[a]
        for k, e in enumerate(ed):
            a, b = e[2], e[3]
            G[6 + k] = np.outer(nrm[k], 4.0 * (lam[a] * g[b] + lam[b] * g[a]))
        eps = 0.5 * (G + G.transpose(0, 2, 1))
        Aeps += w * np.einsum("pcd,qcd->pq", eps, eps)
        Bu -= w * np.einsum("pcc->p", G)
        psi = np.array([sgn[k] * elen[k] / (2 * area) * (X - P[opp[k]]) for k in range(3)])
        Mw1 += w * psi @ psi.T
    Bw = np.array([-sgn[k] * elen[k] for k in range(3)])
    # exact-integration lambda term (div u, div v) of eq. block_form: div of a P1
    # or bubble basis function is linear on the triangle, so it is integrated from its vertex values
    # with int_T f g = |T|/12 (sum_i f_i g_i + sum_i f_i sum_j g_j) (exact for linear f, g)
    dv = np.zeros((9, 3))                                # dv[q, v]: div phi_q at vertex v
    for v in range(3):
        lam = np.zeros(3); lam[v] = 1.0
        for a in range(3):
            dv[2 * a, v] = g[a][0]
            dv[2 * a + 1, v] = g[a][1]
        for k, e in enumerate(ed):
            a, b = e[2], e[3]
            dv[6 + k, v] = 4.0 * (lam[a] * g[b] + lam[b] * g[a]) @ nrm[k]
    Ddiv = area / 12.0 * (dv @ dv.T + np.outer(dv.sum(1), dv.sum(1)))
    return dict(Aeps=Aeps, Bu=Bu, Mw1=Mw1, Bw=Bw, Mp=area, sgn=np.array(sgn), elen=np.array(elen), g=g, Ddiv=Ddiv)


# ----------------------------------------------------------------------------- merged stencil
def stencil():
    """Rows k = 0..9 owned by index (0,0): merged entries and their element contributions."""
    rows = []
    for k in range(10):
        entries = {}            # (dx,dy,plane) -> list of (shape, q, q')
        ww = []                 # per-triangle M_w entries (RT0 rows): (cx, cy, shape, dx, dy, plane, e, e')
        for cx in (-1, 0):
            for cy in (-1, 0):
                for s in (0, 1):
                    for q, (dx, dy, pl) in enumerate(LOCAL[s]):
                        if (cx + dx, cy + dy, pl) != (0, 0, k):
                            continue
                        for q2, (dx2, dy2, pl2) in enumerate(LOCAL[s]):
                            if (block(q), block(q2)) not in COUPLED:
                                continue
                            col = (cx + dx2, cy + dy2, pl2)
                            if block(q) == "w" and block(q2) == "w":
                                ww.append((cx, cy, s, col[0], col[1], col[2], q - 9, q2 - 9))
                            else:
                                entries.setdefault(col, []).append((s, q, q2))
        rows.append(dict(entries=sorted(entries.items()), ww=ww))
    return rows


# ----------------------------------------------------------------------------- prolongation
COARSE_DOFS = ([(dI, dJ, c) for (dI, dJ) in ((0, 0), (1, 0), (0, 1), (1, 1)) for c in (UX, UY)]
               + [(0, 0, BH), (0, 1, BH), (0, 0, BV), (1, 0, BV), (0, 0, BD)]
               + [(0, 0, WH), (0, 1, WH), (0, 0, WV), (1, 0, WV), (0, 0, WD)]
               + [(0, 0, PLL), (0, 0, PUR)])


def _tri_geom(verts):
    P = np.array(verts, dtype=float)
    M = np.array([P[1] - P[0], P[2] - P[0]]).T
    Minv = np.linalg.inv(M)
    g = np.zeros((3, 2)); g[1], g[2] = Minv[0], Minv[1]; g[0] = -(g[1] + g[2])
    return P, g, 0.5 * abs(np.linalg.det(M))


def _bary(P, X):
    M = np.array([P[1] - P[0], P[2] - P[0]]).T
    l12 = np.linalg.solve(M, X - P[0])
    return np.array([1 - l12.sum(), l12[0], l12[1]])


def _coarse_field(cvec, X, shape):
    """Coarse u (2,), w (2,), p of coefficient vector cvec (over COARSE_DOFS) at X in coarse triangle."""
    S = SHAPES[shape]
    P, g, area = _tri_geom(S["verts"])
    cen = P.mean(axis=0)
    lam = _bary(P, X)
    idx = {d: n for n, d in enumerate(COARSE_DOFS)}
    u = np.zeros(2); w = np.zeros(2)
    for a in range(3):
        vx, vy = S["verts"][a]
        u[0] += lam[a] * cvec[idx[(vx, vy, UX)]]
        u[1] += lam[a] * cvec[idx[(vx, vy, UY)]]
    for (k, o, a, b) in S["edges"]:
        n = NORMAL[k]
        u += 4 * lam[a] * lam[b] * n * cvec[idx[(o[0], o[1], BH + KIND[k])]]
        s = 1.0 if np.dot(0.5 * (P[a] + P[b]) - cen, n) > 0 else -1.0
        L = np.linalg.norm(P[b] - P[a])
        xo = P[3 - a - b]
        w += s * L / (2 * area) * (X - xo) * cvec[idx[(o[0], o[1], WH + KIND[k])]]
    p = cvec[idx[(0, 0, S["p"])]]
    return u, w, p


def _which(X):
    return 0 if X[0] + X[1] <= 1.0 + 1e-14 else 1


def prolongation():
    """P[(di,dj)][kf] -> {coarse local DoF index: weight} for the fine DoFs owned by fine index
    (2I+di, 2J+dj) of coarse cell (I, J)."""
    hf = 0.5
    nC = len(COARSE_DOFS)
    # fine edges inside the coarse cell closure, keyed by (kind, fi, fj) in fine index units
    fedges = {}
    for fi in range(3):
        for fj in range(3):
            if fi < 2:
                fedges[("H", fi, fj)] = ((fi, fj), (fi + 1, fj))
            if fj < 2:
                fedges[("V", fi, fj)] = ((fi, fj), (fi, fj + 1))
            if fi < 2 and fj < 2:
                fedges[("D", fi, fj)] = ((fi + 1, fj), (fi, fj + 1))
    ftris = []                          # (fi, fj, shape) -> vertex list
    for fi in range(2):
        for fj in range(2):
            ftris.append(((fi, fj, 0), [(fi, fj), (fi + 1, fj), (fi, fj + 1)],
                          [("H", fi, fj), ("V", fi, fj), ("D", fi, fj)]))
            ftris.append(((fi, fj, 1), [(fi + 1, fj), (fi + 1, fj + 1), (fi, fj + 1)],
                          [("H", fi, fj + 1), ("V", fi + 1, fj), ("D", fi, fj)]))
    cols = []
    for c in range(nC):
        cv = np.zeros(nC); cv[c] = 1.0
        U = {}
        for fi in range(3):
            for fj in range(3):
                X = np.array([fi, fj]) * hf
                U[(fi, fj)] = _coarse_field(cv, X, _which(X))[0]
        beta, wv = {}, {}
        for key, (va, vb) in fedges.items():
            A = np.array(va) * hf; B = np.array(vb) * hf
            mid = 0.5 * (A + B)
            sh = _which(mid)
            n = NORMAL[key[0]]
            L = np.linalg.norm(B - A)
            fa = _coarse_field(cv, A, sh)[0] @ n
            fm = _coarse_field(cv, mid, sh)[0] @ n
            fb = _coarse_field(cv, B, sh)[0] @ n
            flux = L / 6.0 * (fa + 4 * fm + fb)                 # Simpson: exact for quadratics
            flux_p1 = L / 2.0 * (U[va] @ n + U[vb] @ n)
            beta[key] = (flux - flux_p1) / (2.0 * L / 3.0)      # unit bubble carries flux (2/3)|e|
            wv[key] = _coarse_field(cv, mid, sh)[1] @ n
        # divergence-preserving reset (reading A4)
        for (tid, verts, edges) in ftris:
            atc = [v for v in verts if v[0] % 2 == 0 and v[1] % 2 == 0]
            if len(atc) != 1:
                continue                                        # middle child
            P, g, area = _tri_geom([np.array(v) * hf for v in verts])
            cen = P.mean(axis=0)
            cvtx = verts.index(atc[0])
            flux_p1 = area * sum(U[verts[a]] @ g[a] for a in range(3))
            coef = {}
            for ek in edges:
                va, vb = fedges[ek]
                A = np.array(va) * hf; B = np.array(vb) * hf
                n = NORMAL[ek[0]]
                s = 1.0 if np.dot(0.5 * (A + B) - cen, n) > 0 else -1.0
                coef[ek] = s * 2.0 * np.linalg.norm(B - A) / 3.0
            estar = [ek for ek in edges if atc[0] not in fedges[ek]][0]
            rest = sum(coef[ek] * beta[ek] for ek in edges if ek != estar)
            beta[estar] = -(flux_p1 + rest) / coef[estar]
        col = {}
        for di in range(2):
            for dj in range(2):
                vals = [U[(di, dj)][0], U[(di, dj)][1],
                        beta[("H", di, dj)], beta[("V", di, dj)], beta[("D", di, dj)],
                        wv[("H", di, dj)], wv[("V", di, dj)], wv[("D", di, dj)]]
                # P0: copy of the parent coarse triangle (centroid test)
                for s in (0, 1):
                    verts = [v for (t, v, _) in ftris if t == (di, dj, s)][0]
                    cen = np.mean(np.array(verts, float) * hf, axis=0)
                    vals.append(_coarse_field(cv, cen, _which(cen))[2])
                col[(di, dj)] = vals
        cols.append(col)
    P = {}
    for di in range(2):
        for dj in range(2):
            for kf in range(10):
                ent = {}
                for c in range(nC):
                    v = cols[c][(di, dj)][kf]
                    if abs(v) > 1e-14:
                        ent[c] = snap(v)
                P[(di, dj, kf)] = ent
    return P


# ----------------------------------------------------------------------------- emit
def snap(v):
    """Closest p/q or (p/q) sqrt2 (q <= 96) within 1e-12 relative -- removes geometric round-off."""
    v = float(v)
    if abs(v) < 1e-14:
        return 0.0
    for base in (1.0, SQ2):
        for q in range(1, 97):
            p = round(v / base * q)
            if p != 0 and abs(p / q * base - v) <= 1e-12 * abs(v):
                return float(p / q if base == 1.0 else p * SQ2 / q)
    return v


def _f(v):
    return repr(snap(v))


def emit(path):
    E = [element(0), element(1)]
    rows = stencil()
    P = prolongation()
    out = []
    w = out.append
    w("// GENERATED by gen_tables.py -- do not edit.  Geometry of the RQ P1+bubble / RT0 / P0 Biot")
    w("// discretisation (PAPER.md:137-167, 308-317, 1333-1337) and the divergence-preserving")
    w("// prolongation (PAPER.md:477-566).  See gen_tables.py for the definitions.")
    w("#pragma once")
    w("")
    w("// ---- reference element integrals, h = 1 (shape 0 = LL, 1 = UR)")
    w("static const double REF_AEPS[2][9][9] = {")
    for s in range(2):
        w("  {" + ",\n   ".join("{" + ", ".join(_f(v) for v in r) + "}" for r in E[s]["Aeps"]) + "},")
    w("};")
    w("static const double REF_BU[2][9] = {" + ", ".join("{" + ", ".join(_f(v) for v in E[s]["Bu"]) + "}" for s in range(2)) + "};")
    w("static const double REF_MW1[2][3][3] = {" + ", ".join(
        "{" + ", ".join("{" + ", ".join(_f(v) for v in r) + "}" for r in E[s]["Mw1"]) + "}" for s in range(2)) + "};")
    w("static const double REF_BW[2][3] = {" + ", ".join("{" + ", ".join(_f(v) for v in E[s]["Bw"]) + "}" for s in range(2)) + "};")
    w("static const double REF_MP[2] = {" + ", ".join(_f(E[s]["Mp"]) for s in range(2)) + "};")
    # exact minus reduced quadrature of the lambda term: (div u - P_Q div u, div v - P_Q div v) =
    # Ddiv - Bu Bu^T / |T|; zero on the P1 rows (their divergence is constant), a 3 x 3 bubble block
    ex = []
    for s in range(2):
        X = E[s]["Ddiv"] - np.outer(E[s]["Bu"], E[s]["Bu"]) / E[s]["Mp"]
        assert np.abs(X[:6, :]).max() < 1e-13 and np.abs(X[:, :6]).max() < 1e-13
        ex.append(X[6:, 6:])
    w("// exact-integration lambda term minus its reduced quadrature on the bubbles (H, V, D), h-independent")
    w("static const double REF_EXDIV[2][3][3] = {" + ", ".join(
        "{" + ", ".join("{" + ", ".join(_f(v) for v in r) + "}" for r in ex[s]) + "}" for s in range(2)) + "};")
    w("// local DoF q (0..12) of shape s -> (dx, dy, plane) relative to the cell")
    w("static const int LOCAL_DOF[2][13][3] = {" + ", ".join(
        "{" + ", ".join("{%d,%d,%d}" % t for t in LOCAL[s]) + "}" for s in range(2)) + "};")
    w("")
    w("// ---- merged stencil of A^RQ without the M_w block: X(row, dx, dy, plane, coef_index)")
    cidx = 0
    contribs = []
    counts = []
    for k, r in enumerate(rows):
        items = []
        for (col, lst) in r["entries"]:
            items.append("X(%d,%d,%d,%d,%d)" % (k, col[0], col[1], col[2], cidx))
            for (s, q, q2) in lst:
                contribs.append((cidx, s, q, q2))
            cidx += 1
        counts.append(len(items))
        w("#define MG_STENCIL_ROW_%d(X) " % k + " ".join(items))
    w("#define MG_STENCIL_NCOEF %d" % cidx)
    # the same entries interleaved round-robin over the 10 rows (each row keeps its own summation
    # order): consecutive FMAs then belong to independent accumulator chains
    per_row = [[] for _ in range(10)]
    ci = 0
    for k, r in enumerate(rows):
        for (col, lst) in r["entries"]:
            per_row[k].append("X(%d,%d,%d,%d,%d)" % (k, col[0], col[1], col[2], ci))
            ci += 1
    il = []
    for e in range(max(len(x) for x in per_row)):
        for k in range(10):
            if e < len(per_row[k]):
                il.append(per_row[k][e])
    w("#define MG_STENCIL_INTERLEAVED(X) " + " ".join(il))
    # factored form.  Every merged coefficient is a linear combination of the material terms
    # (mu, lambda, alpha h, tau h, h^2 / M) with weights fixed by the reference integrals
    # (elem_entry in mg_setup.cpp).  Coefficients with a zero weight vector vanish for every
    # material (dropped); coefficients with equal weight vectors up to sign share one value cg[g].
    # Row k then reads sum_g (+-cg[g]) * (sum of +-x over the entries of group g): one FMA per
    # group and one add per further entry instead of one FMA (and coefficient load) per entry.
    def wvec(lst):
        v = np.zeros(5)
        for (sh, q, q2) in lst:
            a, b = block(q), block(q2)
            if (a, b) == ("u", "u"):
                v[0] += 2.0 * snap(E[sh]["Aeps"][q][q2])
                v[1] += 2.0 * snap(E[sh]["Bu"][q]) * snap(E[sh]["Bu"][q2])
            elif (a, b) == ("u", "p"):
                v[2] += snap(E[sh]["Bu"][q])
            elif (a, b) == ("p", "u"):
                v[2] += snap(E[sh]["Bu"][q2])
            elif (a, b) == ("w", "p"):
                v[3] += snap(E[sh]["Bw"][q - 9])
            elif (a, b) == ("p", "w"):
                v[3] += snap(E[sh]["Bw"][q2 - 9])
            elif (a, b) == ("p", "p"):
                v[4] -= snap(E[sh]["Mp"])
        v[np.abs(v) < 1e-12] = 0.0
        return v
    groups = []          # [weight vector (first nonzero > 0), representative coef index, its sign]
    fact_rows = [[] for _ in range(10)]   # per row: list of (g, [(dx, dy, pl, sign)])
    ci = 0
    for k, r in enumerate(rows):
        order = []
        terms = {}
        for (col, lst) in r["entries"]:
            v = wvec(lst)
            if np.any(v != 0.0):
                lead = v[np.nonzero(v)[0][0]]
                sg = 1 if lead > 0 else -1
                vn = v * sg
                g = next((gi for gi, (gv, _, _) in enumerate(groups) if np.allclose(gv, vn, rtol=1e-12, atol=0)), None)
                if g is None:
                    g = len(groups)
                    groups.append((vn, ci, sg))
                if g not in terms:
                    terms[g] = []
                    order.append(g)
                terms[g].append((col[0], col[1], col[2], sg))
            ci += 1
        fact_rows[k] = [(g, terms[g]) for g in order]
    w("// factored stencil: A(row, g, sign, expr) adds sign cg[g] * expr to row; XS(dx, dy, plane) is")
    w("// supplied by the user (rows interleaved round-robin: independent accumulator chains)")
    w("#define MG_STENCIL_NGROUP %d" % len(groups))
    w("// cg[g] = sign * coef[ci] for R(g, ci, sign)")
    w("#define MG_STENCIL_GROUP_REP(R) " + " ".join("R(%d,%d,%d)" % (g, rep, sg) for g, (_, rep, sg) in enumerate(groups)))
    fitems = [[] for _ in range(10)]
    for k in range(10):
        for g, lst in fact_rows[k]:
            if all(t[3] < 0 for t in lst):
                msign, lst2 = "-", [(a, b, c, -d) for (a, b, c, d) in lst]
            else:
                msign, lst2 = "+", sorted(lst, key=lambda t: -t[3])   # a positive entry first
            expr = ""
            for j, (dx, dy, pl, sg) in enumerate(lst2):
                op = "" if j == 0 else (" + " if sg > 0 else " - ")
                expr += op + "XS(%d,%d,%d)" % (dx, dy, pl)
            fitems[k].append("A(%d,%d,%s,(%s))" % (k, g, msign, expr))
    fil = []
    for e in range(max(len(x) for x in fitems)):
        for k in range(10):
            if e < len(fitems[k]):
                fil.append(fitems[k][e])
    w("#define MG_STENCIL_FACT(A) " + " ".join(fil))
    w("// coefficient contributions: Y(coef_index, shape, q, q') -- coef = sum of element entries")
    w("#define MG_STENCIL_CONTRIB(Y) " + " ".join("Y(%d,%d,%d,%d)" % c for c in contribs))
    w("// M_w part of the RT0 rows, per triangle: W(row, cell_dx, cell_dy, shape, dx, dy, plane, e, e')")
    for k in (5, 6, 7):
        w("#define MG_STENCIL_WW_%d(W) " % k + " ".join("W(%d,%d,%d,%d,%d,%d,%d,%d,%d)" % ((k,) + t) for t in rows[k]["ww"]))
    w("// triangles incident to the DoF of plane k owned by index (0,0): I(k, cell_dx, cell_dy, shape, q)")
    for k in range(10):
        items = []
        for cx in (-1, 0):
            for cy in (-1, 0):
                for s in (0, 1):
                    for q, (dx, dy, pl) in enumerate(LOCAL[s]):
                        if (cx + dx, cy + dy, pl) == (0, 0, k):
                            items.append("I(%d,%d,%d,%d,%d)" % (k, cx, cy, s, q))
        w("#define MG_INCIDENT_%d(I) " % k + " ".join(items))
    w("// local DoFs of the triangle of shape s in cell (0,0): L(s, q, dx, dy, plane)")
    for s in (0, 1):
        w("#define MG_LOCAL_%d(L) " % s + " ".join("L(%d,%d,%d,%d,%d)" % ((s, q) + LOCAL[s][q]) for q in range(13)))
    w("")
    w("// ---- prolongation on coarse cell (I,J): fine index (2I+di, 2J+dj), fine plane kf")
    w("// coarse local DoFs: C(n) = (dI, dJ, plane)")
    w("static const int COARSE_DOF[%d][3] = {" % len(COARSE_DOFS) + ", ".join("{%d,%d,%d}" % t for t in COARSE_DOFS) + "};")
    for (di, dj, kf), ent in sorted(P.items()):
        items = " ".join("Q(%d,%d,%d,%s)" % (COARSE_DOFS[c] + (_f(v),)) for c, v in sorted(ent.items()))
        w("#define MG_PROLONG_%d_%d_%d(Q) %s" % (di, dj, kf, items))
    # restriction entries of planes 0-4 and 5-9, interleaved round-robin over the planes:
    # U(kc, cell_dI, cell_dJ, di, dj, kf, weight)
    # LO / HI: planes 0-4 / 5-9; G0-G3: four groups of ~23 entries each (one warp per group)
    for name, planes in (("LO", range(0, 5)), ("HI", range(5, 10)), ("G0", (0, 8)), ("G1", (1, 9)),
                         ("G2", (2, 3, 4)), ("G3", (5, 6, 7))):
        lists = []
        for kc in planes:
            lst = []
            for (di, dj, kf), ent in sorted(P.items()):
                for c, v in sorted(ent.items()):
                    dI, dJ, pc = COARSE_DOFS[c]
                    if pc == kc:
                        lst.append("U(%d,%d,%d,%d,%d,%d,%s)" % (kc, dI, dJ, di, dj, kf, _f(v)))
            lists.append(lst)
        il = []
        for e in range(max(len(x) for x in lists)):
            for lst in lists:
                if e < len(lst):
                    il.append(lst[e])
        w("#define MG_RESTRICT_IL_%s(U) " % name + " ".join(il))
    w("// restriction R = P^T for coarse plane kc: T(cell_dI, cell_dJ, di, dj, kf, weight); the fine index is")
    w("// (2(I-cell_dI)+di, 2(J-cell_dJ)+dj) for coarse index (I, J)")
    for kc in range(10):
        items = []
        for (di, dj, kf), ent in sorted(P.items()):
            for c, v in sorted(ent.items()):
                dI, dJ, pc = COARSE_DOFS[c]
                if pc == kc:
                    items.append("T(%d,%d,%d,%d,%d,%s)" % (dI, dJ, di, dj, kf, _f(v)))
        w("#define MG_RESTRICT_%d(T) " % kc + " ".join(items))
    w("")
    with open(path, "w") as f:
        f.write("\n".join(out) + "\n")
    return dict(stencil_counts=counts, ncoef=cidx)


if __name__ == "__main__":
    here = os.path.dirname(os.path.abspath(__file__))
    info = emit(os.path.join(here, "mg_tables.h"))
    print(info)

"""Grid-transfer operators (ORACLE -- test infrastructure only).

PAPER.md:477-484 (eq. block_interp): P = diag(P_u, P_w, P_p), R = P^T, coarse
operators by rediscretisation.  P_w and P_p are the canonical finite-element
interpolations for RT0 and P0.  P_u is the divergence-preserving interpolation
of PAPER.md:510-566 built column-wise exactly as the paper describes:

  1. c_i = \\hat P_u e_i, the standard finite-element interpolation of the coarse
     basis function (fine P1 DoF = point value; fine bubble DoF chosen so that
     the fine interpolant has the same flux as the coarse function across the
     fine edge -- the DoF is a flux);
  2. the entries of c_i on the three interior-edge bubbles of every coarse
     triangle (the edges of its middle fine triangle, Fig. fig:div_free_interp)
     are replaced by the values that make the flux of c_i out of the adjacent
     corner fine triangle vanish (eq. divfreefine, formula PAPER.md:532-537).

Reading A4: the paper's formula is written for flux-normalised
bubble DoFs with a 1/|dt| factor; with the normal-trace normalisation fixed by
Appendix A (reading A1) the same condition "zero outward flux of each corner
triangle t" reads

  0 = |t| sum_{v in t} u_v . grad(lambda_v|_t) + sum_{e in dt} s_{t,e} (2|e|/3) beta_e,

solved for the bubble beta_{e*} of the interior edge e* of t.
"""
from __future__ import annotations

import copy

import numpy as np
import scipy.sparse as sp

from .mesh import Mesh, NORMALS


def _parent(fine: Mesh, coarse: Mesh, t):
    """Coarse triangle containing fine triangle t (by its centroid)."""
    P = fine.tri_coords(t)
    c = P.mean(axis=1)
    Hc = coarse.h
    I = np.floor(c[:, 0] / Hc + 1e-12).astype(np.int64)
    J = np.floor(c[:, 1] / Hc + 1e-12).astype(np.int64)
    lx = c[:, 0] / Hc - I
    ly = c[:, 1] / Hc - J
    shape = np.where(lx + ly < 1.0, 0, 1)
    n = coarse.n
    return shape * n * n + J * n + I          # coarse triangle id (shape-major as in Mesh)


def _barycentric(coarse: Mesh, T, X):
    """Barycentric coordinates (N, 3) of points X (N, 2) in coarse triangles T (N,)."""
    P = coarse.tri_coords(T)                                   # (N, 3, 2)
    M = np.stack([P[:, 1] - P[:, 0], P[:, 2] - P[:, 0]], axis=2)  # columns = edge vectors
    l12 = np.linalg.solve(M, (X - P[:, 0])[..., None])[..., 0]
    return np.concatenate([1.0 - l12.sum(axis=1, keepdims=True), l12], axis=1)


def _coarse_u(coarse: Mesh, T, X):
    """Values (N, 9, 2) of the 9 local u basis functions of coarse triangles T at X,
    and their slots (N, 9): P1 lambda_a e_c, bubble 4 lambda_a lambda_b n_e."""
    lam = _barycentric(coarse, T, X)
    N = len(T)
    vals = np.zeros((N, 9, 2))
    for a in range(3):
        vals[:, 2 * a, 0] = lam[:, a]
        vals[:, 2 * a + 1, 1] = lam[:, a]
    r = np.arange(N)
    for e in range(3):
        a, b = coarse.tri_eloc[T, e, 0], coarse.tri_eloc[T, e, 1]
        vals[:, 6 + e, :] = (4.0 * lam[r, a] * lam[r, b])[:, None] * NORMALS[coarse.tri_ek[T, e]]
    return vals, coarse.local_slots()[T][:, 0:9]


def _coarse_w(coarse: Mesh, T, X):
    """Values (N, 3, 2) of the local RT0 functions of coarse triangles T at X, slots (N, 3)."""
    P = coarse.tri_coords(T)
    cen = P.mean(axis=1)
    e1, e2 = P[:, 1] - P[:, 0], P[:, 2] - P[:, 0]
    area = 0.5 * np.abs(e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0])
    r = np.arange(len(T))
    vals = np.zeros((len(T), 3, 2))
    for e in range(3):
        a, b, o = (coarse.tri_eloc[T, e, q] for q in range(3))
        nrm = NORMALS[coarse.tri_ek[T, e]]
        s = np.where(np.einsum("nd,nd->n", 0.5 * (P[r, a] + P[r, b]) - cen, nrm) > 0, 1.0, -1.0)
        elen = np.linalg.norm(P[r, b] - P[r, a], axis=1)
        vals[:, e, :] = (s * elen / (2.0 * area))[:, None] * (X - P[r, o])
    return vals, coarse.local_slots()[T][:, 9:12]


def _first(keys):
    """Indices of the first occurrence of every distinct key."""
    _, idx = np.unique(keys, return_index=True)
    return idx


def build_P(fine: Mesh, coarse: Mesh):
    """Full-slot prolongation matrices P_u (with divergence fix), P_w, P_p and the
    standard interpolation Phat_u.  Shapes (fine.nslots, coarse.nslots).

    Every weight is invariant under a uniform scaling of the mesh (point values, normal
    traces and the zero-flux condition of PAPER.md:532-537 are all homogeneous), so the
    geometry is evaluated on integer grid coordinates (fine spacing 1, coarse spacing 2),
    which are exact in floating point: the weights then carry only the round-off of the
    formulas, not an O(n u) error from the coordinates i/n."""
    assert fine.n == 2 * coarse.n
    fine, coarse = copy.copy(fine), copy.copy(coarse)
    fine.h, coarse.h = 1.0, 2.0
    Nf, Nc = fine.nslots, coarse.nslots
    h = fine.h
    nt = fine.ntri
    tt = np.arange(nt)
    parent = _parent(fine, coarse, tt)
    fl = fine.local_slots()
    Pf = fine.tri_coords(tt)                                   # (T, 3, 2)
    coo = {"u": ([], [], []), "w": ([], [], []), "p": ([], [], [])}

    def add(key, r, c, v):
        m = v != 0.0
        coo[key][0].append(r[m]); coo[key][1].append(c[m]); coo[key][2].append(v[m])

    # P0: copy the parent value
    add("p", fine.tri_pslot, coarse.tri_pslot[parent], np.ones(nt))
    # P1 at fine vertices: point values of the coarse function (continuous, any containing triangle)
    for c in range(2):
        rows = np.concatenate([fl[:, 2 * a + c] for a in range(3)])
        first = _first(rows)                                   # one (triangle, corner) per fine vertex
        tri = np.concatenate([tt] * 3)[first]
        loc = np.repeat(np.arange(3), nt)[first]
        vals, sl = _coarse_u(coarse, parent[tri], Pf[tri, loc])
        for q in range(9):
            add("u", rows[first], sl[:, q], vals[:, q, c])
    # edges: bubble by flux-preserving interpolation, RT0 by normal trace
    for e in range(3):
        rows = fl[:, 6 + e]
        first = _first(rows)
        t = first
        T = parent[t]
        a, b = fine.tri_eloc[t, e, 0], fine.tri_eloc[t, e, 1]
        Pa, Pb = Pf[t, a], Pf[t, b]
        Pm = 0.5 * (Pa + Pb)
        L = np.linalg.norm(Pb - Pa, axis=1)
        nrm = NORMALS[fine.tri_ek[t, e]]
        fa, sl = _coarse_u(coarse, T, Pa)
        fm, _ = _coarse_u(coarse, T, Pm)
        fb, _ = _coarse_u(coarse, T, Pb)
        na = np.einsum("nqd,nd->nq", fa, nrm)
        nm = np.einsum("nqd,nd->nq", fm, nrm)
        nb = np.einsum("nqd,nd->nq", fb, nrm)
        flux = (L / 6.0)[:, None] * (na + 4.0 * nm + nb)        # Simpson: exact for quadratics
        flux_p1 = (L / 2.0)[:, None] * (na + nb)                # flux of the fine P1 interpolant
        beta = (flux - flux_p1) / (2.0 * L / 3.0)[:, None]      # bubble flux = (2/3)|e| per unit DoF
        beta[np.abs(beta) < 1e-15] = 0.0
        for q in range(9):
            add("u", rows[first], sl[:, q], beta[:, q])
        rows_w = fl[:, 9 + e]
        wv, slw = _coarse_w(coarse, T, Pm)
        tr = np.einsum("nqd,nd->nq", wv, nrm)
        tr[np.abs(tr) < 1e-15] = 0.0
        for q in range(3):
            add("w", rows_w[first], slw[:, q], tr[:, q])
    mats = {}
    for key in coo:
        r, c, v = (np.concatenate(z) for z in coo[key])
        mats[key] = sp.csr_matrix((v, (r, c)), shape=(Nf, Nc))
    Phat_u, P_w, P_p = mats["u"], mats["w"], mats["p"]

    # ---- divergence-preserving fix -----------------------------
    # A corner child t of a coarse triangle has exactly one vertex at a coarse vertex;
    # its opposite edge e* is the edge shared with the middle child.  The middle
    # child has no coarse vertex.
    at_coarse_vertex = (fine.tri_vi % 2 == 0) & (fine.tri_vj % 2 == 0)     # (T, 3)
    ncv = at_coarse_vertex.sum(axis=1)
    assert set(np.unique(ncv)) <= {0, 1}
    corner = np.nonzero(ncv == 1)[0]
    assert corner.size == 3 * coarse.ntri and (ncv == 0).sum() == coarse.ntri
    cv = np.argmax(at_coarse_vertex[corner], axis=1)           # local vertex at the coarse vertex
    Qr, Qc, Qv = [], [], []
    g_all = np.empty((corner.size, 3, 2))
    P = Pf[corner]
    M = np.stack([P[:, 1] - P[:, 0], P[:, 2] - P[:, 0]], axis=2)
    Minv = np.linalg.inv(M)                                    # rows = grad lambda_1, grad lambda_2
    g_all[:, 1] = Minv[:, 0, :]
    g_all[:, 2] = Minv[:, 1, :]
    g_all[:, 0] = -(g_all[:, 1] + g_all[:, 2])
    area = 0.5 * np.abs(np.linalg.det(M))
    cen = P.mean(axis=1)
    r = np.arange(corner.size)
    coef = np.empty((corner.size, 3))
    for e in range(3):
        a, b = fine.tri_eloc[corner, e, 0], fine.tri_eloc[corner, e, 1]
        nrm = NORMALS[fine.tri_ek[corner, e]]
        s = np.where(np.einsum("nd,nd->n", 0.5 * (P[r, a] + P[r, b]) - cen, nrm) > 0, 1.0, -1.0)
        L = np.linalg.norm(P[r, b] - P[r, a], axis=1)
        coef[:, e] = s * 2.0 * L / 3.0                          # outward flux of a unit bubble
    # local edge opposite the coarse vertex
    estar = np.array([[e for e in range(3) if fine.tri_eloc[t, e, 2] == cv[k]][0] for k, t in enumerate(corner)])
    fls = fl[corner]
    bstar = fls[r, 6 + estar]
    cstar = coef[r, estar]
    for a in range(3):
        for c in range(2):
            Qr.append(bstar); Qc.append(fls[:, 2 * a + c]); Qv.append(-(area * g_all[:, a, c]) / cstar)
    for e in range(3):
        m = estar != e
        Qr.append(bstar[m]); Qc.append(fls[m, 6 + e]); Qv.append(-coef[m, e] / cstar[m])
    assert np.unique(bstar).size == bstar.size
    keep = np.ones(Nf)
    keep[bstar] = 0.0
    Q = sp.diags(keep) + sp.csr_matrix((np.concatenate(Qv), (np.concatenate(Qr), np.concatenate(Qc))),
                                       shape=(Nf, Nf))
    P_u = (Q @ Phat_u).tocsr()
    P_u.eliminate_zeros()
    return dict(P_u=P_u, Phat_u=Phat_u, P_w=P_w, P_p=P_p, replaced=np.sort(bstar))


class Transfer:
    """Prolongation P and restriction R = P^T between active DoFs of two levels."""

    def __init__(self, fine: Mesh, coarse: Mesh):
        mats = build_P(fine, coarse)
        self.mats = mats
        P = (mats["P_u"] + mats["P_w"] + mats["P_p"]).tocsr()
        self.P_full = P
        self.P = P[fine.act_idx][:, coarse.act_idx].tocsr()
        self.R = self.P.T.tocsr()
        self.fine, self.coarse = fine, coarse

    def prolong(self, e_c):
        return self.P @ e_c

    def restrict(self, r_f):
        return self.R @ r_f

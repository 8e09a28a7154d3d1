"""Element integrals and the assembled reduced-quadrature operator (ORACLE -- test infrastructure only).

Follows PAPER.md:113-167 (discrete variational form, eq. block_form and the
bilinear forms listed under it), PAPER.md:200-317 (reduced quadrature,
eq. block_form_rq) and PAPER.md:1333-1337 (A_u^RQ = 2 mu A_eps + lambda
B_u^T M_p^{-1} B_u):

    a^RQ(u, v)  = 2 mu (eps(u), eps(v)) + lambda (P_Q div u, P_Q div v)    -> A_u^RQ
    -(div u, q)                                                          -> B_u
    -(div w, q)                                                          -> B_w
    (K^{-1} mu_f w, r)                                                   -> M_w
    (p, q)                                                               -> M_p

    A^RQ = [[A_u^RQ, 0, alpha B_u^T], [0, tau M_w, tau B_w^T], [alpha B_u, tau B_w, -(1/M) M_p]]

Basis functions (reading A1 of DESIGN.md; the paper's printed symbols in
Appendix A fix this normalisation):
  P1       lambda_a e_x, lambda_a e_y
  bubble   phi_e = 4 lambda_a lambda_b n_e           (normal trace 1 at the edge midpoint)
  RT0      psi_e = s_{T,e} |e| / (2|T|) (x - x_opp)   (normal trace 1 along e; s=+1 if n_e points out of T)
  P0       indicator of T
Integrals use the edge-midpoint rule (exact for quadratics; every integrand
here is at most quadratic on a triangle).

Since P_Q is the L2 projection onto piecewise constants,
(P_Q div u, P_Q div v) = sum_T |T|^{-1} (div u, 1_T)(div v, 1_T), i.e.
lambda B_u^T M_p^{-1} B_u exactly.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .mesh import Mesh, NORMALS

# barycentric coordinates of the three edge midpoints
_QP = np.array([[0.5, 0.5, 0.0], [0.0, 0.5, 0.5], [0.5, 0.0, 0.5]])


def p1_geometry(P):
    """P: (3, 2) vertex coordinates -> (grad lambda (3, 2), area)."""
    M = np.array([[P[1, 0] - P[0, 0], P[2, 0] - P[0, 0]],
                  [P[1, 1] - P[0, 1], P[2, 1] - P[0, 1]]])
    Minv = np.linalg.inv(M)
    g = np.empty((3, 2))
    g[1] = Minv[0]
    g[2] = Minv[1]
    g[0] = -(g[1] + g[2])
    return g, 0.5 * abs(np.linalg.det(M))


def element_matrices(P, eloc, ekind):
    """Element integrals on one triangle.

    P      (3, 2) vertex coordinates
    eloc   (3, 3) local edge -> (endpoint a, endpoint b, opposite vertex)
    ekind  (3,)   edge kinds (selects the global normal)
    Returns dict with
      Aeps (9, 9)  (eps(phi_i), eps(phi_j)) over local u DoFs [P1 (a,c) -> 2a+c, bubbles 6..8]
      Bu   (9,)    -(div phi_i, 1_T)
      Mw1  (3, 3)  (psi_e, psi_e')    (multiply by mu_f / K_T)
      Bw   (3,)    -(div psi_e, 1_T)
      Mp   float   |T|
      Ddiv (9, 9)  (div phi_i, div phi_j), integrated exactly (exact-integration lambda term,
                   eq. block_form; div of P1 + bubble is linear on T)
    """
    g, area = p1_geometry(P)
    nrm = NORMALS[ekind]
    elen = np.array([np.linalg.norm(P[eloc[e, 1]] - P[eloc[e, 0]]) for e in range(3)])
    centroid = P.mean(axis=0)
    s = np.array([1.0 if np.dot(0.5 * (P[eloc[e, 0]] + P[eloc[e, 1]]) - centroid, nrm[e]) > 0 else -1.0
                  for e in range(3)])
    Aeps = np.zeros((9, 9))
    Ddiv = np.zeros((9, 9))
    Bu = np.zeros(9)
    Mw1 = np.zeros((3, 3))
    Bw = np.zeros(3)
    for q in range(3):
        L = _QP[q]
        x = L @ P
        w = area / 3.0
        # gradients G[c, d] = d phi_c / d x_d of the 9 u basis functions
        G = np.zeros((9, 2, 2))
        for a in range(3):
            G[2 * a, 0, :] = g[a]
            G[2 * a + 1, 1, :] = g[a]
        for e in range(3):
            a, b = eloc[e, 0], eloc[e, 1]
            gpsi = 4.0 * (L[a] * g[b] + L[b] * g[a])
            G[6 + e] = np.outer(nrm[e], gpsi)
        eps = 0.5 * (G + G.transpose(0, 2, 1))
        Aeps += w * np.einsum("icd,jcd->ij", eps, eps)
        dv = np.trace(G, axis1=1, axis2=2)
        Ddiv += w * np.outer(dv, dv)
        Bu += -w * dv
        # RT0 values at x
        psi = np.array([s[e] * elen[e] / (2.0 * area) * (x - P[eloc[e, 2]]) for e in range(3)])
        Mw1 += w * psi @ psi.T
        divpsi = np.array([s[e] * elen[e] / (2.0 * area) * 2.0 for e in range(3)])
        Bw += -w * divpsi
    return dict(Aeps=Aeps, Ddiv=Ddiv, Bu=Bu, Mw1=Mw1, Bw=Bw, Mp=area, sign=s, elen=elen, grad=g, area=area)


class Operator:
    """Assembled blocks and A^RQ on one mesh level (eq. block_form_rq).

    Kinv: None for scalar K (then K_scalar is used) or a (2, n, n) array of
    per-triangle 1/K ([shape, j, i]).  Matrices are assembled on the full slot
    space (10 (n+1)^2) and then restricted to the active DoFs (symmetric
    elimination of the Dirichlet rows and columns).

    quadrature: "rq" (default) -- lambda (P_Q div u, P_Q div v) = lambda B_u^T M_p^{-1} B_u, the
    reduced-quadrature operator A^RQ of eq. block_form_rq; "exact" -- lambda (div u, div v)
    integrated exactly, the operator A of eq. block_form, whose solver
    incompatibility tab:naive shows.  Only A_u differs.
    """

    def __init__(self, mesh: Mesh, lam, mu, tau, alpha, inv_M, mu_f=1.0, K=1.0, Kinv_field=None,
                 quadrature="rq"):
        if quadrature not in ("rq", "exact"):
            raise ValueError("quadrature must be 'rq' or 'exact'")
        self.quadrature = quadrature
        self.mesh = mesh
        self.lam, self.mu, self.tau, self.alpha, self.inv_M, self.mu_f = lam, mu, tau, alpha, inv_M, mu_f
        T = mesh.ntri
        ls = mesh.local_slots()
        N = mesh.nslots
        if Kinv_field is None:
            kinv_t = np.full(T, 1.0 / K)
        else:
            kinv_t = Kinv_field[mesh.tri_shape, mesh.tri_cj, mesh.tri_ci]
        self.kinv_t = kinv_t
        rows = {k: [] for k in ("Aeps", "Ddiv", "Bu", "Mw", "Bw", "Mp")}
        cols = {k: [] for k in rows}
        vals = {k: [] for k in rows}
        self.elem = {}
        for shape in (0, 1):
            t = np.nonzero(mesh.tri_shape == shape)[0]
            t0 = t[0]
            E = element_matrices(mesh.tri_coords([t0])[0], mesh.tri_eloc[t0], mesh.tri_ek[t0])
            # translation invariance: every triangle of a shape has the same element integrals
            for tt in t[:: max(1, len(t) // 7)]:
                E2 = element_matrices(mesh.tri_coords([tt])[0], mesh.tri_eloc[tt], mesh.tri_ek[tt])
                assert np.allclose(E2["Aeps"], E["Aeps"], rtol=0, atol=1e-12)
            self.elem[shape] = E
            us = ls[t][:, 0:9]
            ws = ls[t][:, 9:12]
            ps = ls[t][:, 12]
            nt = len(t)
            rows["Aeps"].append(np.repeat(us, 9, axis=1).ravel())
            cols["Aeps"].append(np.tile(us, (1, 9)).ravel())
            vals["Aeps"].append(np.tile(E["Aeps"].ravel(), nt))
            if quadrature == "exact":   # assembled only for the exact-integration operator (memory)
                rows["Ddiv"].append(np.repeat(us, 9, axis=1).ravel())
                cols["Ddiv"].append(np.tile(us, (1, 9)).ravel())
                vals["Ddiv"].append(np.tile(E["Ddiv"].ravel(), nt))
            rows["Bu"].append(np.repeat(ps, 9))
            cols["Bu"].append(us.ravel())
            vals["Bu"].append(np.tile(E["Bu"], nt))
            rows["Mw"].append(np.repeat(ws, 3, axis=1).ravel())
            cols["Mw"].append(np.tile(ws, (1, 3)).ravel())
            vals["Mw"].append((mu_f * kinv_t[t][:, None] * E["Mw1"].ravel()[None, :]).ravel())
            rows["Bw"].append(np.repeat(ps, 3))
            cols["Bw"].append(ws.ravel())
            vals["Bw"].append(np.tile(E["Bw"], nt))
            rows["Mp"].append(ps)
            cols["Mp"].append(ps)
            vals["Mp"].append(np.full(nt, E["Mp"]))
        blk = {}
        for k in [k for k in rows if rows[k]]:
            blk[k] = sp.csr_matrix((np.concatenate(vals[k]), (np.concatenate(rows[k]), np.concatenate(cols[k]))),
                                   shape=(N, N))
        self.full = blk
        # M_p^{-1} on the P0 slots
        mpd = blk["Mp"].diagonal()
        mpinv = np.zeros(N)
        mpinv[mpd > 0] = 1.0 / mpd[mpd > 0]
        if quadrature == "rq":
            Au = 2.0 * mu * blk["Aeps"] + lam * (blk["Bu"].T @ sp.diags(mpinv) @ blk["Bu"])
        else:
            Au = 2.0 * mu * blk["Aeps"] + lam * blk["Ddiv"]
        A = (Au + alpha * (blk["Bu"].T + blk["Bu"]) + tau * blk["Mw"] + tau * (blk["Bw"].T + blk["Bw"])
             - inv_M * blk["Mp"])
        act = mesh.act_idx
        self.A_full = A.tocsr()
        self.A = self.A_full[act][:, act].tocsr()
        self.A.sort_indices()
        self.Au_full = Au.tocsr()
        # restricted blocks (rows / cols on the active slots of each field)
        kind = mesh.slot_kind(act)
        self.iu = np.nonzero(kind <= 4)[0]          # positions in the active vector
        self.iw = np.nonzero((kind >= 5) & (kind <= 7))[0]
        self.ip = np.nonzero(kind >= 8)[0]
        su, sw, spp = act[self.iu], act[self.iw], act[self.ip]
        self.Au = Au.tocsr()[su][:, su].tocsr()
        self.Bu = blk["Bu"][spp][:, su].tocsr()
        self.Mw = blk["Mw"][sw][:, sw].tocsr()
        self.Bw = blk["Bw"][spp][:, sw].tocsr()
        self.Mp = blk["Mp"][spp][:, spp].tocsr()
        self.n = mesh.n

    def apply(self, x):
        return self.A @ x

    def residual(self, x, b):
        """r = b - A^RQ x on the active DoFs."""
        return b - self.A @ x

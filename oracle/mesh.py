"""Structured triangular mesh and DoF slots (ORACLE -- test infrastructure only).

Mesh (Appendix A): unit square, n x n square cells of side
h = 1/n, each cut by the diagonal from top-left to bottom-right.  Cell (i, j)
holds the lower-left triangle LL = [(i,j), (i+1,j), (i,j+1)] and the
upper-right triangle UR = [(i+1,j), (i+1,j+1), (i,j+1)].

DoFs (Fig. fig:DoF_structure2 PAPER.md:757-799): P1 vector
displacement at vertices, one face bubble per edge, one RT0 per edge, one P0
per triangle.  The slot of DoF kind k at index (i, j) is
``(k * (n+1) + j) * (n+1) + i`` (10 kinds, see ``mg_inputs``).

Edges: H(i,j) = (i,j)-(i+1,j) normal +y; V(i,j) = (i,j)-(i,j+1) normal +x;
D(i,j) = (i+1,j)-(i,j+1) normal (1,1)/sqrt(2)  (reading A2 of DESIGN.md).

Boundary conditions (PAPER.md:936-945 and BASELINE configs): u = 0 and
w.n = 0 on the whole boundary.  A DoF is eliminated when it sits on the
boundary: P1 at a boundary vertex, bubble / RT0 on an edge that belongs to a
single triangle.  The active set is derived here from mesh topology (edge
triangle counts), independently of ``mg_inputs.active_mask``.
"""
from __future__ import annotations

import numpy as np

H, V, D = 0, 1, 2          # edge kinds
LL, UR = 0, 1              # triangle shapes
SQ2 = np.sqrt(2.0)
NORMALS = np.array([[0.0, 1.0], [1.0, 0.0], [1.0 / SQ2, 1.0 / SQ2]])


class Mesh:
    def __init__(self, n: int):
        if n < 1:
            raise ValueError("n >= 1 required")
        self.n = n
        self.h = 1.0 / n
        self.N1 = n + 1
        self.nslots = 10 * self.N1 * self.N1
        self._build_triangles()
        self._build_active()

    # ---- slots -------------------------------------------------------------
    def slot(self, k, i, j):
        return (np.asarray(k) * self.N1 + np.asarray(j)) * self.N1 + np.asarray(i)

    def vert_xy(self, i, j):
        return np.stack([np.asarray(i, float) * self.h, np.asarray(j, float) * self.h], axis=-1)

    def edge_endpoints(self, kind, i, j):
        """Endpoint vertex indices ((ia, ja), (ib, jb)) of edges (vectorised)."""
        kind = np.asarray(kind); i = np.asarray(i); j = np.asarray(j)
        ia = np.where(kind == D, i + 1, i)
        ja = j.copy() if isinstance(j, np.ndarray) else np.asarray(j)
        ib = np.where(kind == H, i + 1, i)
        jb = np.where(kind == H, j, j + 1)
        return (ia, ja), (ib, jb)

    # ---- triangles ---------------------------------------------------------
    def _build_triangles(self):
        n = self.n
        jj, ii = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        ci = np.concatenate([ii.ravel(), ii.ravel()])
        cj = np.concatenate([jj.ravel(), jj.ravel()])
        shape = np.concatenate([np.full(n * n, LL), np.full(n * n, UR)])
        self.tri_shape, self.tri_ci, self.tri_cj = shape, ci, cj
        self.ntri = 2 * n * n
        # vertices (T, 3, 2) as integer (i, j)
        vi = np.empty((self.ntri, 3), dtype=np.int64)
        vj = np.empty((self.ntri, 3), dtype=np.int64)
        isLL = shape == LL
        vi[isLL] = np.stack([ci, ci + 1, ci], 1)[isLL]
        vj[isLL] = np.stack([cj, cj, cj + 1], 1)[isLL]
        vi[~isLL] = np.stack([ci + 1, ci + 1, ci], 1)[~isLL]
        vj[~isLL] = np.stack([cj, cj + 1, cj + 1], 1)[~isLL]
        self.tri_vi, self.tri_vj = vi, vj
        # local edges: (kind, i, j) and local endpoint / opposite vertex numbers
        ek = np.empty((self.ntri, 3), dtype=np.int64)
        ei = np.empty((self.ntri, 3), dtype=np.int64)
        ej = np.empty((self.ntri, 3), dtype=np.int64)
        ek[:] = [H, V, D]
        ei[isLL] = np.stack([ci, ci, ci], 1)[isLL]
        ej[isLL] = np.stack([cj, cj, cj], 1)[isLL]
        ei[~isLL] = np.stack([ci, ci + 1, ci], 1)[~isLL]
        ej[~isLL] = np.stack([cj + 1, cj, cj], 1)[~isLL]
        self.tri_ek, self.tri_ei, self.tri_ej = ek, ei, ej
        # local endpoint numbering found geometrically (edge endpoints among triangle vertices)
        loc = np.empty((self.ntri, 3, 3), dtype=np.int64)   # [t, e] -> (a, b, opposite)
        (ia, ja), (ib, jb) = self.edge_endpoints(ek, ei, ej)
        for e in range(3):
            a = np.argmax((vi == ia[:, e:e + 1]) & (vj == ja[:, e:e + 1]), axis=1)
            b = np.argmax((vi == ib[:, e:e + 1]) & (vj == jb[:, e:e + 1]), axis=1)
            assert np.all((vi[np.arange(self.ntri), a] == ia[:, e]) & (vj[np.arange(self.ntri), a] == ja[:, e]))
            assert np.all((vi[np.arange(self.ntri), b] == ib[:, e]) & (vj[np.arange(self.ntri), b] == jb[:, e]))
            loc[:, e, 0] = a
            loc[:, e, 1] = b
            loc[:, e, 2] = 3 - a - b
        self.tri_eloc = loc
        self.tri_pslot = self.slot(8 + shape, ci, cj)

    def tri_coords(self, t):
        """(len(t), 3, 2) vertex coordinates."""
        return np.stack([self.tri_vi[t] * self.h, self.tri_vj[t] * self.h], axis=-1).astype(float)

    # ---- local DoF -> global slot map (13 local DoFs per triangle) ----------
    def local_slots(self):
        """(T, 13) slots: [u_x v0, u_y v0, u_x v1, u_y v1, u_x v2, u_y v2,
        bubble e0..e2, RT0 e0..e2, P0]."""
        T = self.ntri
        s = np.empty((T, 13), dtype=np.int64)
        for a in range(3):
            s[:, 2 * a] = self.slot(0, self.tri_vi[:, a], self.tri_vj[:, a])
            s[:, 2 * a + 1] = self.slot(1, self.tri_vi[:, a], self.tri_vj[:, a])
        for e in range(3):
            s[:, 6 + e] = self.slot(2 + self.tri_ek[:, e], self.tri_ei[:, e], self.tri_ej[:, e])
            s[:, 9 + e] = self.slot(5 + self.tri_ek[:, e], self.tri_ei[:, e], self.tri_ej[:, e])
        s[:, 12] = self.tri_pslot
        return s

    # ---- boundary conditions / active set ------------------------------------
    def _build_active(self):
        n = self.n
        exists = np.zeros(self.nslots, dtype=bool)
        ls = self.local_slots()
        exists[ls.ravel()] = True           # slots that are DoFs of some triangle
        # edge -> number of adjacent triangles (1 => boundary edge)
        cnt = np.zeros(self.nslots, dtype=np.int64)
        np.add.at(cnt, ls[:, 6:9].ravel(), 1)
        np.add.at(cnt, ls[:, 9:12].ravel(), 1)
        boundary = np.zeros(self.nslots, dtype=bool)
        boundary[ls[:, 6:12].ravel()] = cnt[ls[:, 6:12].ravel()] == 1
        vi, vj = self.tri_vi.ravel(), self.tri_vj.ravel()
        onb = (vi == 0) | (vi == n) | (vj == 0) | (vj == n)
        boundary[self.slot(0, vi[onb], vj[onb])] = True
        boundary[self.slot(1, vi[onb], vj[onb])] = True
        self.exists = exists
        self.active = exists & ~boundary
        self.act_idx = np.nonzero(self.active)[0]
        self.nact = self.act_idx.size
        self.pos = np.full(self.nslots, -1, dtype=np.int64)
        self.pos[self.act_idx] = np.arange(self.nact)

    def n_dofs_all(self) -> int:
        """All DoF slots before boundary elimination (tab:mgtime 'DoF' column)."""
        return int(self.exists.sum())

    # conversions between (10, n+1, n+1) arrays and active vectors
    def to_active(self, arr):
        return np.asarray(arr, dtype=float).reshape(-1)[self.act_idx]

    def from_active(self, vec):
        out = np.zeros(self.nslots)
        out[self.act_idx] = vec
        return out.reshape(10, self.N1, self.N1)

    def slot_kind(self, s):
        return np.asarray(s) // (self.N1 * self.N1)

    # ---- incidence -------------------------------------------------------------
    def vertex_incidence(self):
        """For every vertex (i, j): incident edges (as (kind,i,j)) and incident triangles.

        Returns dict vertex_id -> (edge list, triangle list); vertex_id = j*(n+1)+i.
        Derived by scanning triangles (a triangle is incident if the vertex is one
        of its corners; an edge is incident if the vertex is an endpoint)."""
        N1 = self.N1
        tris = [[] for _ in range(N1 * N1)]
        edges = [set() for _ in range(N1 * N1)]
        for t in range(self.ntri):
            for a in range(3):
                vid = self.tri_vj[t, a] * N1 + self.tri_vi[t, a]
                tris[vid].append(t)
                for e in range(3):
                    if a in (self.tri_eloc[t, e, 0], self.tri_eloc[t, e, 1]):
                        edges[vid].add((int(self.tri_ek[t, e]), int(self.tri_ei[t, e]), int(self.tri_ej[t, e])))
        return tris, [sorted(s) for s in edges]

"""Relaxation schemes (ORACLE -- test infrastructure only).

Additive Vanka (Appendix C):

    r = b - A x,    x <- x + omega sum_l V_l^T D_l (V_l A V_l^T)^{-1} V_l r

with one vertex patch per mesh vertex (Fig. fig:patches: right panel = 20-DoF
patch for the full system, left panel = 8-DoF displacement patch used inside
BSR), truncated to the active DoFs (reading A8), and D_l the natural weights:
"the reciprocal of the number of patches that the corresponding degree of
freedom appears in" -- counted here, not assumed.

Deflated patch solve (reading A9).  For every patch with m > 0 pressure DoFs,
v = (0, 1_m)/sqrt(m) is an exact eigenvector of K_l = V_l A V_l^T with
eigenvalue -gamma (B_l^T 1 = 0 patchwise, M_p diagonal).  The oracle solves

    K_l^{-1} r = (v^T r / (-gamma)) v + (K_l + sigma v v^T)^{-1} (r - v v^T r),

which is the same vector as the plain solve, written so that the tiny
eigenvalue gamma = h^2/(2M) is only ever divided into the scalar v^T r.  sigma
is the mean diagonal of the patch Schur complement B A_y^{-1} B^T.

Inexact Braess-Sarazin (PAPER.md:654-686 eqs. BSR_standard and bsr_p,
Appendix D-E):
    F = diag(A_{V,u}^RQ, tau D_w), A_{V,u}^{-1} = sum_l V_l^T D_l (A_u^RQ)_l^{-1} V_l (8-DoF patches)
    S = (1/M + alpha^2/(lambda + 2 mu/d)) M_p + tau B_w D_w^{-1} B_w^T,  d = 2
    g = B F^{-1} r_y - r_p;   n_J sweeps of weighted Jacobi on S dp = g from dp = 0
    dy = F^{-1} (r_y - B^T dp);   x <- x + omega (dy, dp)
with B = (alpha B_u, tau B_w).  The paper uses n_J = 1;
BASELINE config 2/4 use n_J = 3.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .mesh import Mesh
from .fem import Operator


def principal_submatrices(A, I, chunk=20000):
    """K[q] = A[I[q]][:, I[q]] (dense) for the stacked index sets I (P, m): V_l A V_l^T of every patch.
    Element lookups A[i, j] of the CSR matrix (scipy csr_sample_values), in chunks of patches; the
    values are the stored entries themselves, so this is the same matrix as slicing patch by patch."""
    P, m = I.shape
    out = np.empty((P, m, m))
    for s0 in range(0, P, chunk):
        J = I[s0:s0 + chunk]
        rows = np.repeat(J, m, axis=1).ravel()
        cols = np.tile(J, (1, m)).ravel()
        out[s0:s0 + chunk] = np.asarray(A[rows, cols]).reshape(-1, m, m)
    return out


def vertex_patches(mesh: Mesh, kind: str):
    """Patch DoF lists (positions in the active vector), one per vertex.

    kind 'full': P1 at the vertex, bubble + RT0 on incident edges, P0 of incident
    triangles (Fig. fig:patches right).  kind 'disp': P1 + bubbles (left panel);
    positions are then within the displacement block (op.iu ordering)."""
    tris, edges = mesh.vertex_incidence()
    N1 = mesh.N1
    patches = []
    for vid in range(N1 * N1):
        i, j = vid % N1, vid // N1
        slots = [mesh.slot(0, i, j), mesh.slot(1, i, j)]
        for (k, ei, ej) in edges[vid]:
            slots.append(mesh.slot(2 + k, ei, ej))
        if kind == "full":
            for (k, ei, ej) in edges[vid]:
                slots.append(mesh.slot(5 + k, ei, ej))
            for t in tris[vid]:
                slots.append(mesh.tri_pslot[t])
        pos = mesh.pos[np.array(slots, dtype=np.int64)]
        patches.append(pos[pos >= 0])
    return patches


class Vanka:
    """Additive Vanka with 20-DoF vertex patches on the full system."""

    def __init__(self, op: Operator, patches=None):
        mesh = op.mesh
        self.op = op
        A = op.A
        self.patches = vertex_patches(mesh, "full") if patches is None else patches
        N = A.shape[0]
        count = np.zeros(N)
        for p in self.patches:
            count[p] += 1
        assert np.all(count > 0), "patches must cover every DoF"
        self.weight = 1.0 / count                               # natural weights
        ispress = np.zeros(N, dtype=bool)
        ispress[op.ip] = True
        self.groups = {}
        for idx in self.patches:
            if idx.size == 0:
                continue
            self.groups.setdefault(idx.size, []).append(idx)
        self.data = []
        for m, plist in sorted(self.groups.items()):
            I = np.array(plist)                                 # (P, m)
            Ks = principal_submatrices(A, I)                    # V_l A V_l^T
            pm = ispress[I]                                     # (P, m) pressure mask
            npress = pm.sum(axis=1)
            Kdef = Ks.copy()
            vs = np.zeros((len(plist), m))
            gam = np.zeros(len(plist))
            for q in range(len(plist)):
                if npress[q] == 0:
                    continue
                v = pm[q] / np.sqrt(npress[q])
                Kv = Ks[q] @ v
                g = -(v @ Kv)                                   # eigenvalue -gamma
                assert np.linalg.norm(Kv + g * v) <= 1e-12 * max(1.0, np.abs(Ks[q]).max()), \
                    "constant pressure must be an exact patch eigenvector"
                y = ~pm[q]
                if y.any():
                    Ay = Ks[q][np.ix_(y, y)]
                    By = Ks[q][np.ix_(pm[q], y)]
                    S = By @ np.linalg.solve(Ay, By.T)
                    sigma = np.trace(S) / npress[q]
                else:
                    sigma = 1.0
                Kdef[q] += sigma * np.outer(v, v)
                vs[q] = v
                gam[q] = g
            self.data.append(dict(I=I, K=Ks, Kdef=Kdef, v=vs, gamma=gam, npress=npress))

    def patch_solve(self, d, R):
        """K_l^{-1} R for the stacked residuals R (P, m) of one group (deflated)."""
        v = d["v"]
        vr = np.einsum("pm,pm->p", v, R)
        Rp = R - vr[:, None] * v
        Y = np.linalg.solve(d["Kdef"], Rp[..., None])[..., 0]
        has = d["npress"] > 0
        Y[has] += (vr[has] / (-d["gamma"][has]))[:, None] * v[has]
        return Y

    def apply_Minv(self, r):
        """M^{-1} r = sum_l V_l^T D_l K_l^{-1} V_l r."""
        out = np.zeros_like(r)
        for d in self.data:
            I = d["I"]
            Y = self.patch_solve(d, r[I])
            np.add.at(out, I.ravel(), (self.weight[I] * Y).ravel())
        return out

    def sweep(self, x, b, omega):
        r = b - self.op.A @ x
        return x + omega * self.apply_Minv(r)


class DispVanka:
    """A_{V,u}^{-1}: additive Vanka with 8-DoF displacement patches on A_u^RQ
    (Fig. fig:patches left, eq. F-Vanka)."""

    def __init__(self, op: Operator, reverse: bool = False):
        mesh = op.mesh
        Au = op.Au
        # positions in the displacement block: active slots of planes 0..4 in op.iu order
        posu = np.full(mesh.nslots, -1, dtype=np.int64)
        posu[mesh.act_idx[op.iu]] = np.arange(op.iu.size)
        tris, edges = mesh.vertex_incidence()
        N1 = mesh.N1
        patches = []
        for vid in range(N1 * N1):
            i, j = vid % N1, vid // N1
            slots = [mesh.slot(0, i, j), mesh.slot(1, i, j)] + [mesh.slot(2 + k, ei, ej) for (k, ei, ej) in edges[vid]]
            pos = posu[np.array(slots)]
            pos = pos[pos >= 0]
            if pos.size:
                patches.append(pos[::-1] if reverse else pos)
        count = np.zeros(Au.shape[0])
        for p in patches:
            count[p] += 1
        assert np.all(count > 0)
        self.weight = 1.0 / count
        groups = {}
        for p in patches:
            groups.setdefault(p.size, []).append(p)
        self.data = []
        for m, plist in sorted(groups.items()):
            I = np.array(plist)
            Ks = principal_submatrices(Au, I)
            self.data.append(dict(I=I, K=Ks))
        self.n = Au.shape[0]

    def apply(self, r):
        out = np.zeros(self.n)
        for d in self.data:
            I = d["I"]
            Y = np.linalg.solve(d["K"], r[I][..., None])[..., 0]
            np.add.at(out, I.ravel(), (self.weight[I] * Y).ravel())
        return out


class BSR:
    """Inexact Braess-Sarazin relaxation; exact=True: exact BSR, the Schur
    complement system S dp = g of eq. bsr_p solved exactly (sparse LU) instead of by n_J Jacobi
    sweeps -- "the method with exact inversion of this system in eq. bsr_p"."""

    def __init__(self, op: Operator, d: int = 2, reverse: bool = False, exact: bool = False):
        self.op = op
        self.exact = exact
        self.Fu = DispVanka(op, reverse)
        self.Dw = op.Mw.diagonal()                              # D_w = diag(M_w)
        s0 = op.inv_M + op.alpha ** 2 / (op.lam + 2.0 * op.mu / d)
        self.S = (s0 * op.Mp + op.tau * (op.Bw @ sp.diags(1.0 / self.Dw) @ op.Bw.T)).tocsr()
        self.diagS = self.S.diagonal()
        if exact:
            import scipy.sparse.linalg as spla
            self.Slu = spla.splu(self.S.tocsc())

    def sweep(self, x, b, omega, omega_J, n_J):
        op = self.op
        r = b - op.A @ x
        ru, rw, rp = r[op.iu], r[op.iw], r[op.ip]
        tau, alpha = op.tau, op.alpha
        zu = self.Fu.apply(ru)                                  # A_{V,u}^{-1} r_u
        zw = rw / (tau * self.Dw)                               # (tau D_w)^{-1} r_w
        g = alpha * (op.Bu @ zu) + tau * (op.Bw @ zw) - rp      # B F^{-1} r_y - r_p
        dp = np.zeros_like(g)
        if self.exact:                                          # exact BSR: S dp = g (eq. bsr_p)
            dp = self.Slu.solve(g)
        else:
            for _ in range(n_J):                                # weighted Jacobi on S dp = g
                dp = dp + omega_J * (g - self.S @ dp) / self.diagS
        du = self.Fu.apply(ru - alpha * (op.Bu.T @ dp))         # F dy = r_y - B^T dp
        dw = (rw - tau * (op.Bw.T @ dp)) / (tau * self.Dw)
        xn = x.copy()
        xn[op.iu] += omega * du
        xn[op.iw] += omega * dw
        xn[op.ip] += omega * dp
        return xn

// Host-side setup of the B200 multigrid path: per-level stencil coefficients, deflated Vanka
// patch inverses, displacement-patch inverses (BSR) and the dense deflated coarsest inverse.
// Pure host fp64 / long double math; no CUDA calls, so the CPU test-suite can call it through
// mg_host_level_tables().  Geometry comes from the generated mg_tables.h (gen_tables.py).
//
//  * element entries of A^RQ: eq. block_form_rq
//  * Vanka patch matrices K_v = V_v A V_v^T and natural weights D_v: PAPER.md:575-590
//  * exact deflation of the constant-pressure eigenvector (reading A9)
//  * displacement patches A^RQ_{u,v} for the inexact BSR smoother: PAPER.md:686, 1682-1688
//  * coarsest direct solve: PAPER.md:945
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "mg_internal.h"
#include "mg_tables.h"

namespace {

const int VSLOT[MG_PSLOTS][3] = MG_VSLOT_TABLE;

int blk(int q) { return q < 9 ? 0 : (q < 12 ? 1 : 2); }   // 0 = u, 1 = w, 2 = p

// Entry (q, q2) of the element matrix of A^RQ on a triangle of shape s at mesh size h.
double elem_entry(int s, int q, int q2, const Material& m, double h, double kinv) {
    int a = blk(q), b = blk(q2);
    if (a == 0 && b == 0) {
        double v = 2.0 * m.mu * REF_AEPS[s][q][q2] + 2.0 * m.lambda * REF_BU[s][q] * REF_BU[s][q2];
        // exact integration of lambda (div u, div v) (eq. block_form) = the reduced quadrature plus the
        // bubble block REF_EXDIV (h-independent)
        if (m.exact && q >= 6 && q2 >= 6) v += m.lambda * REF_EXDIV[s][q - 6][q2 - 6];
        return v;
    }
    if (a == 0 && b == 2) return m.alpha * h * REF_BU[s][q];
    if (a == 2 && b == 0) return m.alpha * h * REF_BU[s][q2];
    if (a == 1 && b == 1) return m.tau * m.mu_f * kinv * h * h * REF_MW1[s][q - 9][q2 - 9];
    if (a == 1 && b == 2) return m.tau * h * REF_BW[s][q - 9];
    if (a == 2 && b == 1) return m.tau * h * REF_BW[s][q2 - 9];
    if (a == 2 && b == 2) return -m.inv_M * h * h * REF_MP[s];
    return 0.0;
}

bool active(int p, int i, int j, int n) {
    if (i < 0 || j < 0 || i > n || j > n) return false;
    switch (p) {
        case 0: case 1: return i > 0 && i < n && j > 0 && j < n;
        case 2: case 5: return i < n && j > 0 && j < n;
        case 3: case 6: return i > 0 && i < n && j < n;
        default: return i < n && j < n;
    }
}

// In-place inverse of the m x m matrix A (row major) by Gauss-Jordan elimination with partial
// pivoting in long double.  Returns false if singular.
bool invert(std::vector<long double>& A, int m) {
    std::vector<long double> I(m * (size_t)m, 0.0L);
    for (int i = 0; i < m; ++i) I[i * (size_t)m + i] = 1.0L;
    for (int c = 0; c < m; ++c) {
        int piv = c;
        for (int r = c + 1; r < m; ++r)
            if (fabsl(A[r * (size_t)m + c]) > fabsl(A[piv * (size_t)m + c])) piv = r;
        if (A[piv * (size_t)m + c] == 0.0L) return false;
        if (piv != c)
            for (int k = 0; k < m; ++k) {
                std::swap(A[c * (size_t)m + k], A[piv * (size_t)m + k]);
                std::swap(I[c * (size_t)m + k], I[piv * (size_t)m + k]);
            }
        // columns < c of A are never read again (pivot search and multipliers look at columns
        // >= c only), so they are not updated: the result I is the same, with 3/4 of the work
        long double d = 1.0L / A[c * (size_t)m + c];
        for (int k = c; k < m; ++k) A[c * (size_t)m + k] *= d;
        for (int k = 0; k < m; ++k) I[c * (size_t)m + k] *= d;
        for (int r = 0; r < m; ++r) {
            if (r == c) continue;
            long double f = A[r * (size_t)m + c];
            if (f == 0.0L) continue;
            for (int k = c; k < m; ++k) A[r * (size_t)m + k] -= f * A[c * (size_t)m + k];
            for (int k = 0; k < m; ++k) I[r * (size_t)m + k] -= f * I[c * (size_t)m + k];
        }
    }
    A.swap(I);
    return true;
}

// Deflated inverse of a symmetric saddle-point block K (m x m, row major) whose pressure
// indicator vector (ispress) spans an exact eigenvector v = 1_p / sqrt(mp) with eigenvalue
// -gamma (reading A9):  K^{-1} r = (v.r / -gamma) v + (K - sigma v v^T)^{-1} (r - v v.r).
// Returns the matrix of that map.  Without pressure DoFs it is the plain inverse.
bool deflated_inverse(const std::vector<double>& K, const std::vector<int>& ispress, int m,
                      std::vector<double>& G, char* err, int errlen) {
    int mp = 0;
    for (int i = 0; i < m; ++i) mp += ispress[i];
    std::vector<long double> Kd(m * (size_t)m);
    for (size_t i = 0; i < Kd.size(); ++i) Kd[i] = K[i];
    G.assign(m * (size_t)m, 0.0);
    if (mp == 0) {
        if (!invert(Kd, m)) { snprintf(err, errlen, "singular displacement patch"); return false; }
        for (size_t i = 0; i < G.size(); ++i) G[i] = (double)Kd[i];
        return true;
    }
    std::vector<long double> v(m, 0.0L);
    for (int i = 0; i < m; ++i) v[i] = ispress[i] ? 1.0L / sqrtl((long double)mp) : 0.0L;
    // gamma = -v^T K v and the eigen-residual check
    std::vector<long double> Kv(m, 0.0L);
    long double kmax = 0.0L;
    for (int i = 0; i < m; ++i)
        for (int k = 0; k < m; ++k) {
            Kv[i] += (long double)K[i * (size_t)m + k] * v[k];
            kmax = fmaxl(kmax, fabsl((long double)K[i * (size_t)m + k]));
        }
    long double gamma = 0.0L;
    for (int i = 0; i < m; ++i) gamma -= v[i] * Kv[i];
    long double res = 0.0L;
    for (int i = 0; i < m; ++i) res = fmaxl(res, fabsl(Kv[i] + gamma * v[i]));
    if (res > 1e-12L * fmaxl(kmax, 1.0L)) {
        snprintf(err, errlen, "constant pressure is not an exact eigenvector (res %.3Le)", res);
        return false;
    }
    if (gamma <= 0.0L) {
        snprintf(err, errlen, "inv_M must be > 0 for the deflated solve (gamma = %.3Le)", gamma);
        return false;
    }
    // sigma: mean diagonal of the pressure Schur complement in the diagonal approximation
    long double sig = 0.0L;
    for (int p = 0; p < m; ++p) {
        if (!ispress[p]) continue;
        for (int y = 0; y < m; ++y)
            if (!ispress[y] && K[y * (size_t)m + y] != 0.0)
                sig += (long double)K[p * (size_t)m + y] * K[p * (size_t)m + y] / K[y * (size_t)m + y];
    }
    sig /= mp;
    if (sig == 0.0L) sig = gamma;
    for (int i = 0; i < m; ++i)
        for (int k = 0; k < m; ++k) Kd[i * (size_t)m + k] -= sig * v[i] * v[k];
    if (!invert(Kd, m)) { snprintf(err, errlen, "singular deflated patch"); return false; }
    // G = Kd^{-1} (I - v v^T) + (-1/gamma) v v^T
    for (int i = 0; i < m; ++i)
        for (int k = 0; k < m; ++k) {
            long double s = 0.0L;
            for (int t = 0; t < m; ++t) s += Kd[i * (size_t)m + t] * ((t == k ? 1.0L : 0.0L) - v[t] * v[k]);
            s += -v[i] * v[k] / gamma;
            G[i * (size_t)m + k] = (double)s;
        }
    return true;
}

// Patch matrix K (ns x ns, row major over the first ns VSLOT entries) of vertex (a, b) at mesh
// size n: sum over the star triangles of the element matrices restricted to active patch DoFs.
// ww_scale multiplies the M_w part (0 for the displacement patches, which use A_u^RQ only).
void patch_matrix(int a, int b, int n, int ns, const Material& m, double h, std::vector<double>& K,
                  std::vector<int>& act) {
    K.assign(ns * (size_t)ns, 0.0);
    act.assign(ns, 0);
    for (int s = 0; s < ns; ++s) act[s] = active(VSLOT[s][2], a + VSLOT[s][0], b + VSLOT[s][1], n);
    for (int cx = -1; cx <= 0; ++cx)
        for (int cy = -1; cy <= 0; ++cy) {
            int ci = a + cx, cj = b + cy;
            if (ci < 0 || cj < 0 || ci >= n || cj >= n) continue;
            for (int sh = 0; sh < 2; ++sh) {
                int loc[13];
                for (int q = 0; q < 13; ++q) {
                    loc[q] = -1;
                    int dx = cx + LOCAL_DOF[sh][q][0], dy = cy + LOCAL_DOF[sh][q][1], p = LOCAL_DOF[sh][q][2];
                    for (int s = 0; s < ns; ++s)
                        if (VSLOT[s][0] == dx && VSLOT[s][1] == dy && VSLOT[s][2] == p && act[s]) loc[q] = s;
                }
                for (int q = 0; q < 13; ++q)
                    for (int q2 = 0; q2 < 13; ++q2) {
                        if (loc[q] < 0 || loc[q2] < 0) continue;
                        K[loc[q] * (size_t)ns + loc[q2]] += elem_entry(sh, q, q2, m, h, 1.0 / m.K);
                    }
            }
        }
}

// weighted, deflated inverse over the active slots, embedded in ns x ns
bool patch_inverse(int a, int b, int n, int ns, const Material& m, double h, double* out, char* err,
                   int errlen) {
    std::vector<double> K;
    std::vector<int> act;
    patch_matrix(a, b, n, ns, m, h, K, act);
    std::vector<int> idx;
    for (int s = 0; s < ns; ++s)
        if (act[s]) idx.push_back(s);
    int mm = (int)idx.size();
    memset(out, 0, sizeof(double) * ns * ns);
    if (mm == 0) return true;
    std::vector<double> Ks(mm * (size_t)mm), G;
    std::vector<int> isp(mm);
    for (int r = 0; r < mm; ++r) {
        isp[r] = idx[r] >= 14;
        for (int c = 0; c < mm; ++c) Ks[r * (size_t)mm + c] = K[idx[r] * (size_t)ns + idx[c]];
    }
    if (!deflated_inverse(Ks, isp, mm, G, err, errlen)) return false;
    for (int r = 0; r < mm; ++r) {
        int s = idx[r];
        double w = s < 2 ? 1.0 : (s < 14 ? 0.5 : 1.0 / 3.0);   // natural weights
        for (int c = 0; c < mm; ++c) out[s * ns + idx[c]] = w * G[r * (size_t)mm + c];
    }
    return true;
}

int class_coord(int c, int n) { return c == 0 ? 1 : (c == 1 ? 0 : n); }

// Eigen-decomposition of a symmetric m x m matrix (m <= 6) by cyclic Jacobi rotations in long
// double: A is destroyed (its diagonal ends up holding the eigenvalues), V receives the eigenvectors
// as columns.
void jacobi_eigen(long double A[6][6], long double V[6][6], int m) {
    for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j) V[i][j] = i == j ? 1.0L : 0.0L;
    for (int sweep = 0; sweep < 100; ++sweep) {
        long double off = 0.0L, tot = 0.0L;
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < m; ++j) {
                tot += A[i][j] * A[i][j];
                if (i != j) off += A[i][j] * A[i][j];
            }
        if (off <= 1e-38L * tot) break;
        for (int p = 0; p < m; ++p)
            for (int q = p + 1; q < m; ++q) {
                if (A[p][q] == 0.0L) continue;
                const long double th = (A[q][q] - A[p][p]) / (2.0L * A[p][q]);
                const long double t = (th >= 0 ? 1.0L : -1.0L) / (fabsl(th) + sqrtl(th * th + 1.0L));
                const long double c = 1.0L / sqrtl(t * t + 1.0L), sn = t * c;
                for (int k = 0; k < m; ++k) {       // A <- A J
                    const long double akp = A[k][p], akq = A[k][q];
                    A[k][p] = c * akp - sn * akq;
                    A[k][q] = sn * akp + c * akq;
                }
                for (int k = 0; k < m; ++k) {       // A <- J^T A
                    const long double apk = A[p][k], aqk = A[q][k];
                    A[p][k] = c * apk - sn * aqk;
                    A[q][k] = sn * apk + c * aqk;
                }
                for (int k = 0; k < m; ++k) {       // V <- V J
                    const long double vkp = V[k][p], vkq = V[k][q];
                    V[k][p] = c * vkp - sn * vkq;
                    V[k][q] = sn * vkp + c * vkq;
                }
            }
    }
}

// Condensed heterogeneous-Vanka tables of the vertex (a, b) (mg_internal.h HetVankaTabs): the patch
// matrix without its M_w block (K0 with kinv = 0) split into y = slots 0..7, 14..19 and r = 8..13.
bool hv_class_tables(int a, int b, int n, const Material& m, double h, double* cls, double* W, double* C,
                     char* err, int errlen, HvInteriorPM* pm = nullptr) {
    Material m0 = m;
    m0.K = INFINITY;                                           // kinv = 0: K0 has no M_w block
    std::vector<double> K;
    std::vector<int> act;
    patch_matrix(a, b, n, MG_PSLOTS, m0, h, K, act);
    static const int YS[14] = {0, 1, 2, 3, 4, 5, 6, 7, 14, 15, 16, 17, 18, 19};
    std::vector<int> yi;                                       // active y slots (positions in YS)
    for (int q = 0; q < 14; ++q)
        if (act[YS[q]]) yi.push_back(q);
    const int my = (int)yi.size();
    memset(cls, 0, sizeof(double) * MG_HV_CLS);
    memset(W, 0, sizeof(double) * MG_HV_W);
    memset(C, 0, sizeof(double) * 36);
    // G_def over the active y slots (long double): deflated_inverse gives G = G_def - v v^T / gamma
    std::vector<double> Ky(my * (size_t)my), G;
    std::vector<int> isp(my);
    int mp = 0;
    for (int r = 0; r < my; ++r) {
        isp[r] = YS[yi[r]] >= 14;
        mp += isp[r];
        for (int c = 0; c < my; ++c) Ky[r * (size_t)my + c] = K[YS[yi[r]] * MG_PSLOTS + YS[yi[c]]];
    }
    std::vector<long double> Gd(14 * 14, 0.0L);
    if (my > 0) {
        if (!deflated_inverse(Ky, isp, my, G, err, errlen)) return false;
        const long double gamma = (long double)m.inv_M * h * h * 0.5L;   // -(1/M) M_p on v, M_p = h^2/2
        for (int r = 0; r < my; ++r)
            for (int c = 0; c < my; ++c) {
                long double g = G[r * (size_t)my + c];
                if (isp[r] && isp[c]) g += 1.0L / (mp * gamma);           // + v v^T / gamma
                Gd[yi[r] * 14 + yi[c]] = g;
            }
        if (mp > 0) cls[MG_HV_PINV] = (double)(1.0L / (mp * gamma));
    }
    // K_yr (y x 6) and K_ry on the active slots; Q = G_def K_yr; C = K_ry Q
    long double Kyr[14][6] = {}, Q[14][6] = {};
    for (int q = 0; q < 14; ++q)
        for (int e = 0; e < 6; ++e)
            if (act[YS[q]] && act[8 + e]) Kyr[q][e] = K[YS[q] * MG_PSLOTS + 8 + e];
    for (int q = 0; q < 14; ++q)
        for (int e = 0; e < 6; ++e) {
            long double s2 = 0.0L;
            for (int t = 0; t < 14; ++t) s2 += Gd[q * 14 + t] * Kyr[t][e];
            Q[q][e] = s2;
        }
    // orthonormal basis U of the active RT0 slots: kernel of K_yr first (eigenvalue ~ 0 of
    // K_yr^T K_yr), then its complement; inactive slots keep unit vectors (they carry no data)
    int ar[6], na = 0;
    for (int e = 0; e < 6; ++e)
        if (act[8 + e]) ar[na++] = e;
    long double U[6][6] = {};
    for (int e = 0; e < 6; ++e) U[e][e] = 1.0L;
    bool isnull[6] = {false, false, false, false, false, false};
    if (pm && na == 6) {
        // interior class: one orthonormal basis per sector of the 180-degree rotation (RT0 pair
        // differences = + sector, sums = - sector), kernel vectors first within each sector; the
        // +/- split of the patch solve (HvInteriorPM) needs U block diagonal in that sense
        const long double r2 = 1.0L / sqrtl(2.0L);
        for (int sg = 0; sg < 2; ++sg) {
            long double Tr[6][3] = {};
            for (int q = 0; q < 3; ++q) {
                Tr[2 * q][q] = r2;
                Tr[2 * q + 1][q] = sg == 0 ? -r2 : r2;
            }
            long double M[6][6] = {}, E[6][6], mmax = 0.0L;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) {
                    long double s2 = 0.0L;
                    for (int t = 0; t < 14; ++t) {
                        long double bi = 0.0L, bj = 0.0L;
                        for (int e = 0; e < 6; ++e) {
                            bi += Kyr[t][e] * Tr[e][i];
                            bj += Kyr[t][e] * Tr[e][j];
                        }
                        s2 += bi * bj;
                    }
                    M[i][j] = s2;
                    mmax = fmaxl(mmax, fabsl(s2));
                }
            jacobi_eigen(M, E, 3);
            int order[3], k = 0;
            for (int i = 0; i < 3; ++i)
                if (M[i][i] <= 1e-14L * mmax) order[k++] = i;
            const int nnull = k;
            for (int i = 0; i < 3; ++i)
                if (!(M[i][i] <= 1e-14L * mmax)) order[k++] = i;
            for (int j = 0; j < 3; ++j) {
                for (int e = 0; e < 6; ++e) {
                    long double v = 0.0L;
                    for (int i = 0; i < 3; ++i) v += Tr[e][i] * E[i][order[j]];
                    U[e][3 * sg + j] = v;
                }
                isnull[3 * sg + j] = j < nnull;
            }
        }
    } else if (na > 0) {
        long double M[6][6] = {}, E[6][6];
        long double mmax = 0.0L;
        for (int i = 0; i < na; ++i)
            for (int j = 0; j < na; ++j) {
                long double s2 = 0.0L;
                for (int t = 0; t < 14; ++t) s2 += Kyr[t][ar[i]] * Kyr[t][ar[j]];
                M[i][j] = s2;
                mmax = fmaxl(mmax, fabsl(s2));
            }
        jacobi_eigen(M, E, na);
        int order[6], k = 0;
        for (int i = 0; i < na; ++i)
            if (M[i][i] <= 1e-14L * mmax) order[k++] = i;
        const int nnull = k;
        for (int i = 0; i < na; ++i)
            if (!(M[i][i] <= 1e-14L * mmax)) order[k++] = i;
        for (int e = 0; e < 6; ++e)
            if (act[8 + e])
                for (int j = 0; j < 6; ++j) U[e][j] = 0.0L;
        // basis vector j (j < na) occupies column ar[j]; inactive slots keep their unit column
        for (int j = 0; j < na; ++j) {
            for (int i = 0; i < na; ++i) U[ar[i]][ar[j]] = E[i][order[j]];
            isnull[ar[j]] = j < nnull;
        }
    }
    // U^T C U (C = K_ry G_def K_yr) with the kernel rows / columns exactly 0
    long double KU[14][6] = {}, QU[14][6] = {};
    for (int t = 0; t < 14; ++t)
        for (int j = 0; j < 6; ++j) {
            long double s2 = 0.0L, s3 = 0.0L;
            for (int e = 0; e < 6; ++e) {
                s2 += Kyr[t][e] * U[e][j];
                s3 += Q[t][e] * U[e][j];
            }
            KU[t][j] = isnull[j] ? 0.0L : s2;
            QU[t][j] = isnull[j] ? 0.0L : s3;
        }
    for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j) {
            long double s2 = 0.0L;
            for (int t = 0; t < 14; ++t) s2 += KU[t][i] * QU[t][j];
            C[i * 6 + j] = (double)s2;
        }
    for (int q = 0; q < MG_PSLOTS; ++q)   // natural weights
        cls[MG_HV_D + q] = act[q] ? (q < 2 ? 1.0 : (q < 14 ? 0.5 : 1.0 / 3.0)) : 0.0;
    for (int q = 0; q < 14; ++q)
        for (int c = 0; c < 14; ++c) cls[MG_HV_G + q * 14 + c] = (double)Gd[q * 14 + c];
    for (int q = 0; q < 14; ++q)
        for (int j = 0; j < 6; ++j) cls[MG_HV_Q + q * 6 + j] = (double)QU[q][j];
    for (int j = 0; j < 6; ++j)
        for (int k = 0; k < 6; ++k) {
            for (int q = 0; q < 8; ++q)   // K_ry has no u / bubble columns (zero (w, u) block of A^RQ)
                if (Kyr[q][j] != 0.0L) { snprintf(err, errlen, "K_ry has a displacement column"); return false; }
            cls[MG_HV_KRP + j * 6 + k] = (double)KU[8 + k][j];
        }
    for (int e = 0; e < 6; ++e)
        for (int j = 0; j < 6; ++j) cls[MG_HV_U + e * 6 + j] = (double)U[e][j];
    // U^T M_w,v U of each star triangle per unit K^{-1}: tau mu_f h^2 REF_MW1 on the RT0 slots
    for (int ty = 0; ty < 2; ++ty)
        for (int tx = 0; tx < 2; ++tx) {
            const int ci = a - 1 + tx, cj = b - 1 + ty;
            if (ci < 0 || cj < 0 || ci >= n || cj >= n) continue;
            for (int sh = 0; sh < 2; ++sh) {
                int loc[3];
                for (int e = 0; e < 3; ++e) {
                    loc[e] = -1;
                    const int q = 9 + e;                       // RT0 local DoFs of the triangle
                    const int dx = tx - 1 + LOCAL_DOF[sh][q][0], dy = ty - 1 + LOCAL_DOF[sh][q][1], p = LOCAL_DOF[sh][q][2];
                    for (int s2 = 8; s2 < 14; ++s2)
                        if (VSLOT[s2][0] == dx && VSLOT[s2][1] == dy && VSLOT[s2][2] == p && act[s2]) loc[e] = s2 - 8;
                }
                long double Wl[6][6] = {};
                for (int e = 0; e < 3; ++e)
                    for (int f = 0; f < 3; ++f)
                        if (loc[e] >= 0 && loc[f] >= 0)
                            Wl[loc[e]][loc[f]] += (long double)m.tau * m.mu_f * h * h * REF_MW1[sh][e][f];
                double* Wt = W + (4 * sh + 2 * ty + tx) * 36;
                for (int i = 0; i < 6; ++i)
                    for (int j = 0; j < 6; ++j) {
                        long double s2 = 0.0L;
                        for (int e = 0; e < 6; ++e)
                            for (int f = 0; f < 6; ++f) s2 += U[e][i] * Wl[e][f] * U[f][j];
                        Wt[i * 6 + j] = (double)s2;
                    }
            }
        }
    if (pm && na == 6 && my == 14) {
        // +/- tables of the interior class (mg_internal.h HvInteriorPM): hat input h = Tin y (pair
        // differences / sums, P0 pairs the other way round), hat output Tout = Tin with 1/2 on the
        // pair rows, so that slot a = hat- + hat+, slot b = hat- - hat+ (P0: a = + + -, b = + - -)
        long double Tin[14][14] = {}, Tout[14][14] = {};
        const int bub[3][2] = {{2, 3}, {4, 5}, {6, 7}}, p0[3][2] = {{8, 9}, {10, 11}, {12, 13}};
        for (int q = 0; q < 3; ++q) {
            Tin[q][bub[q][0]] = 1.0L; Tin[q][bub[q][1]] = -1.0L;              // + : bubble differences
            Tin[3 + q][p0[q][0]] = 1.0L; Tin[3 + q][p0[q][1]] = 1.0L;         // + : P0 sums
            Tin[8 + q][bub[q][0]] = 1.0L; Tin[8 + q][bub[q][1]] = 1.0L;       // - : bubble sums
            Tin[11 + q][p0[q][0]] = 1.0L; Tin[11 + q][p0[q][1]] = -1.0L;      // - : P0 differences
        }
        Tin[6][0] = 1.0L;                                                       // - : u_x, u_y
        Tin[7][1] = 1.0L;
        for (int r = 0; r < 14; ++r)
            for (int c = 0; c < 14; ++c) Tout[r][c] = (r == 6 || r == 7) ? Tin[r][c] : 0.5L * Tin[r][c];
        std::vector<long double> TiI(14 * 14), ToI(14 * 14);
        for (int r = 0; r < 14; ++r)
            for (int c = 0; c < 14; ++c) {
                TiI[r * 14 + c] = Tin[r][c];
                ToI[r * 14 + c] = Tout[r][c];
            }
        if (!invert(TiI, 14) || !invert(ToI, 14)) { snprintf(err, errlen, "hat transform"); return false; }
        // G^ = Tout G_def Tin^{-1}, Q^ = Tout Q U, K^ = U^T K_ry Tout^{-1}
        long double Gh[14][14], Qh[14][6], Kh[6][14], gmax = 0.0L;
        for (int r = 0; r < 14; ++r)
            for (int c = 0; c < 14; ++c) {
                long double s2 = 0.0L;
                for (int t = 0; t < 14; ++t)
                    for (int u = 0; u < 14; ++u) s2 += Tout[r][t] * Gd[t * 14 + u] * TiI[u * 14 + c];
                Gh[r][c] = s2;
                gmax = fmaxl(gmax, fabsl(s2));
            }
        for (int r = 0; r < 14; ++r)
            for (int j2 = 0; j2 < 6; ++j2) {
                long double s2 = 0.0L;
                for (int t = 0; t < 14; ++t) s2 += Tout[r][t] * QU[t][j2];
                Qh[r][j2] = s2;
            }
        for (int j2 = 0; j2 < 6; ++j2)
            for (int c = 0; c < 14; ++c) {
                long double s2 = 0.0L;
                for (int t = 0; t < 14; ++t) s2 += KU[t][j2] * ToI[t * 14 + c];
                Kh[j2][c] = s2;
            }
        auto blk = [](int r) { return r < 6 ? 0 : 1; };   // hat sector of a y component
        long double off = 0.0L, qmax = 0.0L, kmax = 0.0L;
        for (int r = 0; r < 14; ++r)
            for (int c = 0; c < 14; ++c)
                if (blk(r) != blk(c)) off = fmaxl(off, fabsl(Gh[r][c]) / gmax);
        for (int r = 0; r < 14; ++r)
            for (int j2 = 0; j2 < 6; ++j2) qmax = fmaxl(qmax, fabsl(Qh[r][j2]));
        for (int j2 = 0; j2 < 6; ++j2)
            for (int c = 0; c < 14; ++c) kmax = fmaxl(kmax, fabsl(Kh[j2][c]));
        for (int r = 0; r < 14; ++r)
            for (int j2 = 0; j2 < 6; ++j2)
                if (blk(r) != j2 / 3) off = fmaxl(off, fabsl(Qh[r][j2]) / qmax);
        for (int j2 = 0; j2 < 6; ++j2)
            for (int c = 0; c < 14; ++c) {
                const bool keep = (j2 < 3 && c >= 3 && c < 6) || (j2 >= 3 && c >= 11);
                if (!keep) off = fmaxl(off, fabsl(Kh[j2][c]) / kmax);
            }
        if (off > 1e-11L) {
            snprintf(err, errlen, "interior heterogeneous-Vanka tables are not +/- block diagonal (%.3Le)", off);
            return false;
        }
        for (int r = 0; r < 6; ++r)
            for (int c = 0; c < 6; ++c) pm->gp[r][c] = (double)Gh[r][c];
        for (int r = 0; r < 8; ++r)
            for (int c = 0; c < 8; ++c) pm->gm[r][c] = (double)Gh[6 + r][6 + c];
        for (int j2 = 0; j2 < 3; ++j2)
            for (int k = 0; k < 3; ++k) {
                pm->kp[j2][k] = (double)Kh[j2][3 + k];
                pm->km[j2][k] = (double)Kh[3 + j2][11 + k];
                pm->up[j2][k] = (double)U[2 * k][j2];          // applied to RT0 differences / sums
                pm->um[j2][k] = (double)U[2 * k][3 + j2];
            }
        for (int r = 0; r < 6; ++r)
            for (int j2 = 0; j2 < 3; ++j2) pm->qp[r][j2] = (double)Qh[r][j2];
        for (int r = 0; r < 8; ++r)
            for (int j2 = 0; j2 < 3; ++j2) pm->qm[r][j2] = (double)Qh[6 + r][3 + j2];
        pm->pinv = cls[MG_HV_PINV];
    }
    return true;
}

// +/- basis of the 180-degree rotation for ns = 20 (Vanka) or 8 (displacement).  comp[t] lists
// hat component t as (slot a, slot b, sign): hat_t = r_a + sign r_b (b < 0: single).
struct HatComp { int a, b, sg; };
void hat_basis(int ns, std::vector<HatComp>& plus, std::vector<HatComp>& minus) {
    plus.clear(); minus.clear();
    minus.push_back({0, -1, 0});
    minus.push_back({1, -1, 0});
    int npair_edge = ns == 20 ? 6 : 3;
    for (int q = 0; q < npair_edge; ++q) {          // bubble / RT0 pairs: diff in +, sum in -
        plus.push_back({2 + 2 * q, 3 + 2 * q, -1});
        minus.push_back({2 + 2 * q, 3 + 2 * q, +1});
    }
    if (ns == 20)
        for (int q = 0; q < 3; ++q) {               // P0 pairs: sum in +, diff in -
            plus.push_back({14 + 2 * q, 15 + 2 * q, +1});
            minus.push_back({14 + 2 * q, 15 + 2 * q, -1});
        }
}

// Split the interior weighted inverse G (ns x ns) into the +/- blocks (with 1/2 folded into pair
// rows).  Checks block diagonality.
bool split_pm(const double* G, int ns, double* gp, double* gm, char* err, int errlen) {
    std::vector<HatComp> P, M;
    hat_basis(ns, P, M);
    std::vector<HatComp> all(P);
    all.insert(all.end(), M.begin(), M.end());
    int np = (int)P.size();
    // T (ns x ns): hat = T r ; Tinv: r = Tinv hat
    std::vector<double> T(ns * ns, 0.0), Ti(ns * ns, 0.0);
    for (int t = 0; t < ns; ++t) {
        T[t * ns + all[t].a] = 1.0;
        if (all[t].b >= 0) T[t * ns + all[t].b] = all[t].sg;
    }
    for (int t = 0; t < ns; ++t) {                    // columns of Tinv
        if (all[t].b < 0) { Ti[all[t].a * ns + t] = 1.0; continue; }
        Ti[all[t].a * ns + t] = 0.5;
        Ti[all[t].b * ns + t] = 0.5 * all[t].sg;
    }
    std::vector<double> TG(ns * ns, 0.0), Gh(ns * ns, 0.0);
    for (int i = 0; i < ns; ++i)
        for (int k = 0; k < ns; ++k) {
            double s = 0;
            for (int t = 0; t < ns; ++t) s += T[i * ns + t] * G[t * ns + k];
            TG[i * ns + k] = s;
        }
    double gmax = 0;
    for (int i = 0; i < ns; ++i)
        for (int k = 0; k < ns; ++k) {
            double s = 0;
            for (int t = 0; t < ns; ++t) s += TG[i * ns + t] * Ti[t * ns + k];
            Gh[i * ns + k] = s;
            gmax = fmax(gmax, fabs(s));
        }
    for (int i = 0; i < ns; ++i)
        for (int k = 0; k < ns; ++k)
            if ((i < np) != (k < np) && fabs(Gh[i * ns + k]) > 1e-11 * gmax) {
                snprintf(err, errlen, "interior patch inverse is not block diagonal in the +/- basis (%d,%d: %g)",
                         i, k, Gh[i * ns + k]);
                return false;
            }
    int nm = ns - np;
    for (int i = 0; i < np; ++i)
        for (int k = 0; k < np; ++k) gp[i * np + k] = Gh[i * ns + k] * (P[i].b >= 0 ? 0.5 : 1.0);
    for (int i = 0; i < nm; ++i)
        for (int k = 0; k < nm; ++k) gm[i * nm + k] = Gh[(np + i) * ns + np + k] * (M[i].b >= 0 ? 0.5 : 1.0);
    return true;
}

}  // namespace

int64_t n_active_of(int n) { return 10LL * n * n - 8LL * n + 2; }

int host_level_tables(int n, const Material& m, HostLevelTables* t, char* err, int errlen) {
    if (n < 2) { snprintf(err, errlen, "level n = %d < 2", n); return -1; }
    memset(t, 0, sizeof(*t));
    double h = 1.0 / n;
    t->n = n;
    t->h = h;
    LevelParams& L = t->L;
    L.n = n;
    double kinv = 1.0 / m.K;
    // the merged / factored stencil is the reduced-quadrature one; an exact-integration level adds
    // its bubble term separately in the residual (L.lamx)
    Material m_rq = m;
    m_rq.exact = 0;
    L.lamx = m.exact ? m.lambda : 0.0;
#define Y(ci, s, q, q2) L.coef[ci] += elem_entry(s, q, q2, m_rq, h, kinv);
    MG_STENCIL_CONTRIB(Y)
#undef Y
    static_assert(MG_STENCIL_NGROUP == MG_NGROUP, "factored stencil size");
#define R(g, ci, sg) L.cg[g] = (sg) * L.coef[ci];
    MG_STENCIL_GROUP_REP(R)
#undef R
    for (int s = 0; s < 2; ++s)
        for (int e = 0; e < 3; ++e) {
            for (int e2 = 0; e2 < 3; ++e2) L.ww[s][e][e2] = m.tau * m.mu_f * h * h * REF_MW1[s][e][e2];
            L.bw[s][e] = h * REF_BW[s][e];
            L.mw1d[s][e] = m.mu_f * h * h * REF_MW1[s][e][e];
        }
    for (int s = 0; s < 2; ++s)
        for (int q = 0; q < 9; ++q) L.bu[s][q] = h * REF_BU[s][q];
    L.kinv = kinv;
    L.tau = m.tau;
    L.alpha = m.alpha;
    L.s0h2 = (m.inv_M + m.alpha * m.alpha / (m.lambda + m.mu)) * h * h * 0.5;   // d = 2 (reading A19)
    // Vanka and displacement patch inverses per vertex class
    Material mu_only = m;
    for (int cy = 0; cy < 3; ++cy)
        for (int cx = 0; cx < 3; ++cx) {
            int c = cx + 3 * cy, a = class_coord(cx, n), b = class_coord(cy, n);
            if (!patch_inverse(a, b, n, MG_PSLOTS, m, h, t->vanka[c], err, errlen)) return -1;
            if (!patch_inverse(a, b, n, MG_USLOTS, mu_only, h, t->disp[c], err, errlen)) return -1;
        }
    if (!split_pm(t->vanka[0], MG_PSLOTS, &t->gp[0][0], &t->gm[0][0], err, errlen)) return -1;
    if (!split_pm(t->disp[0], MG_USLOTS, &t->up[0][0], &t->um[0][0], err, errlen)) return -1;
    return 0;
}

int host_hv_tables(int n, const Material& m, double* cls, double* W, double* C, HvInteriorPM* pm, char* err,
                   int errlen) {
    const double h = 1.0 / n;
    for (int cy = 0; cy < 3; ++cy)
        for (int cx = 0; cx < 3; ++cx) {
            const int c = cx + 3 * cy;
            if (!hv_class_tables(class_coord(cx, n), class_coord(cy, n), n, m, h, cls + c * MG_HV_CLS,
                                 W + c * MG_HV_W, C + c * 36, err, errlen, c == 0 ? pm : nullptr))
                return -1;
        }
    return 0;
}

int host_coarse_inverse(int n, int pitch, const Material& m, const double* kinvf, double* Ginv,
                        int64_t* slots, int* Nout, char* err, int errlen) {
    double h = 1.0 / n;
    // active numbering in plane-major slot order
    std::vector<int> num(10 * (size_t)(n + 1) * (n + 1), -1);
    int N = 0;
    for (int p = 0; p < 10; ++p)
        for (int j = 0; j <= n; ++j)
            for (int i = 0; i <= n; ++i)
                if (active(p, i, j, n)) {
                    num[(p * (size_t)(n + 1) + j) * (n + 1) + i] = N;
                    if (slots) slots[N] = (int64_t)p * (n + 1) * pitch + (int64_t)j * pitch + i;
                    ++N;
                }
    *Nout = N;
    if (!Ginv) return 0;
    std::vector<double> A(N * (size_t)N, 0.0);
    for (int cj = 0; cj < n; ++cj)
        for (int ci = 0; ci < n; ++ci)
            for (int sh = 0; sh < 2; ++sh) {
                double kinv = kinvf ? kinvf[(sh * (size_t)n + cj) * n + ci] : 1.0 / m.K;
                int g[13];
                for (int q = 0; q < 13; ++q) {
                    int i = ci + LOCAL_DOF[sh][q][0], j = cj + LOCAL_DOF[sh][q][1], p = LOCAL_DOF[sh][q][2];
                    g[q] = num[(p * (size_t)(n + 1) + j) * (n + 1) + i];
                }
                for (int q = 0; q < 13; ++q)
                    for (int q2 = 0; q2 < 13; ++q2)
                        if (g[q] >= 0 && g[q2] >= 0)
                            A[g[q] * (size_t)N + g[q2]] += elem_entry(sh, q, q2, m, h, kinv);
            }
    std::vector<int> isp(N, 0);
    for (int p = 8; p < 10; ++p)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) isp[num[(p * (size_t)(n + 1) + j) * (n + 1) + i]] = 1;
    std::vector<double> G;
    if (!deflated_inverse(A, isp, N, G, err, errlen)) return -1;
    for (int r = 0; r < N; ++r)
        for (int c = 0; c < N; ++c) Ginv[c * (size_t)N + r] = G[r * (size_t)N + c];   // column major
    return 0;
}

extern "C" int mg_host_level_tables(int32_t n, double lambda, double mu, double K, double tau, double alpha,
                                    double inv_M, double mu_f, double* stencil_coef, double* ww,
                                    double* vanka, double* disp) {
    Material m{lambda, mu, K, tau, alpha, inv_M, mu_f};
    static thread_local char err[256];
    HostLevelTables* t = new HostLevelTables;
    int rc = host_level_tables(n, m, t, err, sizeof(err));
    if (rc == 0) {
        if (stencil_coef) memcpy(stencil_coef, t->L.coef, sizeof(t->L.coef));
        if (ww)
            for (int s = 0; s < 2; ++s)
                for (int e = 0; e < 3; ++e)
                    for (int e2 = 0; e2 < 3; ++e2) ww[(s * 3 + e) * 3 + e2] = t->L.ww[s][e][e2] * t->L.kinv;
        if (vanka) memcpy(vanka, t->vanka, sizeof(t->vanka));
        if (disp) memcpy(disp, t->disp, sizeof(t->disp));
    }
    delete t;
    return rc == 0 ? 0 : -1;
}

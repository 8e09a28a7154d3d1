// Internal definitions shared by the host setup (mg_setup.cpp), the kernels (mg_kernels.cu) and
// the C ABI (mg_api.cu).  Not part of the public ABI (include/mg.h).
#pragma once
#include <stdint.h>

#define MG_NCOEF 141      // merged stencil coefficients (mg_tables.h MG_STENCIL_NCOEF)
#define MG_NGROUP 17      // distinct coefficients of the factored stencil (mg_tables.h MG_STENCIL_NGROUP)
#define MG_PSLOTS 20      // Vanka patch slots
#define MG_USLOTS 8       // displacement patch slots (BSR)
#define MG_NCLASS 9       // vertex classes: cx + 3 cy, cx = 0 interior, 1 at i = 0, 2 at i = n

// Patch slot s of the vertex (a, b) sits at (a + dx, b + dy) in plane p:  VSLOT[s] = {dx, dy, p}.
// Order: u_x, u_y, bubbles on the spokes E, W, N, S, NW, SE, RT0 on the same spokes, P0 of the
// triangles LL(a,b), UR(a-1,b-1), LL(a-1,b), UR(a,b-1), UR(a-1,b), LL(a,b-1) (Fig. fig:patches,
// PAPER.md:592-652).  Consecutive pairs (2,3) ... (18,19) are images of each other under the 180
// degree rotation about the vertex.
#define MG_VSLOT_TABLE {                                                           \
    {0, 0, 0}, {0, 0, 1},                                                          \
    {0, 0, 2}, {-1, 0, 2}, {0, 0, 3}, {0, -1, 3}, {-1, 0, 4}, {0, -1, 4},          \
    {0, 0, 5}, {-1, 0, 5}, {0, 0, 6}, {0, -1, 6}, {-1, 0, 7}, {0, -1, 7},          \
    {0, 0, 8}, {-1, -1, 9}, {-1, 0, 8}, {0, -1, 9}, {-1, 0, 9}, {0, -1, 8} }

// Geometry + coefficients of one level, passed by value to every kernel (constant bank).
struct LevelParams {
    int32_t n, pitch;
    int64_t plane;               // (n+1) * pitch
    double coef[MG_NCOEF];       // merged stencil of A^RQ without M_w (mg_tables.h order)
    double cg[MG_NGROUP];        // factored stencil: cg[g] = coef[representative of group g]
    double ww[2][3][3];          // tau mu_f h^2 (M_w1)_{shape,e,e'}; multiplied by K^{-1}_T
    double kinv;                 // scalar K^{-1} (used when kinv_field == nullptr)
    const double* kinv_field;    // 2 planes [shape][j][i] with row pitch `pitch`, or nullptr
    // BSR data: S = s0 M_p + tau B_w D_w^{-1} B_w^T
    double s0h2;                 // s0 |T| = (1/M + alpha^2/(lambda+mu)) h^2/2
    double tau, alpha;
    double bw[2][3];             // h (B_w1)_{shape,e}
    double bu[2][9];             // h (B_u1)_{shape,q}
    double mw1d[2][3];           // mu_f h^2 (M_w1)_{shape,e,e}   (diagonal, times K^{-1}_T)
    const int* stop;             // device flag of mg_solve: every kernel returns at entry if *stop != 0
    double lamx;                 // exact-integration operator (eq. block_form): lambda, else 0;
                                 // the residual adds lamx * REF_EXDIV on the bubbles of every triangle
};

// Device state of mg_solve, updated by the block that finishes a fused residual norm:
// hist[k] = ||b - A x_k||^2, then *stop = 1 (converged: hist[k] <= rtol2 hist[0], k > 0),
// 2 (diverged: non-finite or > 1e16 hist[0]) or 3 (k == maxk).
struct SolveState {
    int k;                       // next history slot
    int maxk;                    // max_cycles
    double rtol2;                // rtol^2
    double* hist;                // maxk + 1 doubles
    int* stop;                   // the flag every kernel polls (LevelParams::stop)
};

// Interior (symmetric) patch inverse in the +/- basis of the 180-degree rotation:
// + block (9): bubble diffs (3), RT0 diffs (3), P0 sums (3)
// - block (11): u_x, u_y, bubble sums (3), RT0 sums (3), P0 diffs (3)
// with 1/2 folded into the rows of pair components.
struct ProlSrc {                  // coarse iterate e_H for a sweep with fused prolongation
    const double* e;
    int nc, pitchc;
    int64_t planec;
};

// Heterogeneous-K Vanka (DESIGN.md section 4 "Heterogeneous Vanka"): every
// patch matrix K_v = K0_v + blockdiag(0, tau M_w,v(K)) differs only in its 6x6 RT0 block, so the
// patch solve is condensed onto the RT0 slots r = {8..13}: with y = the other 14 slots (order
// 0..7, 14..19),  a = G_def r_y,  c = -(1^T r_p)/(m gamma),  s = r_r - K_ry a,  z_r = S_v^{-1} s,
// z_y = a + c 1_p - Q z_r,  out = D z,  where G_def = K_yy^{-1} + v v^T / gamma is the deflated
// (well-conditioned) part of K_yy^{-1} (reading A9), Q = G_def K_yr, and
// S_v = tau M_w,v(K) - K_ry G_def K_yr is the per-vertex 6x6 RT0 Schur complement.
// The RT0 block is handled in an orthonormal basis U = [N, R] of the patch's RT0 slots, N spanning
// the kernel of K_yr (the divergence-free circulation around the vertex: B_w N = 0), R its
// complement.  In that basis the N rows of K_ry U and the N columns of Q U and of U^T C U are
// exactly 0, so the small circulation eigenvalue of S_v (~ tau mu_f h^2 K^{-1}) is formed from
// M_w alone, free of the rounding of the large K_ry G_def K_yr part (cond(S_v) reaches 1e6-1e9 for
// lognormal K fields).  S~_v = U^T S_v U is stored inverted per vertex.
#define MG_HV_CLS 384             // doubles per vertex-class table
#define MG_HV_G 0                 // [14][14] G_def (row major, y order)
#define MG_HV_Q 196               // [14][6]  Q U
#define MG_HV_KRP 280             // [6][6]   U^T K_ry restricted to the P0 columns ([basis row][P0 slot 14 + k])
#define MG_HV_PINV 316            // 1 / (m gamma), m = active P0 slots of the class (0 if none)
#define MG_HV_D 320               // [20] natural weights D (1, 1/2, 1/3) on the active slots, 0 elsewhere
#define MG_HV_U 344               // [6][6] U (row = RT0 slot, column = basis vector)
#define MG_HV_NSINV 21            // per-vertex planes: upper triangle of S~_v^{-1}, row by row
#define MG_HV_W 288               // setup: per class 8 triangles x [6][6] U^T M_w,v U per unit K^{-1}
// the interior vertex class's condensed patch solve in the +/- basis of the 180-degree rotation
// (kernel parameter, constant-bank operands): y inputs h+ = (bubble differences, P0 sums), h- =
// (u_x, u_y, bubble sums, P0 differences); RT0 differences (+) and sums (-); the RT0 basis U is
// orthonormal per sector (kernel vector first), so every table is block diagonal:
//   a+ = gp h+, a- = gm h-;  s~+ = up d - kp a+[3..5],  s~- = um s - km a-[5..7];
//   z~ = S~_v^{-1} s~ (per vertex, mixes the sectors);  z+ = a+ + cp (P0 sums) - qp z~+,
//   z- = a- - qm z~-;  RT0: y+ = up^T z~+, y- = um^T z~-;  slots a = (-) + (+), b = (-) - (+)
//   (P0: a = (+) + (-), b = (+) - (-)), times the natural weights.
struct HvInteriorPM {
    double gp[6][6], gm[8][8];
    double kp[3][3], km[3][3];
    double up[3][3], um[3][3];     // [basis j][pair q]
    double qp[6][3], qm[8][3];
    double pinv;
};
struct HvInterior {
    HvInteriorPM pm;
};
struct HetVankaTabs {
    const double* cls;            // device: MG_NCLASS x MG_HV_CLS
    const double* sinv;           // device: MG_HV_NSINV planes of (n+1) x pitch
};

struct VankaParams {
    LevelParams L;
    HetVankaTabs hv;              // heterogeneous K only (cls == nullptr otherwise)
    double gpT[9][9];            // transposed: gpT[c][a] = G+[a][c] (column-outer FMA loops read pairs)
    double gmT[11][11];
    const double* gbnd;          // device: MG_NCLASS x 20 x 20 (weighted, deflated), row major
    double omega;
    double* bcorr;               // device scratch of the warp-marching sweep: the 20 patch outputs of the 4n
                                 // boundary vertices ([20][4n], vanka_bnd_kernel), read instead of recomputed
};

struct DispParams {               // 8-DoF displacement Vanka (F_u^{-1} of BSR)
    double upT[3][3];             // + block: bubble diffs (transposed, [c][a])
    double umT[5][5];             // - block: u_x, u_y, bubble sums (transposed)
    const double* ubnd;           // device: MG_NCLASS x 8 x 8
};

// host tables of one level (mg_setup.cpp)
struct HostLevelTables {
    int n;
    double h;
    LevelParams L;                // device pointers left null
    double vanka[MG_NCLASS][MG_PSLOTS * MG_PSLOTS];
    double gp[9][9], gm[11][11];
    double disp[MG_NCLASS][MG_USLOTS * MG_USLOTS];
    double up[3][3], um[5][5];
};

struct Material {
    double lambda, mu, K, tau, alpha, inv_M, mu_f;
    int exact = 0;                // 1: exact-integration lambda term (eq. block_form), 0: A^RQ
};

// mg_setup.cpp
int host_level_tables(int n, const Material& m, HostLevelTables* t, char* err, int errlen);
// condensed heterogeneous-Vanka tables of one level (see HetVankaTabs): cls[MG_NCLASS][MG_HV_CLS],
// W[MG_NCLASS][MG_HV_W] (tau mu_f h^2 M_w1 of triangle (cell a-1+tx, b-1+ty, shape sh), tri = 4 sh + 2 ty + tx,
// mapped onto the 6 RT0 patch slots), C[MG_NCLASS][36] (K_ry G_def K_yr)
int host_hv_tables(int n, const Material& m, double* cls, double* W, double* C, HvInteriorPM* pm, char* err,
                   int errlen);
// dense coarsest operator: Ginv (N x N, column major: G[col*N + row]) of the deflated inverse and
// the slot offsets (k*(n+1)*pitch + j*pitch + i) of the N active unknowns.  kinv: nullptr (scalar)
// or 2 x n x n [shape][j][i].
int host_coarse_inverse(int n, int pitch, const Material& m, const double* kinv, double* Ginv,
                        int64_t* slots, int* N, char* err, int errlen);
int64_t n_active_of(int n);

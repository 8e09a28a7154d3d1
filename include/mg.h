/*
 * mg.h -- C ABI of the B200 (sm_100a) monolithic multigrid hot path for the
 * reduced-quadrature P1+bubble / RT0 / P0 three-field Biot discretisation of
 * arXiv 2107.04060 ("Monolithic multigrid for a reduced-quadrature
 * discretization of poroelasticity").  Citations "PAPER.md:N" are lines of the
 * paper's LaTeX source; "SURVEY" is /root/repo/SURVEY.md; "reading Ak" is the
 * numbered reading in DESIGN.md.
 *
 * PROBLEM (eq. block_form_rq).  One
 * backward-Euler step of the three-field Biot model on the unit square, n x n
 * cells each cut top-left -> bottom-right, u = 0 and w.n = 0 on
 * the whole boundary:
 *
 *   A^RQ [u; w; p] = b,   A^RQ = [[A_u^RQ, 0, alpha B_u^T],
 *                                 [0, tau M_w, tau B_w^T],
 *                                 [alpha B_u, tau B_w, -(1/M) M_p]],
 *   A_u^RQ = 2 mu A_eps + lambda B_u^T M_p^{-1} B_u,
 *   M_w = (mu_f K^{-1} w, r),  K scalar or per triangle.
 *
 * VECTOR LAYOUT (every x, b, r, e below).  A level-l vector is 10 fp64 planes;
 * plane k holds (n_l + 1) rows of mg_pitch(ctx, l) doubles; entry (k, j, i)
 * is at k*(n_l+1)*pitch + j*pitch + i, 0 <= i, j <= n_l, x = i h, y = j h.
 * Index (i, j) owns vertex (i,j), the edges H(i,j) = (i,j)-(i+1,j) [normal +y],
 * V(i,j) = (i,j)-(i,j+1) [normal +x], D(i,j) = (i+1,j)-(i,j+1) [normal
 * (1,1)/sqrt2] and the triangles LL = [(i,j),(i+1,j),(i,j+1)] and
 * UR = [(i+1,j),(i+1,j+1),(i,j+1)] of cell (i,j)  (readings A1, A2):
 *
 *   plane 0/1  u_x / u_y (P1)          active iff 0<i<n, 0<j<n
 *   plane 2    face bubble on H(i,j)   active iff i<n, 0<j<n
 *   plane 3    face bubble on V(i,j)   active iff 0<i<n, j<n
 *   plane 4    face bubble on D(i,j)   active iff i<n, j<n
 *   plane 5-7  RT0 on H / V / D        as planes 2-4
 *   plane 8/9  P0 on LL / UR           active iff i<n, j<n
 *
 * Bubbles are 4 lambda_a lambda_b n_e (normal trace 1 at the midpoint), RT0
 * functions have normal trace 1 (reading A1).  Inactive and padding slots are
 * 0 on input and are written as 0 on output.  The number of active unknowns is
 * 10 n^2 - 8 n + 2 (the paper counts 10 n^2 + 8 n + 2 slots, tab:mgtime
 * PAPER.md:1100-1104).
 *
 * HIERARCHY.  Level l has n_l = n / 2^l cells per side, l = 0 .. levels-1;
 * operators are rediscretised on every level; level
 * levels-1 is solved exactly.  A per-triangle K field is
 * coarsened by averaging K^{-1} over the four children (reading A11).
 *
 * OWNERSHIP.  The caller owns every pointer passed in (x, b, r, e: DEVICE
 * pointers to mg_vec_len(ctx, level) doubles, 16-byte aligned -- the kernels
 * move column pairs as double2 and the TMA descriptors need 16-byte global
 * addresses; a misaligned pointer is rejected with MG_EINVAL; *_host: host
 * pointers) and every stream.  The context owns all per-level tables, the
 * level >= 1 work vectors, one scratch vector per level, the K^{-1} pyramid
 * and the coarsest inverse; they are allocated in mg_setup through the
 * allocator installed with mg_set_allocator (default cudaMalloc) and released
 * by mg_free.  The allocator in force at mg_setup is recorded in the context and
 * used for all of its later allocations (FGMRES work space, history) and frees.  A context must not be used from two host threads or two
 * streams at the same time.
 *
 * ERRORS.  Every int function returns MG_OK (0) on success, a negative code on
 * failure (message in mg_last_error(), thread local), or a positive status
 * (MG_NOTCONV, MG_DIVERGED) from mg_solve.  Nothing aborts or throws across
 * the ABI.  Device work is enqueued asynchronously on the given stream unless
 * stated otherwise; functions returning host data synchronise that stream.
 */
#ifndef MG_H
#define MG_H

#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MG_OK        0
#define MG_NOTCONV   1   /* mg_solve: max_cycles reached; history filled              */
#define MG_DIVERGED  2   /* mg_solve: ||r_k|| > 1e8 ||r_0|| or non-finite  */
#define MG_EINVAL   (-1) /* bad argument: see mg_last_error()                           */
#define MG_ECUDA    (-2) /* CUDA runtime / driver error                                 */
#define MG_ENOMEM   (-3) /* allocation failed                                           */

#define MG_VANKA 0       /* additive Vanka, 20-DoF vertex patches    */
#define MG_BSR   1       /* inexact Braess-Sarazin                   */
#define MG_BSR_EXACT 2   /* exact Braess-Sarazin: S dp = g solved exactly */

#define MG_RQ    0       /* reduced quadrature of lambda (div u, div v): A^RQ, eq. block_form_rq */
#define MG_EXACT 1       /* exact integration: A of eq. block_form (tab:naive) */

typedef struct mg_ctx mg_ctx;

typedef struct {
    int32_t n;              /* finest cells per side; h = 1/n.  n divisible by 2^(levels-1)  */
    const double* K_field;  /* NULL -> scalar K of mg_setup.  Else DEVICE pointer to 2 x n x n
                               doubles [shape (0 = LL, 1 = UR)][j][i], the permeability of each
                               triangle (> 0, finite); copied during mg_setup                     */
    double inv_M;           /* 1/M > 0 (Biot modulus); 0 is rejected (MG_EINVAL):
                               the exactly deflated patch and coarsest solves divide by the
                               constant-pressure eigenvalue gamma = (1/M) h^2/2 (reading A9).
                               BASELINE configs run 1/M = 1 (reading A5), not SURVEY 8(b)'s
                               proposed 1e-6: at 1e-6 the rediscretised V(1,1) cycle diverges
                               (factor ~ 1/gamma growth, tests/golden/a5_invM_scan.json).        */
    double mu_f;            /* fluid viscosity > 0; 1                            */
    int32_t quadrature;     /* MG_RQ (0, the paper's method) or MG_EXACT: lambda (div u, div v)
                               integrated exactly (eq. block_form), the "solver-incompatible"
                               operator of PAPER.md:169-198.  MG_EXACT contexts run the 2-D tile
                               kernels on every level (the row-marching kernels are RQ only)     */
} mg_grid;

typedef struct {
    int32_t nu1, nu2;       /* pre / post relaxation sweeps (BASELINE: 1, 1)                 */
    int32_t relax;          /* MG_VANKA, MG_BSR or MG_BSR_EXACT (n <= 1024)                   */
    double  omega;          /* outer damping                              */
    double  omega_J;        /* BSR: weight of the Jacobi sweeps on S          */
    int32_t jacobi_sweeps;  /* BSR: sweeps on S from dp = 0 (BASELINE: 3; paper: 1)          */
} mg_cycle_opts;

/* Device memory hooks: alloc(bytes, user) -> device pointer (16-byte aligned) or NULL;
 * free(ptr, user).  Installed for the contexts created afterwards; each context keeps the pair it
 * was created with until mg_free.  NULL, NULL restores cudaMalloc/cudaFree. */
typedef void* (*mg_alloc_fn)(size_t bytes, void* user);
typedef void  (*mg_free_fn)(void* ptr, void* user);
void mg_set_allocator(mg_alloc_fn alloc, mg_free_fn free_, void* user);

/* Build the hierarchy (host fp64 tables: stencils, deflated patch inverses, coarsest inverse;
 * PAPER.md:477-484, 572-590, 945) and upload it to the current device.  Synchronous.
 * lambda >= 0, mu > 0, K > 0 (ignored when grid->K_field != NULL), tau > 0, alpha finite,
 * 1 <= levels, n_{levels-1} = n / 2^(levels-1) >= 2.  The dense coarsest solve needs
 * n_{levels-1} <= 20; a context with a larger coarsest level supports the per-level operations
 * only (mg_coarse_solve / mg_cycle / mg_solve then return MG_EINVAL).  The dense inverse is formed
 * on the host in long double, O(m^3) for m ~ 10 n_c^2 unknowns: milliseconds at n_c = 4 (every
 * BASELINE config), about a second at the paper's n_c = 8, a minute at n_c = 16.
 * Errors: MG_EINVAL, MG_ECUDA, MG_ENOMEM. */
int mg_setup(const mg_grid* grid, double lambda, double mu, double K, double tau, double alpha,
             int32_t levels, mg_ctx** out);
void mg_free(mg_ctx* ctx);

int32_t mg_levels (const mg_ctx* ctx);
int32_t mg_level_n(const mg_ctx* ctx, int32_t level);  /* n_l, or -1 if level out of range   */
int32_t mg_pitch  (const mg_ctx* ctx, int32_t level);  /* row pitch in doubles (multiple of 32) */
int64_t mg_vec_len(const mg_ctx* ctx, int32_t level);  /* 10 (n_l+1) pitch                     */
int64_t mg_n_active(const mg_ctx* ctx, int32_t level); /* 10 n_l^2 - 8 n_l + 2                 */

/* r = b - A_l x on the active slots (eq. block_form_rq), r = 0 elsewhere.  r may be NULL (norm
 * only).  norm2_dev: NULL or a DEVICE double receiving ||r||_2^2 over the active slots
 * (deterministic order).  r must not alias x or b. */
int mg_residual(mg_ctx* ctx, int32_t level, const double* x, const double* b, double* r,
                double* norm2_dev, cudaStream_t s);

/* `sweeps` additive Vanka sweeps on level l:
 *   x <- x + omega sum_v V_v^T D_v (V_v A_l V_v^T)^{-1} V_v (b - A_l x),
 * one patch per vertex, truncated to active DoFs (reading A8), natural weights D (1, 1/2, 1/3;
 * PAPER.md:586-587), exactly deflated patch solves (reading A9).  In place on x; the context's
 * level-l scratch vector is used for the out-of-place sweep, so an odd sweep count ends with one
 * device copy back into x (the cycle itself ping-pongs without copies).  Constant K only
 * (reading A20). */
int mg_relax_vanka(mg_ctx* ctx, int32_t level, double* x, const double* b, double omega,
                   int32_t sweeps, cudaStream_t s);

/* One inexact Braess-Sarazin relaxation on level l (App. D-E):
 *   r = b - A x;  z_u = F_u^{-1} r_u (8-DoF displacement Vanka, weights 1, 1/2);
 *   z_w = (tau D_w)^{-1} r_w;  g = alpha B_u z_u + tau B_w z_w - r_p;
 *   dp = jacobi_sweeps weighted-Jacobi sweeps (weight omega_J) on
 *        S dp = g,  S = (1/M + alpha^2/(lambda + mu)) M_p + tau B_w D_w^{-1} B_w^T, from dp = 0;
 *   du = F_u^{-1}(r_u - alpha B_u^T dp);  dw = (tau D_w)^{-1}(r_w - tau B_w^T dp);
 *   x += omega (du, dw, dp).   In place on x.  `sweeps` repetitions. */
int mg_relax_bsr(mg_ctx* ctx, int32_t level, double* x, const double* b, double omega,
                 double omega_J, int32_t jacobi_sweeps, int32_t sweeps, cudaStream_t s);

/* `sweeps` exact Braess-Sarazin relaxations on level l: as mg_relax_bsr with
 * the Jacobi sweeps replaced by the exact solution of S dp = g (eq. bsr_p), computed on the device
 * by Jacobi-preconditioned conjugate gradients to 1e-14 in the D_S^{-1} norm (at most 24 n + 64
 * iterations).  Level n <= 1024 (a full S solve per relaxation is the cost the paper avoids with
 * inexact BSR).  Work space allocated on first use.  In place on x.  cg_iters_out: NULL or
 * receives the CG iterations of the last S solve (the stream is then synchronised, and MG_NOTCONV is
 * returned if that solve stopped at the iteration cap instead of the tolerance). */
int mg_relax_bsr_exact(mg_ctx* ctx, int32_t level, double* x, const double* b, double omega, int32_t sweeps,
                       int32_t* cg_iters_out, cudaStream_t s);

/* b_coarse = P^T r_fine between levels fine_level and fine_level+1 (R = P^T, PAPER.md:484;
 * P_u divergence preserving PAPER.md:510-566, P_w / P_p canonical).  Overwrites b_coarse. */
int mg_restrict(mg_ctx* ctx, int32_t fine_level, const double* r_fine, double* b_coarse,
                cudaStream_t s);
/* x_fine += P e_coarse (same P).  In place on x_fine. */
int mg_prolong(mg_ctx* ctx, int32_t fine_level, const double* e_coarse, double* x_fine,
               cudaStream_t s);
/* The fused production variants the V-cycle launches, exposed for testing at full size:
 * mg_residual_restrict: b_coarse = P^T (b - A_l x) on levels l -> l+1 in one pass (row-marching TMA
 * kernel on levels with n >= 512, scalar K); mg_prolong_relax_vanka: x <- one Vanka sweep of
 * x + P e_coarse (the first post-smoothing sweep with the coarse-grid correction fused in,
 * PAPER.md:471-476; producer warps add P e to each TMA row of x) -- in place on x (level-l scratch
 * used). Constant K; levels 0 .. levels-2. */
int mg_residual_restrict(mg_ctx* ctx, int32_t fine_level, const double* x, const double* b, double* b_coarse,
                         cudaStream_t s);
int mg_prolong_relax_vanka(mg_ctx* ctx, int32_t level, double* x, const double* e_coarse, const double* b,
                           double omega, cudaStream_t s);

/* x = A_L^{-1} b on the coarsest level L = levels-1 (dense deflated inverse, reading A9). */
int mg_coarse_solve(mg_ctx* ctx, const double* b, double* x, cudaStream_t s);

/* One V(nu1, nu2) cycle on level 0 (recursed), in place on x.
 * res_norm_host: NULL or receives ||b - A_0 x||_2 after the cycle (then the stream is
 * synchronised).  The level sequence is captured once into a CUDA graph per (x, b, opts) and
 * replayed. */
int mg_cycle(mg_ctx* ctx, double* x, const double* b, const mg_cycle_opts* opts,
             double* res_norm_host, cudaStream_t s);

/* One V-cycle without any host synchronisation (the building block of mg_solve and of the
 * benchmark).  in_norm2_dev: NULL or a DEVICE double receiving ||b - A_0 x_in||_2^2 for the INPUT
 * x, fused into the level-0 pre-relaxation (no extra pass; deterministic order).  Graph-cached
 * like mg_cycle. */
int mg_cycle_async(mg_ctx* ctx, double* x, const double* b, const mg_cycle_opts* opts,
                   double* in_norm2_dev, cudaStream_t s);

/* Kernel-class tracing.  enable != 0: cycles captured afterwards record CUDA events between the
 * level-0 phases; mg_timing (synchronises the stream of the last cycle) returns the elapsed ms of
 * the most recent cycle per phase: [0] level-0 pre-relaxation, [1] level-0 residual+restriction,
 * [2] all coarser levels including the coarsest solve, [3] level-0 prolongation, [4] level-0
 * post-relaxation.  Returns MG_EINVAL if no traced cycle ran. */
int mg_set_timing(mg_ctx* ctx, int32_t enable);
/* Number of kernel nodes of the most recently captured cycle graph (all of them libmg kernels). */
int32_t mg_cycle_kernels(const mg_ctx* ctx);
int mg_timing(mg_ctx* ctx, float* ms5);
/* Per-level intervals of the most recent traced cycle, in execution order: for l = 0 .. L-2
 * [pre-relaxation(l), residual+restriction(l)], then the coarsest solve, then for l = L-2 .. 0
 * [prolongation(l), post-relaxation(l)] -- 4 (L-1) + 1 values.  Returns the count (>= 0) or a
 * negative error (cap too small, no traced cycle). */
int mg_timing_levels(mg_ctx* ctx, float* ms, int32_t cap);

/* Stationary iteration of V-cycles from the given x until ||r_k|| <= rtol ||r_0|| or
 * max_cycles.  history_host: NULL or max_cycles+1 doubles, history[k] = ||b - A x_k||_2
 * (history[0] for the input x).  *n_cycles = cycles done.  Returns MG_OK, MG_NOTCONV or
 * MG_DIVERGED (or an error).  Synchronous. */
int mg_solve(mg_ctx* ctx, double* x, const double* b, const mg_cycle_opts* opts, double rtol,
             int32_t max_cycles, double* history_host, int32_t* n_cycles, cudaStream_t s);

/* Flexible GMRES(restart) on level 0, right-preconditioned by one V(nu1, nu2) cycle from a zero
 * initial guess per iteration -- the paper's solver for every timed experiment (PAPER.md:922,
 * SURVEY 8(f) rank 1).  Arnoldi by classical Gram-Schmidt with a second pass when the first one
 * cancelled the vector by more than 10x (the DGKS test with eta = 0.1; one pass then leaves the new
 * vector orthogonal to ~10 u, enough for a basis of at most 31 vectors), fused into passes over memory (dots;
 * first update + second dots; second update + norm) on an unscaled basis whose scales are kept on
 * the host; deterministic device dot products; Givens rotations on the host.  Starts from the given x, stops at estimated
 * ||r_k|| <= rtol ||r_0|| or max_iters.  history_host: NULL or max_iters+1 doubles: history[0] =
 * ||b - A x_0||, history[i] = the residual-norm estimate after i iterations (equal to
 * ||b - A x_i|| in exact arithmetic).  Work space: 2 restart + 2 level-0 vectors (allocated on
 * first use; 1 <= restart <= 31).  Returns MG_OK or MG_NOTCONV.  Synchronous. */
int mg_fgmres(mg_ctx* ctx, double* x, const double* b, const mg_cycle_opts* opts, double rtol,
              int32_t max_iters, int32_t restart, double* history_host, int32_t* n_iters, cudaStream_t s);

/* Backward-Euler time stepping.  At step m the system matrix is the same
 * A^RQ (tau is the step size of mg_setup) and the previous step enters the right-hand side only
 * through the pressure rows, eq. discrete3 scaled by -1 with
 *   (f_hat, q) = tau (f, q) + (1/M)(p^{m-1}, q) + (alpha div u^{m-1}, q):
 *   b^m = b_load^m + [0; 0; -(1/M) M_p p^{m-1} + alpha B_u u^{m-1}],
 * b_load^m = [(rho g, v); tau (rho_f g, r); -tau (f^m, q)] being the caller's loads at t_m.
 * mg_step_rhs writes b^m to b_out (DEVICE, level-0 layout; may alias b_load, not x_prev).
 * mg_time_step forms b^m from x = x^{m-1} and b_load, then runs mg_fgmres from x as the initial
 * guess, leaving x^m in x (work vector allocated on first use).  Returns as mg_fgmres. */
int mg_step_rhs(mg_ctx* ctx, const double* x_prev, const double* b_load, double* b_out, cudaStream_t s);
int mg_time_step(mg_ctx* ctx, double* x, const double* b_load, const mg_cycle_opts* opts, double rtol,
                 int32_t max_iters, int32_t restart, double* history_host, int32_t* n_iters, cudaStream_t s);

/* mg_solve with HOST vectors in the unpadded layout [10][n+1][n+1] (the end-to-end path):
 * b_host is copied to the device, x starts at x_host, the solution is copied back to x_host.
 * Host buffers should be pinned for full copy bandwidth.  Synchronous. */
int mg_solve_host(mg_ctx* ctx, double* x_host, const double* b_host, const mg_cycle_opts* opts,
                  double rtol, int32_t max_cycles, double* history_host, int32_t* n_cycles,
                  cudaStream_t s);

const char* mg_last_error(void);

/* ---- host-only diagnostics (no GPU needed; used by the CPU test-suite) -------------------
 * Fill the level tables mg_setup would upload, for a level of n cells, scalar K:
 *   stencil_coef[141]  merged stencil coefficients of A^RQ without M_w (mg_tables.h order)
 *   ww[18]             tau mu_f K^{-1} h^2 (M_w1)_{shape,e,e'}
 *   vanka[9*400]       per vertex class c = cx + 3 cy (cx: 0 interior, 1 at i=0, 2 at i=n),
 *                      the weighted deflated patch inverse D_v K_v^{-1} (20x20, slot order of
 *                      DESIGN.md section 4), rows/cols of inactive slots 0
 *   disp[9*64]         same for the 8-DoF displacement patches of BSR: D_v (A_u^RQ)_v^{-1}
 * Returns MG_OK or MG_EINVAL. */
int mg_host_level_tables(int32_t n, double lambda, double mu, double K, double tau, double alpha,
                         double inv_M, double mu_f, double* stencil_coef, double* ww,
                         double* vanka, double* disp);

#ifdef __cplusplus
}
#endif
#endif /* MG_H */

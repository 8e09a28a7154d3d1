// Kernel declarations and launch helpers (sm_100a, fp64).  See mg_kernels.cu.
#pragma once
#include <cuda_runtime.h>
#include "mg_internal.h"

// Deterministic norm accumulation: one partial per block, the last block sums them in index order.
struct NormSink {
    double* out;          // device double receiving sum of squares (nullptr: no norm)
    double* partials;     // >= number of blocks of the launch
    unsigned* counter;    // zero-initialised; reset by the last block
    SolveState* state;    // non-null: append the norm to state->hist and decide state->stop
};
void kernels_init();
// preferred L1 / shared carveout (percent) of every kernel, applied by kernels_init (-1: driver default)
void set_carveout(int pct);

// up to 8 vector pointers for the FGMRES multi-vector kernels
struct VecPtrs {
    const double* p[8];
};

// Gram-Schmidt pass over up to GS_KMAX basis vectors in one sweep of memory (vec_gs_kernel):
//   mode 0: out[q] = <w, V_q> (q < k), out[k] = <w, w>
//   mode 1: o = w - sum_q c_q V_q (written to wo, may alias w), out[q] = <o, V_q>, out[k] = <o, o>
// (c_q is scaled by sc[q] when sc != nullptr)
//   mode 2: o = w - sum_q c_q V_q (written to wo), out[0] = <o, o>
//   mode 3: o = w - sum_q c_q V_q (written to wo), no reduction
// Reductions are deterministic (per-block partials summed in block order by the last block).
constexpr int GS_KMAX = 32;
struct GsPtrs {
    const double* p[GS_KMAX];
};
cudaError_t launch_gs(int mode, const double* w, double* wo, const GsPtrs& V, int k, const double* c,
                      const double* sc, int64_t len, double* partials, unsigned* counter, double* out, cudaStream_t s);
int gs_partials_needed();

// The bottom of a Vanka V-cycle in one grid-wide kernel (bottom_kernel, cooperative launch): levels
// lb .. lb + nl - 1 and the coarsest lb + nl.  Index l below is relative to lb.
constexpr int BOT_MAXL = 6;
struct BottomArgs {
    int nl, nu1, nu2;
    VankaParams vp[BOT_MAXL];          // omega set
    double* x[BOT_MAXL + 1];           // per level: iterate buffer (context-owned Lv.x)
    double* t[BOT_MAXL];               // scratch
    double* b[BOT_MAXL + 1];           // right-hand sides (b[l+1] written by the restriction)
    int pitch[BOT_MAXL + 1];
    int N;                             // coarsest dense inverse (column major) and slots
    const double* G;
    const int64_t* slots;
    const int* stop;
};
cudaError_t launch_bottom(const BottomArgs& A, cudaStream_t s);

// All launchers return cudaGetLastError() of the launch.
cudaError_t launch_residual(const LevelParams& L, const double* x, const double* b, double* r,
                            NormSink norm, cudaStream_t s);
// y = A x (masked), the FGMRES operator application
cudaError_t launch_apply(const LevelParams& L, const double* x, double* y, NormSink norm, cudaStream_t s);
// FGMRES vector kernels (deterministic): out[q] = <w, V.p[q]>, q < k <= 8;  w -= sum c[q] V.p[q];  y = sc x
cudaError_t launch_dots(const double* w, const VecPtrs& V, int k, int64_t len, double* partials, unsigned* counter,
                        double* out, cudaStream_t s);
cudaError_t launch_update(double* w, const VecPtrs& V, int k, const double* c, int64_t len, cudaStream_t s);
cudaError_t launch_scale(double* y, const double* x, double sc, int64_t len, cudaStream_t s);
// dst = src (len doubles), skipped when *stop != 0 (mg_solve's flag)
cudaError_t launch_copy(double* dst, const double* src, int64_t len, const int* stop, cudaStream_t s);
int dot_partials_needed();
// exact BSR: S dp = g by Jacobi-PCG on the P0 planes (g is overwritten by the residual), up to
// max_iters iterations, stopping (device-side flag) at r.z <= st[4] r0.z0; st: 8 device doubles
// (st[4] = tol^2 set by the caller, st[6] = iterations done)
cudaError_t launch_cg_exact(const LevelParams& L, const double* tab, double* g, double* dp, double* z, double* p,
                            double* q, double* partials, unsigned* counter, double* st, int max_iters,
                            cudaStream_t s);
int cg_partials_needed(int n);
// backward-Euler history term added to the pressure rows of b (x = the previous step's iterate)
cudaError_t launch_step_rhs(const LevelParams& L, double inv_M, double alpha, const double* x, double* b,
                            cudaStream_t s);
// per-vertex S_v^{-1} planes of the heterogeneous Vanka patches (setup; L.kinv_field set)
cudaError_t launch_hv_sinv(const LevelParams& L, const double* W, const double* C, double* sinv, cudaStream_t s);
// P.hv.cls != nullptr: heterogeneous-K sweep (condensed patch solves, 2-D tiles on every level)
// E != nullptr (levels with n <= small_tile_n, MG_SMALL_DIET): relax x + P e_H (prolongation fused in)
cudaError_t launch_vanka(const VankaParams& P, const double* x, const double* b, double* xout,
                         bool x_zero, NormSink norm, cudaStream_t s, const HvInterior* Ti = nullptr,
                         const ProlSrc* E = nullptr);
int small_tile_n();
int small_diet();
// row-marching TMA variant of the same sweep (identical arithmetic); the production kernel
// E != nullptr: relax x + P e_H (prolongation of the coarse iterate E->e fused into the sweep)
cudaError_t launch_vanka_march2(const VankaParams& P, const double* x, const double* b, double* xout,
                                bool x_zero, NormSink norm, cudaStream_t s, const ProlSrc* E = nullptr);
int blocks_vanka_march2(int n);
// heterogeneous-K warp-marching sweep (vanka_hwarp_kernel; bitwise vanka_het_kernel) and its boundary kernel
cudaError_t launch_vanka_hwarp(const VankaParams& P, const HvInterior& Ti, const double* x, const double* b,
                               double* xout, bool x_zero, NormSink norm, cudaStream_t s);
// levels with n >= N run the plain Vanka sweeps through the warp-marching kernel (0: never)
void set_warp_min_n(int N);
// the fused-prolongation post-sweep through the warp-marching kernel as well (1) or the CTA kernel (0)
void set_warp_prol(int on);
// boundary-vertex patches of the warp sweep: 1 precomputed by vanka_bnd_kernel, 0 inline (out-of-line call)
void set_warp_bk(int on);
// BSR stage B through the warp-marching kernel on the levels with n >= MG_WARP_MIN_N (1) or the CTA kernel (0)
void set_warp_bsr(int on);
int blocks_residual_march(int n);
// levels with n <= N use small 2-D tiles (8 x 4 owners / 4 x 2 coarse indices) in the single-pass
// kernels: more, shorter CTAs for the latency-bound coarse levels (process-wide knob)
void set_small_tile_n(int N);
// small-tile sweeps with every global read in the first round trip (vanka_small_kernel) or vanka_kernel
void set_small_diet(int on);
// programmatic dependent launch of every kernel (1, default) or plain stream order (0)
void set_pdl(int on);
// fused-prolongation sweep variant: 1 warp-specialised with setmaxnreg (default), 0 the 6-warp kernel
void set_prol_ws(int on);
// residual / operator application on levels with n >= N through the marching kernel (scalar K)
void set_resid_march_n(int N);
// per-level Jacobi table (tau / D_w per RT0 edge, 1 / diag S per triangle; 5 planes) and the sweep using it
cudaError_t launch_jtable(const LevelParams& L, double* tab, cudaStream_t s);
// two table sweeps in one launch (bitwise two launch_bsr_jacobi_t)
cudaError_t launch_bsr_jacobi2_t(const LevelParams& L, double omega_J, const double* g, const double* tab,
                                 const double* dp_in, double* dp_out, cudaStream_t s);
cudaError_t launch_bsr_jacobi_t(const LevelParams& L, double omega_J, const double* g, const double* tab,
                                const double* dp_in, double* dp_out, cudaStream_t s);
// two Jacobi sweeps in one launch (same arithmetic as two launch_bsr_jacobi)
// row-marching TMA variants of the two BSR stages (same arithmetic as launch_bsr_a / launch_bsr_b)
cudaError_t launch_bsr_a_march(const LevelParams& L, const DispParams& U, double omJ, const double* x, const double* b,
                               double* g, double* dp, NormSink S, bool x_zero, cudaStream_t s, const double* jtab,
                               double* rs = nullptr);
// rs != nullptr (and not x_zero): stage A stores r_u, r_w (8 planes) there and stage B reads them instead of
// evaluating the residual a second time (same values: bitwise the two-residual path)
cudaError_t launch_bsr_b_march(const LevelParams& L, const DispParams& U, double omega, const double* x,
                               const double* b, const double* dp, double* xo, bool x_zero, cudaStream_t s,
                               const double* rs = nullptr);
// row-marching TMA variant of the fused residual + restriction (mode 1)
cudaError_t launch_restrict_march(const LevelParams& Lf, int n_coarse, int pitch_coarse, const double* x_fine,
                                  const double* b_fine, double* b_coarse, cudaStream_t s);
// mode 0: r_fine given (x_fine, b_fine unused); 1: r = b - A x fused; 2: x == 0 (r = b)
cudaError_t launch_restrict(const LevelParams& Lf, int n_coarse, int pitch_coarse, int mode,
                            const double* x_fine, const double* b_or_r_fine, double* b_coarse,
                            cudaStream_t s);
cudaError_t launch_prolong(int n_fine, int pitch_fine, int n_coarse, int pitch_coarse,
                           const double* e_coarse, double* x_fine, const int* stop, cudaStream_t s);
cudaError_t launch_coarse(int N, const double* Ginv, const int64_t* slots, const double* b, double* x,
                          const int* stop, cudaStream_t s);
// BSR
cudaError_t launch_bsr_a(const LevelParams& L, const DispParams& U, double omega_J, const double* x,
                         const double* b, double* g, double* dp, NormSink norm, bool x_zero,
                         cudaStream_t s);
cudaError_t launch_bsr_jacobi(const LevelParams& L, double omega_J, const double* g, const double* dp_in,
                              double* dp_out, cudaStream_t s);
// jg != nullptr: the last two table Jacobi sweeps run inside the kernel (dp holds the sweep before them; g = jg,
// table = jtab, weight omJ): bitwise two launch_bsr_jacobi_t + the plain stage B
cudaError_t launch_bsr_b(const LevelParams& L, const DispParams& U, double omega, const double* x,
                         const double* b, const double* dp, double* xout, bool x_zero, cudaStream_t s,
                         const double* jg = nullptr, const double* jtab = nullptr, double omJ = 0.0);
cudaError_t launch_kinv_coarsen(int n_fine, int pitch_fine, const double* kf, int pitch_coarse, double* kc,
                                cudaStream_t s);
cudaError_t launch_kinv_from_K(int n, int pitch, const double* K, double* kinv, cudaStream_t s);
int blocks_residual(int n);
int blocks_vanka(int n);
int blocks_bsr(int n);

// fp64 sm_100a kernels of the monolithic multigrid V-cycle for the RQ Biot operator
// (arXiv 2107.04060).  Every kernel is matrix free: the operator stencil and the prolongation
// weights come from mg_tables.h (generated geometry) and the per-level coefficients from the
// LevelParams passed by value (constant bank).  Layout: include/mg.h.
//
//   residual_kernel     r = b - A^RQ x                      (eq. block_form_rq)
//   vanka_kernel        fused additive Vanka sweep
//   restrict_kernel     b_H = P^T (b - A x), fused
//   prolong_kernel      x += P e_H
//   coarse_kernel       dense deflated coarsest solve       (reading A9)
//   bsr_a/jacobi/b      inexact Braess-Sarazin stages
// and their production forms on the big levels (same arithmetic, bitwise-tested against the tile kernels):
//   vanka_warp_kernel / vanka_hwarp_kernel (+ vanka_bnd2_kernel)   warp-marching sweeps, scalar K / K field
//   restrict_march_kernel, residual_march_kernel                   row-marching TMA rings (K^{-1} ring with a K field)
//   bsr_a_march_kernel, bsr_jacobi2_t_kernel, bsr_b_march_kernel   marching BSR stages; stage B reads stage A's residual
//   prolong_planes_kernel                                          plane-split prolongation
//
// Tiles: a CTA owns TX x TY grid indices (each index owns 10 DoFs) and recomputes the residual
// on a halo ring instead of exchanging it, so every sweep reads x and b once and writes x once
// (owner computes; no atomics; deterministic).  The Vanka sweep is out of place (x -> xout):
// neighbouring CTAs read x in their halos.
#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <cuda.h>
#include <cooperative_groups.h>

#include "mg_kernels.cuh"
#include "mg_tables.h"

// displacement DoFs (q = 0..8: P1 x/y of the 3 vertices, 3 bubbles) of triangle `sh` of a cell as
// (dx, dy, plane) -- mg_tables.h LOCAL_DOF (generated geometry), copied to the constant bank by
// kernels_init
__constant__ int c_local_dof[2][9][3];

namespace {

// Programmatic dependent launch (sm_90+): every kernel waits for the completion (and memory) of the
// grid it depends on before touching memory, so the host may launch it with programmatic stream
// serialization -- the next grid is scheduled while the previous one drains, which removes most of
// the launch gap between the short kernels of the coarse levels.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// allow the dependent grid to be scheduled: once every CTA of this grid has started, the next
// grid's CTAs fill the SMs this grid's tail frees (they block in pdl_wait until it completes)
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// bit p set <=> is_active(p, i, j, n), for all ten planes at once
__device__ __forceinline__ unsigned active_mask(int i, int j, int n) {
    if (i < 0 || j < 0 || i > n || j > n) return 0u;
    const bool ii = i > 0 && i < n, ij = j > 0 && j < n, li = i < n, lj = j < n;
    return (ii && ij ? 0x003u : 0u) | (li && ij ? 0x024u : 0u) | (ii && lj ? 0x048u : 0u) |
           (li && lj ? 0x390u : 0u);
}

// register slot of the coarse value e_H(I + dI, J + dJ, pl) in the fused prolongation: planes 0-4
// use 13 slots, planes 5-9 use 7 (the union over both fine-row parities of MG_PROLONG's operands)
__host__ __device__ constexpr int pslot(int dI, int dJ, int pl) {
    return pl >= 5 ? (dI == 0 && dJ == 0 ? pl - 5 : (dJ == 1 ? 5 : 6))
                   : (dI == 0 && dJ == 0 ? pl : dI == 0 ? 5 + pl : dJ == 0 ? (pl == 3 ? 10 : 8 + pl) : 11 + pl);
}
static_assert(pslot(0, 1, 2) == 7 && pslot(1, 0, 3) == 10 && pslot(1, 1, 1) == 12 && pslot(1, 0, 6) == 6, "pslot");
__host__ __device__ constexpr int pslot20(int dI, int dJ, int pl) { return pl >= 5 ? 13 + pslot(dI, dJ, pl) : pslot(dI, dJ, pl); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// plane p of index (i, j) is an unknown (not Dirichlet, not outside the mesh; SURVEY 8 layout table).
// Through the ten-plane mask: the unrolled per-plane tests of one index share one mask.
__device__ __forceinline__ bool is_active(int p, int i, int j, int n) { return (active_mask(i, j, n) >> p) & 1u; }


template <int NT>
__device__ __forceinline__ double block_sum(double v) {
    __shared__ double ws[NT / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int k = 0; k < NT / 32; ++k) t += ws[k];
    return t;  // valid in thread 0
}

// one partial per block; the last block to arrive sums the partials in block order
template <int NT>
__device__ void norm_finish(const NormSink& S, double v) {
    const int nb = gridDim.x * gridDim.y;
    const int bid = blockIdx.y * gridDim.x + blockIdx.x;
    double t = block_sum<NT>(v);
    __shared__ unsigned last;
    if (threadIdx.x == 0) {
        S.partials[bid] = t;
        __threadfence();
        unsigned prev = atomicAdd(S.counter, 1u);
        last = (prev == (unsigned)nb - 1u);
    }
    __syncthreads();
    if (last) {
        __threadfence();
        double acc = 0.0;
        for (int k = threadIdx.x; k < nb; k += NT) acc += __ldcg(S.partials + k);
        double tot = block_sum<NT>(acc);
        if (threadIdx.x == 0) {
            if (S.state) {
                SolveState* st = S.state;
                const int k = st->k;
                st->hist[k] = tot;
                const double h0 = k == 0 ? tot : st->hist[0];
                int stop = 0;
                if (!isfinite(tot)) stop = 2;
                else if (k > 0 && tot <= st->rtol2 * h0) stop = 1;
                else if (k > 0 && tot > 1e16 * h0) stop = 2;
                else if (k >= st->maxk) stop = 3;
                st->k = k + 1;
                if (stop) *st->stop = stop;
            } else {
                *S.out = tot;
            }
            *S.counter = 0u;
        }
    }
}

// zero-padded tile load: dst[p][ly][lx] = src(p, j0+ly, i0+lx) for 0 <= i, j <= n, else 0
// global load through the read-only path (NC) or a plain load (coherent with earlier writes of the
// same kernel on this SM: the single-CTA bottom kernel reads what it wrote)
template <bool NC>
__device__ __forceinline__ double gld(const double* p) {
    if (NC) return __ldg(p);
    return __ldcg(p);   // L2: coherent with what other CTAs of this kernel wrote before a grid barrier
}

template <int W, int HT, int NP, bool NC = true, int U = 8>
__device__ __forceinline__ void load_tile(double* __restrict__ dst, const double* __restrict__ src, int i0,
                                          int j0, int n, int pitch, int64_t plane, int p0 = 0, int t0 = -1,
                                          int nt = 0) {
    if (t0 < 0) {
        t0 = threadIdx.x;
        nt = blockDim.x;
    }
    // U elements per thread in flight: all loads of a batch are issued before its shared-memory
    // stores (one element per iteration would serialise ~NP W HT / nt global-load latencies, which
    // is what bounds the latency-bound coarse levels)
    constexpr int TOT = NP * W * HT;
    for (int base = t0; base < TOT; base += U * nt) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int t = base + u * nt;
            v[u] = 0.0;
            if (t < TOT) {
                const int p = t / (W * HT);
                const int rem = t - p * (W * HT);
                const int ly = rem / W;
                const int lx = rem - ly * W;
                const int i = i0 + lx, j = j0 + ly;
                if (i >= 0 && i <= n && j >= 0 && j <= n) v[u] = gld<NC>(src + (p0 + p) * plane + (int64_t)j * pitch + i);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int t = base + u * nt;
            if (t < TOT) dst[t] = v[u];
        }
    }
}

// K^{-1} of triangle `sh` of cell (ci, cj); 0 outside the mesh
template <bool HET>
__device__ __forceinline__ double kinv_at(const LevelParams& L, int ci, int cj, int sh) {
    if (!HET) return L.kinv;
    if (ci < 0 || cj < 0 || ci >= L.n || cj >= L.n) return 0.0;
    return __ldg(L.kinv_field + sh * L.plane + (int64_t)cj * L.pitch + ci);
}

// scale of the per-triangle M_w entries in the residual: L.ww already holds K^{-1} when K is scalar
template <bool HET>
__device__ __forceinline__ double kinv_ww(const LevelParams& L, int ci, int cj, int sh) {
    if (!HET) return 1.0;
    return kinv_at<true>(L, ci, cj, sh);
}

// A x for the 10 DoFs of index (i, j) (eq. block_form_rq): xm, x0, xp point at (i, j-1), (i, j),
// (i, j+1) in plane 0 of a shared-memory tile whose planes are PS doubles apart and whose rows
// hold the column neighbours contiguously (all offsets compile-time constants).
// ROWS: bit k set -> row k is evaluated (a row subset for the small-tile kernels that split a
// position's rows over several threads; each row's accumulation is the same sequence either way)
template <int PS, bool HET, unsigned ROWS = 0x3FFu>
__device__ __forceinline__ void apply_rows(const LevelParams& L, const double* xm, const double* x0, const double* xp,
                                           int i, int j, double av[10]) {
#define XS(dx, dy, pl) ((dy) < 0 ? xm : ((dy) > 0 ? xp : x0))[(pl) * PS + (dx)]
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0, a6 = 0, a7 = 0, a8 = 0, a9 = 0;
    // factored stencil (mg_tables.h MG_STENCIL_FACT): entries sharing a coefficient up to sign are
    // summed first, then one FMA per coefficient group; rows interleaved round-robin (10
    // independent accumulator chains)
#define MG_A(row, g, sg, e) if ((ROWS >> (row)) & 1u) a##row = fma(sg L.cg[g], e, a##row);
    MG_STENCIL_FACT(MG_A)
#undef MG_A
#define MG_W(row, cdx, cdy, sh, dx, dy, pl, e, e2) \
    if ((ROWS >> (row)) & 1u) a##row = fma(L.ww[sh][e][e2] * kinv_ww<HET>(L, i + (cdx), j + (cdy), sh), XS(dx, dy, pl), a##row);
    MG_STENCIL_WW_5(MG_W)
    MG_STENCIL_WW_6(MG_W)
    MG_STENCIL_WW_7(MG_W)
#undef MG_W
#undef XS
    av[0] = a0; av[1] = a1; av[2] = a2; av[3] = a3; av[4] = a4;
    av[5] = a5; av[6] = a6; av[7] = a7; av[8] = a8; av[9] = a9;
}

// apply_rows with K^{-1} of the per-triangle M_w terms read from a shared-memory ring instead of
// global memory (marching kernels, heterogeneous K): km / k0 point at cell (i, j-1) / (i, j) of
// plane LL, plane UR is KPS doubles further (cells outside the mesh hold 0, like kinv_at)
template <int PS, int KPS>
__device__ __forceinline__ void apply_rows_kr(const LevelParams& L, const double* xm, const double* x0,
                                              const double* xp, const double* km, const double* k0, double av[10]) {
#define XS(dx, dy, pl) ((dy) < 0 ? xm : ((dy) > 0 ? xp : x0))[(pl) * PS + (dx)]
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0, a6 = 0, a7 = 0, a8 = 0, a9 = 0;
#define MG_A(row, g, sg, e) a##row = fma(sg L.cg[g], e, a##row);
    MG_STENCIL_FACT(MG_A)
#undef MG_A
#define MG_W(row, cdx, cdy, sh, dx, dy, pl, e, e2) \
    a##row = fma(L.ww[sh][e][e2] * ((cdy) < 0 ? km : k0)[(sh) * KPS + (cdx)], XS(dx, dy, pl), a##row);
    MG_STENCIL_WW_5(MG_W)
    MG_STENCIL_WW_6(MG_W)
    MG_STENCIL_WW_7(MG_W)
#undef MG_W
#undef XS
    av[0] = a0; av[1] = a1; av[2] = a2; av[3] = a3; av[4] = a4;
    av[5] = a5; av[6] = a6; av[7] = a7; av[8] = a8; av[9] = a9;
}

// exact-integration operator (L.lamx = lambda != 0): the bubble rows add lambda * REF_EXDIV over the
// two triangles of each edge -- H(i,j): LL(i,j), UR(i,j-1); V(i,j): LL(i,j), UR(i-1,j); D(i,j): LL(i,j),
// UR(i,j) -- whose bubbles are LL(i,j): H(i,j), V(i,j), D(i,j) and UR(i,j): H(i,j+1), V(i+1,j), D(i,j)
__device__ __forceinline__ void exact_bubble_add(double lx, const double* xm, const double* x0, const double* xp,
                                                 int PS, double av[10]) {
#define XB(dx, dy, pl) ((dy) < 0 ? xm : ((dy) > 0 ? xp : x0))[(pl) * PS + (dx)]
    // REF_EXDIV is the same for both shapes in the local (H, V, D) order
    constexpr double EHH = 4.0 / 9.0, EHV = -2.0 / 9.0, EHD = -0.15713484026367724, EDD = 2.0 / 9.0;
    av[2] = fma(lx, 2.0 * EHH * XB(0, 0, 2) + EHV * (XB(0, 0, 3) + XB(1, -1, 3)) + EHD * (XB(0, 0, 4) + XB(0, -1, 4)), av[2]);
    av[3] = fma(lx, 2.0 * EHH * XB(0, 0, 3) + EHV * (XB(0, 0, 2) + XB(-1, 1, 2)) + EHD * (XB(0, 0, 4) + XB(-1, 0, 4)), av[3]);
    av[4] = fma(lx, 2.0 * EDD * XB(0, 0, 4) + EHD * (XB(0, 0, 2) + XB(0, 1, 2)) + EHD * (XB(0, 0, 3) + XB(1, 0, 3)), av[4]);
#undef XB
}

// r = b - A x for the 10 DoFs of index (i, j); xs is a W x HT x 10 tile holding (i, j) at
// (lx, ly) with a ring of at least 1.  Inactive rows give 0.
template <int W, int HT, bool HET, bool NC = true>
__device__ __forceinline__ void residual_at(const LevelParams& L, const double* __restrict__ xs, int lx, int ly,
                                            int i, int j, const double* __restrict__ b, double r[10]) {
    const double* x0 = xs + ly * W + lx;
    double av[10];
    apply_rows<W * HT, HET>(L, x0 - W, x0, x0 + W, i, j, av);
    if (L.lamx != 0.0) exact_bubble_add(L.lamx, x0 - W, x0, x0 + W, W * HT, av);
    const int n = L.n;
    const int64_t o = (int64_t)j * L.pitch + i;
    const bool in = i >= 0 && j >= 0 && i <= n && j <= n;
#pragma unroll
    for (int k = 0; k < 10; ++k) r[k] = is_active(k, i, j, n) ? (gld<NC>(b + k * L.plane + (in ? o : 0)) - av[k]) : 0.0;
}

// residual_at with b already in registers (bp[k] = b of plane k at (i, j), anything where inactive): the
// latency-bound tile kernels issue these loads together with the x tile instead of after it
template <int W, int HT, bool HET>
__device__ __forceinline__ void residual_at_b(const LevelParams& L, const double* __restrict__ xs, int lx, int ly,
                                              int i, int j, const double bp[10], double r[10]) {
    const double* x0 = xs + ly * W + lx;
    double av[10];
    apply_rows<W * HT, HET>(L, x0 - W, x0, x0 + W, i, j, av);
    if (L.lamx != 0.0) exact_bubble_add(L.lamx, x0 - W, x0, x0 + W, W * HT, av);
#pragma unroll
    for (int k = 0; k < 10; ++k) r[k] = is_active(k, i, j, L.n) ? (bp[k] - av[k]) : 0.0;
}
// the b values residual_at would read for position (i, j) (0 outside the mesh)
__device__ __forceinline__ void load_b10(const LevelParams& L, const double* __restrict__ b, int i, int j, bool on,
                                         double bp[10]) {
    const int n = L.n;
    const bool in = on && i >= 0 && j >= 0 && i <= n && j <= n;
    const int64_t o = in ? (int64_t)j * L.pitch + i : 0;
#pragma unroll
    for (int k = 0; k < 10; ++k) bp[k] = in ? __ldg(b + k * L.plane + o) : 0.0;
}

// ------------------------------------------------------------------------------------------
// residual
constexpr int RTX = 32, RTY = 8, RNT = 256;

template <bool HET, bool APPLY>
__global__ void __launch_bounds__(RNT) residual_kernel(const LevelParams L, const double* __restrict__ x,
                                                       const double* __restrict__ b, double* __restrict__ r,
                                                       NormSink S) {
    pdl_wait();
    pdl_trigger();
    constexpr int XW = RTX + 2, XH = RTY + 2;
    __shared__ double xs[10 * XW * XH];
    if (*L.stop) return;
    const int i0 = blockIdx.x * RTX, j0 = blockIdx.y * RTY;
    load_tile<XW, XH, 10>(xs, x, i0 - 1, j0 - 1, L.n, L.pitch, L.plane);
    __syncthreads();
    const int lx = threadIdx.x % RTX, ly = threadIdx.x / RTX;
    const int i = i0 + lx, j = j0 + ly;
    double nrm = 0.0;
    if (i <= L.n && j <= L.n) {
        double rv[10];
        if (APPLY) {
            // out = A x (masked): the operator application of FGMRES (b unused)
            const double* x0 = xs + (ly + 1) * XW + (lx + 1);
            apply_rows<XW * XH, HET>(L, x0 - XW, x0, x0 + XW, i, j, rv);
            if (L.lamx != 0.0) exact_bubble_add(L.lamx, x0 - XW, x0, x0 + XW, XW * XH, rv);
#pragma unroll
            for (int k = 0; k < 10; ++k) rv[k] = is_active(k, i, j, L.n) ? rv[k] : 0.0;
        } else {
            residual_at<XW, XH, HET>(L, xs, lx + 1, ly + 1, i, j, b, rv);
        }
        const int64_t o = (int64_t)j * L.pitch + i;
#pragma unroll
        for (int k = 0; k < 10; ++k) {
            if (r) r[k * L.plane + o] = rv[k];
            nrm = fma(rv[k], rv[k], nrm);
        }
    }
    if (S.out || S.state) norm_finish<RNT>(S, nrm);
}

// ------------------------------------------------------------------------------------------
// additive Vanka sweep: xout = x + omega sum_v V^T D K_v^{-1} V (b - A x)
constexpr int VTX = 32, VTY = 8, VNT = 352;   // (VTX+2)(VTY+2) = 340 residual positions, one per thread
// 2-D tile geometry of the single-pass Vanka sweep for a TX x TY owner tile (x tile +2 ring,
// residual +1 ring, patches +1 high ring); small tiles for the latency-bound coarse levels
template <int TX, int TY>
struct VTile {
    static constexpr int XW = TX + 4, XH = TY + 4, RW = TX + 2, RH = TY + 2, PW = TX + 1, PH = TY + 1;
    static constexpr int XSZ = 10 * XW * XH, CSZ = 20 * PW * PH, USZ = XSZ > CSZ ? XSZ : CSZ;
    static constexpr int SMEM = (USZ + 10 * RW * RH) * 8;
    static constexpr int NT = ((RW * RH + 31) / 32) * 32;   // >= PW * PH, TX * TY
};
constexpr int VSX = 8, VSY = 4;                // small tiles: 64 threads
constexpr int V_XW = VTX + 4, V_XH = VTY + 4, V_RW = VTX + 2, V_RH = VTY + 2, V_PW = VTX + 1, V_PH = VTY + 1;
constexpr int V_XSZ = 10 * V_XW * V_XH, V_CSZ = 20 * V_PW * V_PH;
constexpr int V_USZ = V_XSZ > V_CSZ ? V_XSZ : V_CSZ;
constexpr int V_SMEM = (V_USZ + 10 * V_RW * V_RH) * 8;

// gather the 20 patch residuals of the vertex at r-tile position r00 (MG_VSLOT_TABLE order)
template <int RW, int RH>
__device__ __forceinline__ void gather20(const double* r00, double rr[20]) {
#define RR(dx, dy, pl) r00[(pl) * (RW * RH) + (dy) * RW + (dx)]
    rr[0] = RR(0, 0, 0);   rr[1] = RR(0, 0, 1);
    rr[2] = RR(0, 0, 2);   rr[3] = RR(-1, 0, 2);  rr[4] = RR(0, 0, 3);   rr[5] = RR(0, -1, 3);
    rr[6] = RR(-1, 0, 4);  rr[7] = RR(0, -1, 4);
    rr[8] = RR(0, 0, 5);   rr[9] = RR(-1, 0, 5);  rr[10] = RR(0, 0, 6);  rr[11] = RR(0, -1, 6);
    rr[12] = RR(-1, 0, 7); rr[13] = RR(0, -1, 7);
    rr[14] = RR(0, 0, 8);  rr[15] = RR(-1, -1, 9); rr[16] = RR(-1, 0, 8); rr[17] = RR(0, -1, 9);
    rr[18] = RR(-1, 0, 9); rr[19] = RR(0, -1, 8);
#undef RR
}

__device__ __forceinline__ int vertex_class(int a, int b, int n) {
    return (a == 0 ? 1 : (a == n ? 2 : 0)) + 3 * (b == 0 ? 1 : (b == n ? 2 : 0));
}

// out[s * os] = (D K^{-1} r)_s for one 20-DoF patch (interior: +/- blocks; boundary class: dense
// table), written straight to shared memory.  UNROLL_BND: the five passes over the dense table are
// unrolled (the small-tile kernels of the latency-bound coarse levels, where the boundary patches
// are the critical path); same summation order either way
template <bool UNROLL_BND = false>
__device__ __forceinline__ void patch_apply20(const VankaParams& P, int cls, const double rr[20], double* out, int os) {
    if (cls == 0) {
        double hp[9], hm[11];
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            hp[q] = rr[2 + 2 * q] - rr[3 + 2 * q];
            hm[2 + q] = rr[2 + 2 * q] + rr[3 + 2 * q];
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            hp[6 + q] = rr[14 + 2 * q] + rr[15 + 2 * q];
            hm[8 + q] = rr[14 + 2 * q] - rr[15 + 2 * q];
        }
        hm[0] = rr[0];
        hm[1] = rr[1];
        // column-outer loops: the 20 output chains advance together (same per-output summation order)
        double yp[9], ym[11];
#pragma unroll
        for (int a = 0; a < 9; ++a) yp[a] = 0.0;
#pragma unroll
        for (int a = 0; a < 11; ++a) ym[a] = 0.0;
#pragma unroll
        for (int c = 0; c < 11; ++c) {
#pragma unroll
            for (int a = 0; a < 11; ++a) ym[a] = fma(P.gmT[c][a], hm[c], ym[a]);
            if (c < 9) {
#pragma unroll
                for (int a = 0; a < 9; ++a) yp[a] = fma(P.gpT[c][a], hp[c], yp[a]);
            }
        }
        out[0] = ym[0];
        out[os] = ym[1];
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            out[(2 + 2 * q) * os] = ym[2 + q] + yp[q];
            out[(3 + 2 * q) * os] = ym[2 + q] - yp[q];
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            out[(14 + 2 * q) * os] = yp[6 + q] + ym[8 + q];
            out[(15 + 2 * q) * os] = yp[6 + q] - ym[8 + q];
        }
    } else {
        // boundary class: dense 20 x 20 (row major in gbnd), four output rows per pass so four
        // independent chains hide the load and fp64 latency (each output sums c = 0 .. 19 in order)
        const double2* G = reinterpret_cast<const double2*>(P.gbnd + cls * 400);
        auto pass = [&](int a) {
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
            for (int c2 = 0; c2 < 10; ++c2) {
                const double2 g0 = __ldg(G + (a + 0) * 10 + c2), g1 = __ldg(G + (a + 1) * 10 + c2);
                const double2 g2 = __ldg(G + (a + 2) * 10 + c2), g3 = __ldg(G + (a + 3) * 10 + c2);
                s0 = fma(g0.x, rr[2 * c2], s0); s0 = fma(g0.y, rr[2 * c2 + 1], s0);
                s1 = fma(g1.x, rr[2 * c2], s1); s1 = fma(g1.y, rr[2 * c2 + 1], s1);
                s2 = fma(g2.x, rr[2 * c2], s2); s2 = fma(g2.y, rr[2 * c2 + 1], s2);
                s3 = fma(g3.x, rr[2 * c2], s3); s3 = fma(g3.y, rr[2 * c2 + 1], s3);
            }
            out[(a + 0) * os] = s0;
            out[(a + 1) * os] = s1;
            out[(a + 2) * os] = s2;
            out[(a + 3) * os] = s3;
        };
        if (UNROLL_BND) {
#pragma unroll
            for (int a = 0; a < 20; a += 4) pass(a);
        } else {
#pragma unroll 1
            for (int a = 0; a < 20; a += 4) pass(a);
        }
    }
}

// Heterogeneous-K patch solve (mg_internal.h HetVankaTabs): the class-constant condensed tables
// and the per-vertex inverse RT0 Schur complement S_v^{-1} (upper triangle, MG_HV_NSINV planes).
// out[s * os] = (D K_v^{-1} r)_s for the vertex (a, b) of class cls.
// T: the class table (the interior class's from the kernel parameter block -- constant-bank operands
// -- the 8 boundary classes' from global memory); LD(k) reads entry k
template <bool CONST_T>
__device__ __forceinline__ void patch_apply_het_t(const VankaParams& P, const double* __restrict__ T, int a, int b,
                                                  const double rr[20], double* out, int os) {
#define LD(k) (CONST_T ? T[k] : __ldg(T + (k)))
    double ry[14];
#pragma unroll
    for (int q = 0; q < 8; ++q) ry[q] = rr[q];
#pragma unroll
    for (int q = 0; q < 6; ++q) ry[8 + q] = rr[14 + q];
    // a = G_def r_y (column-outer: 14 independent chains)
    double ad[14];
#pragma unroll
    for (int q = 0; q < 14; ++q) ad[q] = 0.0;
#pragma unroll
    for (int c = 0; c < 14; ++c) {          // column-outer: the 14 output chains advance together
#pragma unroll
        for (int q = 0; q < 14; ++q) ad[q] = fma(LD(MG_HV_G + q * 14 + c), ry[c], ad[q]);
    }
    // constant-pressure part of K_yy^{-1} r_y: -(1^T r_p) / (m gamma) on every active P0 slot
    double psum = 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k) psum += ry[8 + k];
    const double cp = -psum * LD(MG_HV_PINV);
    // s~ = U^T r_r - (U^T K_ry) a_def  (in the basis U; K_ry: P0 columns only)
    double sv[6];
#pragma unroll
    for (int j = 0; j < 6; ++j) {
        double v = 0.0;
#pragma unroll
        for (int e = 0; e < 6; ++e) v = fma(LD(MG_HV_U + e * 6 + j), rr[8 + e], v);
#pragma unroll
        for (int k = 0; k < 6; ++k) v = fma(-LD(MG_HV_KRP + j * 6 + k), ad[8 + k], v);
        sv[j] = v;
    }
    // z~ = S~_v^{-1} s~ (symmetric, upper triangle per vertex)
    const double* si = P.hv.sinv + (int64_t)b * P.L.pitch + a;
    double zr[6];
#pragma unroll
    for (int e = 0; e < 6; ++e) {
        double v = 0.0;
#pragma unroll
        for (int f = 0; f < 6; ++f) {
            const int lo = e < f ? e : f, hi = e < f ? f : e;
            v = fma(__ldg(si + (lo * 6 - lo * (lo - 1) / 2 + (hi - lo)) * P.L.plane), sv[f], v);
        }
        zr[e] = v;
    }
    // z_y = a_def + cp 1_p - (Q U) z~; weights
#pragma unroll
    for (int q = 0; q < 14; ++q) {
        double v = ad[q] + (q >= 8 ? cp : 0.0);
#pragma unroll
        for (int e = 0; e < 6; ++e) v = fma(-LD(MG_HV_Q + q * 6 + e), zr[e], v);
        const int sl = q < 8 ? q : q + 6;
        out[sl * os] = LD(MG_HV_D + sl) * v;
    }
    // z_r = U z~
#pragma unroll
    for (int e = 0; e < 6; ++e) {
        double v = 0.0;
#pragma unroll
        for (int j = 0; j < 6; ++j) v = fma(LD(MG_HV_U + e * 6 + j), zr[j], v);
        out[(8 + e) * os] = LD(MG_HV_D + 8 + e) * v;
    }
#undef LD
}

// interior vertex: the +/- form of the condensed solve (mg_internal.h HvInteriorPM), 232 FMA instead
// of the slot form's 424; every table entry is a constant-bank operand
// PRE: the vertex's 21 S~^{-1} entries come preloaded in sq (registers) instead of being read here
template <bool PRE = false>
__device__ __forceinline__ void patch_apply_het_pm(const VankaParams& P, const HvInteriorPM& T, int a, int b,
                                                   const double rr[20], double* out, int os,
                                                   const double* sq = nullptr) {
    double hp[6], hm[8], rd[3], rs[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        hp[q] = rr[2 + 2 * q] - rr[3 + 2 * q];
        hp[3 + q] = rr[14 + 2 * q] + rr[15 + 2 * q];
        hm[2 + q] = rr[2 + 2 * q] + rr[3 + 2 * q];
        hm[5 + q] = rr[14 + 2 * q] - rr[15 + 2 * q];
        rd[q] = rr[8 + 2 * q] - rr[9 + 2 * q];
        rs[q] = rr[8 + 2 * q] + rr[9 + 2 * q];
    }
    hm[0] = rr[0];
    hm[1] = rr[1];
    double ap[6], am[8];
#pragma unroll
    for (int r = 0; r < 6; ++r) ap[r] = 0.0;
#pragma unroll
    for (int r = 0; r < 8; ++r) am[r] = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {            // column-outer: independent output chains
#pragma unroll
        for (int r = 0; r < 8; ++r) am[r] = fma(T.gm[r][c], hm[c], am[r]);
        if (c < 6) {
#pragma unroll
            for (int r = 0; r < 6; ++r) ap[r] = fma(T.gp[r][c], hp[c], ap[r]);
        }
    }
    const double cp = -(hp[3] + hp[4] + hp[5]) * T.pinv;   // -(1^T r_p) / (m gamma)
    double sv[6];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        double vp = 0.0, vm = 0.0;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            vp = fma(T.up[j][q], rd[q], vp);
            vm = fma(T.um[j][q], rs[q], vm);
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            vp = fma(-T.kp[j][k], ap[3 + k], vp);
            vm = fma(-T.km[j][k], am[5 + k], vm);
        }
        sv[j] = vp;
        sv[3 + j] = vm;
    }
    const double* si = P.hv.sinv + (int64_t)b * P.L.pitch + a;
    double zt[6];
#pragma unroll
    for (int e = 0; e < 6; ++e) {
        double v = 0.0;
#pragma unroll
        for (int f = 0; f < 6; ++f) {
            const int lo = e < f ? e : f, hi = e < f ? f : e;
            const int q = lo * 6 - lo * (lo - 1) / 2 + (hi - lo);
            v = fma(PRE ? sq[q] : __ldg(si + q * P.L.plane), sv[f], v);
        }
        zt[e] = v;
    }
#pragma unroll
    for (int r = 0; r < 6; ++r) {
        double v = ap[r] + (r >= 3 ? cp : 0.0);
#pragma unroll
        for (int j = 0; j < 3; ++j) v = fma(-T.qp[r][j], zt[j], v);
        ap[r] = v;
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        double v = am[r];
#pragma unroll
        for (int j = 0; j < 3; ++j) v = fma(-T.qm[r][j], zt[3 + j], v);
        am[r] = v;
    }
    // slots with the natural weights: u 1, bubble and RT0 1/2, P0 1/3
    out[0] = am[0];
    out[os] = am[1];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        out[(2 + 2 * q) * os] = 0.5 * (am[2 + q] + ap[q]);
        out[(3 + 2 * q) * os] = 0.5 * (am[2 + q] - ap[q]);
        double yp = 0.0, ym = 0.0;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            yp = fma(T.up[j][q], zt[j], yp);
            ym = fma(T.um[j][q], zt[3 + j], ym);
        }
        out[(8 + 2 * q) * os] = 0.5 * (ym + yp);
        out[(9 + 2 * q) * os] = 0.5 * (ym - yp);
        out[(14 + 2 * q) * os] = (1.0 / 3.0) * (ap[3 + q] + am[5 + q]);
        out[(15 + 2 * q) * os] = (1.0 / 3.0) * (ap[3 + q] - am[5 + q]);
    }
}

__device__ __forceinline__ void patch_apply_het(const VankaParams& P, const HvInterior* Ti, int cls, int a, int b,
                                                const double rr[20], double* out, int os) {
    if (cls == 0 && Ti) patch_apply_het_pm(P, Ti->pm, a, b, rr, out, os);
    else patch_apply_het_t<false>(P, P.hv.cls + cls * MG_HV_CLS, a, b, rr, out, os);
}

// per-vertex S~_v^{-1} of the heterogeneous Vanka patches of one level (setup), in the basis U of
// the class (mg_internal.h): S~_v = sum over the star triangles of K^{-1}_T W~[cls][tri] - C~[cls];
// inactive RT0 slots get a unit diagonal (their right-hand side is always 0).  Gauss-Jordan with
// partial pivoting in fp64.
__global__ void __launch_bounds__(256) hv_sinv_kernel(const LevelParams L, const double* __restrict__ W,
                                                      const double* __restrict__ C, double* __restrict__ sinv) {
    const int a = blockIdx.x * 32 + (threadIdx.x & 31), b = blockIdx.y * 8 + (threadIdx.x >> 5);
    const int n = L.n;
    if (a > n || b > n) return;
    const int cls = (a == 0 ? 1 : (a == n ? 2 : 0)) + 3 * (b == 0 ? 1 : (b == n ? 2 : 0));
    double S[6][6], I[6][6];
    for (int e = 0; e < 6; ++e)
        for (int f = 0; f < 6; ++f) {
            S[e][f] = -C[cls * 36 + e * 6 + f];
            I[e][f] = e == f ? 1.0 : 0.0;
        }
    for (int sh = 0; sh < 2; ++sh)
        for (int ty = 0; ty < 2; ++ty)
            for (int tx = 0; tx < 2; ++tx) {
                const int ci = a - 1 + tx, cj = b - 1 + ty;
                if (ci < 0 || cj < 0 || ci >= n || cj >= n) continue;
                const double k = L.kinv_field[sh * L.plane + (int64_t)cj * L.pitch + ci];
                const double* Wt = W + cls * MG_HV_W + (4 * sh + 2 * ty + tx) * 36;
                for (int e = 0; e < 36; ++e) S[e / 6][e % 6] = fma(k, Wt[e], S[e / 6][e % 6]);
            }
    for (int e = 0; e < 6; ++e) {
        bool zero = true;
        for (int f = 0; f < 6; ++f) zero = zero && S[e][f] == 0.0 && S[f][e] == 0.0;
        if (zero) S[e][e] = 1.0;
    }
    for (int c = 0; c < 6; ++c) {
        int piv = c;
        for (int r = c + 1; r < 6; ++r)
            if (fabs(S[r][c]) > fabs(S[piv][c])) piv = r;
        if (piv != c)
            for (int k = 0; k < 6; ++k) {
                double t = S[c][k]; S[c][k] = S[piv][k]; S[piv][k] = t;
                t = I[c][k]; I[c][k] = I[piv][k]; I[piv][k] = t;
            }
        const double d = 1.0 / S[c][c];
        for (int k = 0; k < 6; ++k) { S[c][k] *= d; I[c][k] *= d; }
        for (int r = 0; r < 6; ++r) {
            if (r == c) continue;
            const double f = S[r][c];
            for (int k = 0; k < 6; ++k) { S[r][k] = fma(-f, S[c][k], S[r][k]); I[r][k] = fma(-f, I[c][k], I[r][k]); }
        }
    }
    const int64_t o = (int64_t)b * L.pitch + a;
    int k = 0;
    for (int e = 0; e < 6; ++e)
        for (int f = e; f < 6; ++f) sinv[(k++) * L.plane + o] = 0.5 * (I[e][f] + I[f][e]);
}

// one TX x TY tile of the sweep, run by threads t = 0 .. T::NT-1 of a (virtual) block with shared
// memory sm; every thread executes the three barriers, `active` = false skips the work (tiles of
// the bottom kernel's last round).  Returns the thread's share of ||r||^2.
template <bool XZERO, int TX, int TY, bool NC, bool HET = false>
__device__ __forceinline__ double vanka_tile(const VankaParams& P, const double* __restrict__ x,
                                             const double* __restrict__ b, double* __restrict__ xo, int bx, int by,
                                             int t, double* sm, bool active, const HvInterior* Ti = nullptr) {
    using T = VTile<TX, TY>;
    double* xs = sm;          // x tile (phase 1)
    double* cs = sm;          // patch corrections (phase 2-3), overlays xs
    double* rs = sm + T::USZ;  // residual tile
    const LevelParams& L = P.L;
    const int n = L.n, pitch = L.pitch;
    const int64_t plane = L.plane;
    const int i0 = bx * TX, j0 = by * TY;
    const int tl = active ? t : 1 << 20;   // inactive: no thread takes a position
    // phase 1: r = b - A x on the tile + 1 ring (one index per thread; straight-line code keeps
    // the stencil coefficients as constant-bank operands instead of hoisted registers)
    if (!XZERO) {
        if (active) load_tile<T::XW, T::XH, 10, NC>(xs, x, i0 - 2, j0 - 2, n, pitch, plane, 0, t, T::NT);
        __syncthreads();
        if (tl < T::RW * T::RH) {
            const int ly = t / T::RW, lx = t - ly * T::RW;
            double rv[10];
            residual_at<T::XW, T::XH, HET, NC>(L, xs, lx + 1, ly + 1, i0 - 1 + lx, j0 - 1 + ly, b, rv);
#pragma unroll
            for (int k = 0; k < 10; ++k) rs[k * T::RW * T::RH + t] = rv[k];
        }
    } else {
        if (active) load_tile<T::RW, T::RH, 10, NC>(rs, b, i0 - 1, j0 - 1, n, pitch, plane, 0, t, T::NT);  // r = b (x = 0)
    }
    __syncthreads();
    // phase 2: patch solves at the vertices of the tile + high ring
    if (tl < T::PW * T::PH) {
        const int py = t / T::PW, px = t - py * T::PW;
        const int a = i0 + px, bb = j0 + py;
        if (a <= n && bb <= n) {
            double rr[20];
            gather20<T::RW, T::RH>(rs + (py + 1) * T::RW + (px + 1), rr);
            if (HET) patch_apply_het(P, Ti, vertex_class(a, bb, n), a, bb, rr, cs + t, T::PW * T::PH);
            else patch_apply20<(TX <= 8)>(P, vertex_class(a, bb, n), rr, cs + t, T::PW * T::PH);
        } else {
#pragma unroll
            for (int q = 0; q < 20; ++q) cs[q * T::PW * T::PH + t] = 0.0;
        }
    }
    __syncthreads();
    // phase 3: owners sum the corrections of the (up to) 4 patches touching their DoFs
    double nrm = 0.0;
    if (tl < TX * TY) {
        const int lx = t % TX, ly = t / TX;
        const int i = i0 + lx, j = j0 + ly;
        if (i <= n && j <= n) {
            const double* c00 = cs + ly * T::PW + lx;
#define CC(s, dx, dy) c00[(s) * (T::PW * T::PH) + (dy) * T::PW + (dx)]
            double d[10];
            d[0] = CC(0, 0, 0);
            d[1] = CC(1, 0, 0);
            d[2] = CC(2, 0, 0) + CC(3, 1, 0);
            d[3] = CC(4, 0, 0) + CC(5, 0, 1);
            d[4] = CC(6, 1, 0) + CC(7, 0, 1);
            d[5] = CC(8, 0, 0) + CC(9, 1, 0);
            d[6] = CC(10, 0, 0) + CC(11, 0, 1);
            d[7] = CC(12, 1, 0) + CC(13, 0, 1);
            d[8] = CC(14, 0, 0) + CC(16, 1, 0) + CC(19, 0, 1);
            d[9] = CC(15, 1, 1) + CC(17, 0, 1) + CC(18, 1, 0);
#undef CC
            const int64_t o = (int64_t)j * pitch + i;
            const double* r00 = rs + (ly + 1) * T::RW + (lx + 1);
#pragma unroll
            for (int k = 0; k < 10; ++k) {
                const double xv = XZERO ? 0.0 : gld<NC>(x + k * plane + o);
                xo[k * plane + o] = is_active(k, i, j, n) ? fma(P.omega, d[k], xv) : 0.0;
                const double rv = r00[k * T::RW * T::RH];
                nrm = fma(rv, rv, nrm);
            }
        }
    }
    return nrm;
}

// Small-tile sweep of the latency-bound coarse levels (8 x 4 owners, 64 threads): the arithmetic of
// vanka_tile, with every global read the kernel needs issued in its first round trip -- the stop flag,
// the x tile, b at the residual positions and x at the owners (registers), and the dense inverses of
// the boundary classes the tile touches (staged in shared memory) -- instead of one L2 round trip
// per phase (stop flag, tile, b, boundary table, owner x).  Bitwise vanka_tile's results.
struct VSmall {
    using T = VTile<VSX, VSY>;
    static constexpr int XS = T::XSZ, RS = 10 * T::RW * T::RH, CS = T::CSZ, GS = 8 * 400;
    static constexpr int SMEM = (XS + RS + CS + GS) * 8 + 16 * 4;
    static constexpr int SMEM_P = SMEM + 10 * ((VSX + 4) / 2 + 1) * ((VSY + 4) / 2 + 1) * 8;
};
// the boundary classes present among the vertices (a, b), a in [i0, i0 + TX], b in [j0, j0 + TY]
__device__ __forceinline__ unsigned tile_classes(int i0, int j0, int tx, int ty, int n) {
    const int a1 = min(i0 + tx, n), b1 = min(j0 + ty, n);
    unsigned cxm = 0, cym = 0;
    if (i0 <= a1) {
        if (i0 == 0) cxm |= 2u;
        if (a1 == n) cxm |= 4u;
        if (max(i0, 1) <= min(a1, n - 1)) cxm |= 1u;
    }
    if (j0 <= b1) {
        if (j0 == 0) cym |= 2u;
        if (b1 == n) cym |= 4u;
        if (max(j0, 1) <= min(b1, n - 1)) cym |= 1u;
    }
    unsigned m = 0;
    for (int cy = 0; cy < 3; ++cy)
        for (int cx = 0; cx < 3; ++cx)
            if (((cxm >> cx) & 1u) && ((cym >> cy) & 1u)) m |= 1u << (cx + 3 * cy);
    return m & ~1u;   // interior class 0: constant bank
}

// PROL: the first post-sweep relaxes x + P e_H (the coarse-grid correction fused in):
// the coarse tile under the x tile arrives with the first round trip, one thread per coarse cell adds
// P e_H to its 2 x 2 fine indices of the x tile (prolong_kernel's table chains), bitwise prolong_kernel
// followed by the sweep; the launch of prolong_kernel on the level disappears.
constexpr int VS_CW = (VSX + 4) / 2 + 1, VS_CH = (VSY + 4) / 2 + 1, VS_CS = 10 * VS_CW * VS_CH;
template <bool XZERO, bool PROL = false>
__global__ void __launch_bounds__(VTile<VSX, VSY>::NT, 4) vanka_small_kernel(const VankaParams P,
                                                                             const double* __restrict__ x,
                                                                             const double* __restrict__ b,
                                                                             double* __restrict__ xo, NormSink S,
                                                                             const ProlSrc E) {
    pdl_wait();
    pdl_trigger();
    using T = VTile<VSX, VSY>;
    extern __shared__ __align__(16) double sm[];
    double* xs = sm;                      // x tile [10][XH][XW]
    double* rs = xs + VSmall::XS;         // residual tile [10][RH][RW]
    double* cs = rs + VSmall::RS;         // patch corrections [20][PH][PW]
    double* gs = cs + VSmall::CS;         // dense inverses of the boundary classes present, in class order
    double* es = gs + VSmall::GS;         // PROL: coarse tile [10][VS_CH][VS_CW] from coarse (i0/2 - 1, j0/2 - 1)
    const LevelParams& L = P.L;
    const int stopv = *L.stop;            // checked after the loads are in flight
    const int n = L.n, pitch = L.pitch, t = threadIdx.x;
    const int64_t plane = L.plane;
    const int i0 = blockIdx.x * VSX, j0 = blockIdx.y * VSY;
    // b at this thread's residual position, x at its owner index (registers)
    double bpre[10], xown[10];
    const int ly = t / T::RW, lx = t - ly * T::RW;
    {
        const int i = i0 - 1 + lx, j = j0 - 1 + ly;
        const bool in = t < T::RW * T::RH && i >= 0 && j >= 0 && i <= n && j <= n;
        const int64_t o = in ? (int64_t)j * pitch + i : 0;
#pragma unroll
        for (int k = 0; k < 10; ++k) bpre[k] = in ? __ldg(b + k * plane + o) : 0.0;
    }
    const int ox = t % VSX, oy = t / VSX;
    if (!PROL) {
        const int i = i0 + ox, j = j0 + oy;
        const bool in = !XZERO && t < VSX * VSY && i <= n && j <= n;
        const int64_t o = in ? (int64_t)j * pitch + i : 0;
#pragma unroll
        for (int k = 0; k < 10; ++k) xown[k] = in ? __ldg(x + k * plane + o) : 0.0;
    }
    const unsigned cm = tile_classes(i0, j0, VSX, VSY, n);
    {
        // cp.async: every 16-byte piece of the staged tables in flight at once, no registers
        int slot = 0;
        for (int c = 1; c < 9; ++c) {
            if (!((cm >> c) & 1u)) continue;
            const double* src = P.gbnd + c * 400;
            double* dst = gs + slot * 400;
            for (int q = t; q < 200; q += T::NT)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + 2 * q)), "l"(src + 2 * q)
                             : "memory");
            ++slot;
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    if (!XZERO) load_tile<T::XW, T::XH, 10, true, 16>(xs, x, i0 - 2, j0 - 2, n, pitch, plane, 0, t, T::NT);
    if (PROL) load_tile<VS_CW, VS_CH, 10, true, 16>(es, E.e, i0 / 2 - 1, j0 / 2 - 1, E.nc, E.pitchc, E.planec, 0, t, T::NT);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    if (stopv) return;
    if (PROL) {
        // x tile + P e_H: thread c < 24 takes coarse cell (I, J) = (i0/2 - 1 + cx, j0/2 - 1 + cy) and its fine
        // indices (2I + di, 2J + dj) at tile position (2cx + di, 2cy + dj)
        constexpr int NCX = T::XW / 2, NCY = T::XH / 2;
        if (t < NCX * NCY) {
            const int cy = t / NCX, cx = t - cy * NCX;
            const int I = i0 / 2 - 1 + cx, J = j0 / 2 - 1 + cy;
            if (I >= 0 && J >= 0 && I < E.nc && J < E.nc) {
                const double* e0 = es + cy * VS_CW + cx;
#define EQ(dI, dJ, pl, wt) v = fma(wt, e0[(pl) * (VS_CW * VS_CH) + (dJ) * VS_CW + (dI)], v);
#define P2(dj, kf)                                                                       \
    {                                                                                    \
        double v = 0.0;                                                                  \
        MG_PROLONG_0_##dj##_##kf(EQ) const double v0 = v;                                \
        v = 0.0;                                                                         \
        MG_PROLONG_1_##dj##_##kf(EQ) const double v1 = v;                                \
        double* xp2 = xs + (kf) * (T::XW * T::XH) + (2 * cy + (dj)) * T::XW + 2 * cx;    \
        if (is_active(kf, 2 * I, 2 * J + (dj), n)) xp2[0] += v0;                         \
        if (is_active(kf, 2 * I + 1, 2 * J + (dj), n)) xp2[1] += v1;                     \
    }
#define P4(kf) P2(0, kf) P2(1, kf)
                P4(0) P4(1) P4(2) P4(3) P4(4) P4(5) P4(6) P4(7) P4(8) P4(9)
#undef P4
#undef P2
#undef EQ
            }
        }
        __syncthreads();
        // the owners' x: the prolongated tile value
        if (t < VSX * VSY) {
#pragma unroll
            for (int k = 0; k < 10; ++k) xown[k] = xs[k * (T::XW * T::XH) + (oy + 2) * T::XW + (ox + 2)];
        }
    }
    // phase 1: r = b - A x on the tile + 1 ring
    if (t < T::RW * T::RH) {
        const int i = i0 - 1 + lx, j = j0 - 1 + ly;
        double rv[10];
        if (!XZERO) {
            const double* x0 = xs + (ly + 1) * T::XW + (lx + 1);
            double av[10];
            apply_rows<T::XW * T::XH, false>(L, x0 - T::XW, x0, x0 + T::XW, i, j, av);
            if (L.lamx != 0.0) exact_bubble_add(L.lamx, x0 - T::XW, x0, x0 + T::XW, T::XW * T::XH, av);
#pragma unroll
            for (int k = 0; k < 10; ++k) rv[k] = is_active(k, i, j, n) ? (bpre[k] - av[k]) : 0.0;
        } else {
#pragma unroll
            for (int k = 0; k < 10; ++k) rv[k] = bpre[k];
        }
#pragma unroll
        for (int k = 0; k < 10; ++k) rs[k * T::RW * T::RH + t] = rv[k];
    }
    __syncthreads();
    // phase 2: patch solves at the vertices of the tile + high ring
    if (t < T::PW * T::PH) {
        const int py = t / T::PW, px = t - py * T::PW;
        const int a = i0 + px, bb = j0 + py;
        constexpr int OS = T::PW * T::PH;
        if (a <= n && bb <= n) {
            double rr[20];
            gather20<T::RW, T::RH>(rs + (py + 1) * T::RW + (px + 1), rr);
            const int cls = vertex_class(a, bb, n);
            if (cls == 0) {
                patch_apply20<true>(P, 0, rr, cs + t, OS);
            } else {
                const double2* G = reinterpret_cast<const double2*>(gs + __popc(cm & ((1u << cls) - 1u)) * 400);
#pragma unroll
                for (int a4 = 0; a4 < 20; a4 += 4) {
                    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
                    for (int c2 = 0; c2 < 10; ++c2) {
                        const double2 g0 = G[(a4 + 0) * 10 + c2], g1 = G[(a4 + 1) * 10 + c2];
                        const double2 g2 = G[(a4 + 2) * 10 + c2], g3 = G[(a4 + 3) * 10 + c2];
                        s0 = fma(g0.x, rr[2 * c2], s0); s0 = fma(g0.y, rr[2 * c2 + 1], s0);
                        s1 = fma(g1.x, rr[2 * c2], s1); s1 = fma(g1.y, rr[2 * c2 + 1], s1);
                        s2 = fma(g2.x, rr[2 * c2], s2); s2 = fma(g2.y, rr[2 * c2 + 1], s2);
                        s3 = fma(g3.x, rr[2 * c2], s3); s3 = fma(g3.y, rr[2 * c2 + 1], s3);
                    }
                    cs[(a4 + 0) * OS + t] = s0;
                    cs[(a4 + 1) * OS + t] = s1;
                    cs[(a4 + 2) * OS + t] = s2;
                    cs[(a4 + 3) * OS + t] = s3;
                }
            }
        } else {
#pragma unroll
            for (int q = 0; q < 20; ++q) cs[q * OS + t] = 0.0;
        }
    }
    __syncthreads();
    // phase 3: owners
    double nrm = 0.0;
    if (t < VSX * VSY) {
        const int i = i0 + ox, j = j0 + oy;
        if (i <= n && j <= n) {
            const double* c00 = cs + oy * T::PW + ox;
#define CC(s_, dx, dy) c00[(s_) * (T::PW * T::PH) + (dy) * T::PW + (dx)]
            double d[10];
            d[0] = CC(0, 0, 0);
            d[1] = CC(1, 0, 0);
            d[2] = CC(2, 0, 0) + CC(3, 1, 0);
            d[3] = CC(4, 0, 0) + CC(5, 0, 1);
            d[4] = CC(6, 1, 0) + CC(7, 0, 1);
            d[5] = CC(8, 0, 0) + CC(9, 1, 0);
            d[6] = CC(10, 0, 0) + CC(11, 0, 1);
            d[7] = CC(12, 1, 0) + CC(13, 0, 1);
            d[8] = CC(14, 0, 0) + CC(16, 1, 0) + CC(19, 0, 1);
            d[9] = CC(15, 1, 1) + CC(17, 0, 1) + CC(18, 1, 0);
#undef CC
            const int64_t o = (int64_t)j * pitch + i;
            const double* r00 = rs + (oy + 1) * T::RW + (ox + 1);
#pragma unroll
            for (int k = 0; k < 10; ++k) {
                xo[k * plane + o] = is_active(k, i, j, n) ? fma(P.omega, d[k], xown[k]) : 0.0;
                const double rv = r00[k * T::RW * T::RH];
                nrm = fma(rv, rv, nrm);
            }
        }
    }
    if (S.out || S.state) norm_finish<T::NT>(S, nrm);
}

// Four threads per position (vanka_small4_kernel, MG_SMALL_DIET=2): the small-tile sweep above with each
// residual position's ten rows split over four threads (rows {0,2}, {1,3}, {4,5,6}, {7,8,9}: ~48 FMA +
// loads each), each patch solve's twenty outputs split over four threads (the +/- blocks by output
// pairs, the dense boundary inverses 5 rows each) and the prolongation's planes split likewise -- on the
// latency-bound coarse levels a kernel is one warp's serial instruction stream, which this cuts ~4x.
// Same arithmetic and order per value: bitwise vanka_small_kernel.
constexpr int VS4_NT = 256;
template <int G> struct RowGroup;
template <> struct RowGroup<0> { static constexpr unsigned M = 0x005u; };
template <> struct RowGroup<1> { static constexpr unsigned M = 0x00Au; };
template <> struct RowGroup<2> { static constexpr unsigned M = 0x070u; };
template <> struct RowGroup<3> { static constexpr unsigned M = 0x380u; };
template <bool XZERO, bool PROL = false>
__global__ void __launch_bounds__(VS4_NT, 2) vanka_small4_kernel(const VankaParams P, const double* __restrict__ x,
                                                                 const double* __restrict__ b, double* __restrict__ xo,
                                                                 NormSink S, const ProlSrc E) {
    pdl_wait();
    pdl_trigger();
    using T = VTile<VSX, VSY>;
    extern __shared__ __align__(16) double sm[];
    double* xs = sm;
    double* rs = xs + VSmall::XS;
    double* cs = rs + VSmall::RS;
    double* gs = cs + VSmall::CS;
    double* es = gs + VSmall::GS;
    const LevelParams& L = P.L;
    const int stopv = *L.stop;
    const int n = L.n, pitch = L.pitch, t = threadIdx.x;
    const int64_t plane = L.plane;
    const int i0 = blockIdx.x * VSX, j0 = blockIdx.y * VSY;
    const int pos = t & 63, grp = t >> 6;   // grp warp-uniform (two warps per group)
    const unsigned gm = grp == 0 ? RowGroup<0>::M : grp == 1 ? RowGroup<1>::M : grp == 2 ? RowGroup<2>::M : RowGroup<3>::M;
    const int ly = pos / T::RW, lx = pos - ly * T::RW;
    double bpre[10];
    {
        const int i = i0 - 1 + lx, j = j0 - 1 + ly;
        const bool in = pos < T::RW * T::RH && i >= 0 && j >= 0 && i <= n && j <= n;
        const int64_t o = in ? (int64_t)j * pitch + i : 0;
#pragma unroll
        for (int k = 0; k < 10; ++k) bpre[k] = (in && ((gm >> k) & 1u)) ? __ldg(b + k * plane + o) : 0.0;
    }
    const int ox = t % VSX, oy = t / VSX;
    double xown[10];
    if (!PROL) {
        const int i = i0 + ox, j = j0 + oy;
        const bool in = !XZERO && t < VSX * VSY && i <= n && j <= n;
        const int64_t o = in ? (int64_t)j * pitch + i : 0;
#pragma unroll
        for (int k = 0; k < 10; ++k) xown[k] = in ? __ldg(x + k * plane + o) : 0.0;
    }
    const unsigned cm = tile_classes(i0, j0, VSX, VSY, n);
    {
        int slot = 0;
        for (int c = 1; c < 9; ++c) {
            if (!((cm >> c) & 1u)) continue;
            const double* src = P.gbnd + c * 400;
            double* dst = gs + slot * 400;
            for (int q = t; q < 200; q += VS4_NT)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + 2 * q)), "l"(src + 2 * q)
                             : "memory");
            ++slot;
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    if (!XZERO) load_tile<T::XW, T::XH, 10, true, 4>(xs, x, i0 - 2, j0 - 2, n, pitch, plane, 0, t, VS4_NT);
    if (PROL) load_tile<VS_CW, VS_CH, 10, true, 4>(es, E.e, i0 / 2 - 1, j0 / 2 - 1, E.nc, E.pitchc, E.planec, 0, t, VS4_NT);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    if (stopv) return;
    if (PROL) {
        // coarse cell c = t % 32 (24 used), plane group grp: {0,1,2}, {3,4}, {5,6,7}, {8,9}
        constexpr int NCX = T::XW / 2, NCY = T::XH / 2;
        const int c = t & 31, pg = t >> 5;
        if (c < NCX * NCY && pg < 4) {
            const int cy = c / NCX, cx = c - cy * NCX;
            const int I = i0 / 2 - 1 + cx, J = j0 / 2 - 1 + cy;
            if (I >= 0 && J >= 0 && I < E.nc && J < E.nc) {
                const double* e0 = es + cy * VS_CW + cx;
#define EQ(dI, dJ, pl, wt) v = fma(wt, e0[(pl) * (VS_CW * VS_CH) + (dJ) * VS_CW + (dI)], v);
#define P2(dj, kf)                                                                       \
    {                                                                                    \
        double v = 0.0;                                                                  \
        MG_PROLONG_0_##dj##_##kf(EQ) const double v0 = v;                                \
        v = 0.0;                                                                         \
        MG_PROLONG_1_##dj##_##kf(EQ) const double v1 = v;                                \
        double* xp2 = xs + (kf) * (T::XW * T::XH) + (2 * cy + (dj)) * T::XW + 2 * cx;    \
        if (is_active(kf, 2 * I, 2 * J + (dj), n)) xp2[0] += v0;                         \
        if (is_active(kf, 2 * I + 1, 2 * J + (dj), n)) xp2[1] += v1;                     \
    }
#define P4(kf) P2(0, kf) P2(1, kf)
                if (pg == 0) { P4(0) P4(1) P4(2) }
                else if (pg == 1) { P4(3) P4(4) }
                else if (pg == 2) { P4(5) P4(6) P4(7) }
                else { P4(8) P4(9) }
#undef P4
#undef P2
#undef EQ
            }
        }
        __syncthreads();
        if (t < VSX * VSY) {
#pragma unroll
            for (int k = 0; k < 10; ++k) xown[k] = xs[k * (T::XW * T::XH) + (oy + 2) * T::XW + (ox + 2)];
        }
    }
    // phase 1: rows of group grp at residual position pos
    if (pos < T::RW * T::RH) {
        const int i = i0 - 1 + lx, j = j0 - 1 + ly;
        double av[10];
#pragma unroll
        for (int k = 0; k < 10; ++k) av[k] = 0.0;
        if (!XZERO) {
            const double* x0 = xs + (ly + 1) * T::XW + (lx + 1);
            if (grp == 0) apply_rows<T::XW * T::XH, false, RowGroup<0>::M>(L, x0 - T::XW, x0, x0 + T::XW, i, j, av);
            else if (grp == 1) apply_rows<T::XW * T::XH, false, RowGroup<1>::M>(L, x0 - T::XW, x0, x0 + T::XW, i, j, av);
            else if (grp == 2) apply_rows<T::XW * T::XH, false, RowGroup<2>::M>(L, x0 - T::XW, x0, x0 + T::XW, i, j, av);
            else apply_rows<T::XW * T::XH, false, RowGroup<3>::M>(L, x0 - T::XW, x0, x0 + T::XW, i, j, av);
            if (L.lamx != 0.0) exact_bubble_add(L.lamx, x0 - T::XW, x0, x0 + T::XW, T::XW * T::XH, av);
        }
#pragma unroll
        for (int k = 0; k < 10; ++k)
            if ((gm >> k) & 1u)
                rs[k * T::RW * T::RH + pos] = XZERO ? bpre[k] : (is_active(k, i, j, n) ? (bpre[k] - av[k]) : 0.0);
    }
    __syncthreads();
    // phase 2: patch part grp of vertex pos
    constexpr int OS = T::PW * T::PH;
    if (pos < OS) {
        const int py = pos / T::PW, px = pos - py * T::PW;
        const int a = i0 + px, bb = j0 + py;
        if (a <= n && bb <= n) {
            double rr[20];
            gather20<T::RW, T::RH>(rs + (py + 1) * T::RW + (px + 1), rr);
            const int cls = vertex_class(a, bb, n);
            double* out = cs + pos;
            if (cls == 0) {
                double hp[9], hm[11];
#pragma unroll
                for (int q = 0; q < 6; ++q) {
                    hp[q] = rr[2 + 2 * q] - rr[3 + 2 * q];
                    hm[2 + q] = rr[2 + 2 * q] + rr[3 + 2 * q];
                }
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    hp[6 + q] = rr[14 + 2 * q] + rr[15 + 2 * q];
                    hm[8 + q] = rr[14 + 2 * q] - rr[15 + 2 * q];
                }
                hm[0] = rr[0];
                hm[1] = rr[1];
                auto ymr = [&](int r) { double v = 0.0;
#pragma unroll
                    for (int c = 0; c < 11; ++c) v = fma(P.gmT[c][r], hm[c], v);
                    return v; };
                auto ypr = [&](int r) { double v = 0.0;
#pragma unroll
                    for (int c = 0; c < 9; ++c) v = fma(P.gpT[c][r], hp[c], v);
                    return v; };
                // output pair of unit q (0..5: (yp[q], ym[2+q]) -> 2+2q, 3+2q; 6..8: (yp[q], ym[2+q]) -> 14+2(q-6), +1)
                auto unit = [&](int q) {
                    const double p = ypr(q), m = ymr(2 + q);
                    if (q < 6) {
                        out[(2 + 2 * q) * OS] = m + p;
                        out[(3 + 2 * q) * OS] = m - p;
                    } else {
                        out[(14 + 2 * (q - 6)) * OS] = p + m;
                        out[(15 + 2 * (q - 6)) * OS] = p - m;
                    }
                };
                if (grp == 0) { out[0] = ymr(0); out[OS] = ymr(1); unit(0); unit(1); }
                else if (grp == 1) { unit(2); unit(3); unit(4); }
                else if (grp == 2) { unit(5); unit(6); }
                else { unit(7); unit(8); }
            } else {
                const double2* G = reinterpret_cast<const double2*>(gs + __popc(cm & ((1u << cls) - 1u)) * 400);
#pragma unroll
                for (int u = 0; u < 5; ++u) {
                    const int k = 5 * grp + u;
                    double sacc = 0.0;
#pragma unroll
                    for (int c2 = 0; c2 < 10; ++c2) {
                        const double2 g = G[k * 10 + c2];
                        sacc = fma(g.x, rr[2 * c2], sacc);
                        sacc = fma(g.y, rr[2 * c2 + 1], sacc);
                    }
                    out[k * OS] = sacc;
                }
            }
        } else {
#pragma unroll
            for (int u = 0; u < 5; ++u) cs[(5 * grp + u) * OS + pos] = 0.0;
        }
    }
    __syncthreads();
    double nrm = 0.0;
    if (t < VSX * VSY) {
        const int i = i0 + ox, j = j0 + oy;
        if (i <= n && j <= n) {
            const double* c00 = cs + oy * T::PW + ox;
#define CC(s_, dx, dy) c00[(s_) * (T::PW * T::PH) + (dy) * T::PW + (dx)]
            double d[10];
            d[0] = CC(0, 0, 0);
            d[1] = CC(1, 0, 0);
            d[2] = CC(2, 0, 0) + CC(3, 1, 0);
            d[3] = CC(4, 0, 0) + CC(5, 0, 1);
            d[4] = CC(6, 1, 0) + CC(7, 0, 1);
            d[5] = CC(8, 0, 0) + CC(9, 1, 0);
            d[6] = CC(10, 0, 0) + CC(11, 0, 1);
            d[7] = CC(12, 1, 0) + CC(13, 0, 1);
            d[8] = CC(14, 0, 0) + CC(16, 1, 0) + CC(19, 0, 1);
            d[9] = CC(15, 1, 1) + CC(17, 0, 1) + CC(18, 1, 0);
#undef CC
            const int64_t o = (int64_t)j * pitch + i;
            const double* r00 = rs + (oy + 1) * T::RW + (ox + 1);
#pragma unroll
            for (int k = 0; k < 10; ++k) {
                xo[k * plane + o] = is_active(k, i, j, n) ? fma(P.omega, d[k], xown[k]) : 0.0;
                const double rv = r00[k * T::RW * T::RH];
                nrm = fma(rv, rv, nrm);
            }
        }
    }
    if (S.out || S.state) norm_finish<VS4_NT>(S, nrm);
}

template <bool XZERO, int TX = VTX, int TY = VTY, bool HET = false>
__global__ void __launch_bounds__(VTile<TX, TY>::NT, 2) vanka_kernel(const VankaParams P, const double* __restrict__ x,
                                                       const double* __restrict__ b, double* __restrict__ xo,
                                                       NormSink S) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ double sm[];
    if (*P.L.stop) return;
    const double nrm =
        vanka_tile<XZERO, TX, TY, true, HET>(P, x, b, xo, blockIdx.x, blockIdx.y, threadIdx.x, sm, true);
    if (S.out || S.state) norm_finish<VTile<TX, TY>::NT>(S, nrm);
}

// heterogeneous-K sweep: the interior class table travels in the parameter block
#ifndef MG_HET_MINB
#define MG_HET_MINB 2   // CTAs per SM the heterogeneous sweep is compiled for (measured at 2048^2: 2 CTAs with 80
                        // registers and spills 1.33 ms per sweep, 1 CTA with 168 registers 1.51 ms)
#endif
template <bool XZERO, int TX = VTX, int TY = VTY>
__global__ void __launch_bounds__(VTile<TX, TY>::NT, MG_HET_MINB) vanka_het_kernel(const VankaParams P,
                                                           const __grid_constant__ HvInterior Ti,
                                                           const double* __restrict__ x, const double* __restrict__ b,
                                                           double* __restrict__ xo, NormSink S) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ double sm[];
    if (*P.L.stop) return;
    const double nrm =
        vanka_tile<XZERO, TX, TY, true, true>(P, x, b, xo, blockIdx.x, blockIdx.y, threadIdx.x, sm, true, &Ti);
    if (S.out || S.state) norm_finish<VTile<TX, TY>::NT>(S, nrm);
}

// ------------------------------------------------------------------------------------------
// restriction b_H = P^T r (R = P^T), optionally fused with r = b - A x
constexpr int CX = 16, CY = 4, CNT = 352;   // fine residual region 34 x 10 = 340 positions
constexpr int C_RW = 2 * CX + 2, C_RH = 2 * CY + 2, C_XW = C_RW + 2, C_XH = C_RH + 2;
constexpr int C_SMEM_FUSED = (10 * C_RW * C_RH + 10 * C_XW * C_XH) * 8;
constexpr int C_SMEM_PLAIN = 10 * C_RW * C_RH * 8;
// geometry of a restriction tile of CX x CY coarse indices (small tiles for the coarse levels)
template <int CX_, int CY_>
struct CTile {
    static constexpr int RW = 2 * CX_ + 2, RH = 2 * CY_ + 2, XW = RW + 2, XH = RH + 2;
    static constexpr int SMEM_FUSED = (10 * RW * RH + 10 * XW * XH) * 8, SMEM_PLAIN = 10 * RW * RH * 8;
    static constexpr int NT0 = RW * RH > 5 * CX_ * CY_ ? RW * RH : 5 * CX_ * CY_;
    static constexpr int NT = ((NT0 + 31) / 32) * 32;
};
constexpr int CSX = 4, CSY = 2;             // small restriction tiles: 64 threads

// one tile of the restriction (see vanka_tile for t / sm / active); both barriers are executed by
// every thread
template <int MODE, bool HET, int TX, int TY, bool NC>
__device__ __forceinline__ void restrict_tile(const LevelParams& L, int nc, int pitchc, const double* __restrict__ x,
                                              const double* __restrict__ br, double* __restrict__ bc, int bx,
                                              int by, int t, double* sm, bool active) {
    using T = CTile<TX, TY>;
    double* rs = sm;
    double* xs = sm + 10 * T::RW * T::RH;
    const int I0 = bx * TX, J0 = by * TY;
    const int fi0 = 2 * I0 - 2, fj0 = 2 * J0 - 2;
    if (MODE == 1) {
        if (active) load_tile<T::XW, T::XH, 10, NC>(xs, x, fi0 - 1, fj0 - 1, L.n, L.pitch, L.plane, 0, t, T::NT);
        __syncthreads();
        if (active && t < T::RW * T::RH) {
            const int ly = t / T::RW, lx = t - ly * T::RW;
            double rv[10];
            residual_at<T::XW, T::XH, HET, NC>(L, xs, lx + 1, ly + 1, fi0 + lx, fj0 + ly, br, rv);
#pragma unroll
            for (int k = 0; k < 10; ++k) rs[k * T::RW * T::RH + t] = rv[k];
        }
    } else {
        if (active) load_tile<T::RW, T::RH, 10, NC>(rs, br, fi0, fj0, L.n, L.pitch, L.plane, 0, t, T::NT);
    }
    __syncthreads();
    // coarse outputs: (coarse index, pair of planes) per thread; the plane pair is warp uniform
    if (!active || t >= 5 * TX * TY) return;
    const int c = t % (TX * TY), grp = t / (TX * TY);
    const int cy = c / TX, cx = c - cy * TX;
    const int I = I0 + cx, J = J0 + cy;
    if (I > nc || J > nc) return;
    const double* r00 = rs + (2 * cy + 2) * T::RW + (2 * cx + 2);
    const int64_t planec = (int64_t)(nc + 1) * pitchc;
    const int64_t o = (int64_t)J * pitchc + I;
#define RF(cdI, cdJ, di, dj, kf) r00[(kf) * (T::RW * T::RH) + (-2 * (cdJ) + (dj)) * T::RW + (-2 * (cdI) + (di))]
#define MG_T(cdI, cdJ, di, dj, kf, w) acc = fma(w, RF(cdI, cdJ, di, dj, kf), acc);
#define OUT(k)                                                       \
    {                                                                \
        double acc = 0.0;                                            \
        MG_RESTRICT_##k(MG_T) bc[k * planec + o] = is_active(k, I, J, nc) ? acc : 0.0; \
    }
    switch (grp) {
        case 0: OUT(0) OUT(1) break;
        case 1: OUT(2) OUT(3) break;
        case 2: OUT(4) OUT(5) break;
        case 3: OUT(6) OUT(7) break;
        default: OUT(8) OUT(9) break;
    }
#undef OUT
#undef MG_T
#undef RF
}

// Small-tile fused residual + restriction (4 x 2 coarse indices, 64 threads) with the stop flag, the x
// tile and b at the residual positions all read in the first round trip; bitwise restrict_tile<1>.
template <bool HET>
__global__ void __launch_bounds__(CTile<CSX, CSY>::NT, 4) restrict_small_kernel(const LevelParams L, int nc, int pitchc,
                                                                              const double* __restrict__ x,
                                                                              const double* __restrict__ br,
                                                                              double* __restrict__ bc) {
    pdl_wait();
    pdl_trigger();
    using T = CTile<CSX, CSY>;
    extern __shared__ double sm[];
    double* rs = sm;
    double* xs = sm + 10 * T::RW * T::RH;
    const int stopv = *L.stop;
    const int t = threadIdx.x;
    const int I0 = blockIdx.x * CSX, J0 = blockIdx.y * CSY;
    const int fi0 = 2 * I0 - 2, fj0 = 2 * J0 - 2;
    const int ly = t / T::RW, lx = t - ly * T::RW;
    const int i = fi0 + lx, j = fj0 + ly;
    double bpre[10];
    {
        const bool in = t < T::RW * T::RH && i >= 0 && j >= 0 && i <= L.n && j <= L.n;
        const int64_t o = in ? (int64_t)j * L.pitch + i : 0;
#pragma unroll
        for (int k = 0; k < 10; ++k) bpre[k] = in ? __ldg(br + k * L.plane + o) : 0.0;
    }
    load_tile<T::XW, T::XH, 10, true, 16>(xs, x, fi0 - 1, fj0 - 1, L.n, L.pitch, L.plane, 0, t, T::NT);
    __syncthreads();
    if (stopv) return;
    if (t < T::RW * T::RH) {
        const double* x0 = xs + (ly + 1) * T::XW + (lx + 1);
        double av[10];
        apply_rows<T::XW * T::XH, HET>(L, x0 - T::XW, x0, x0 + T::XW, i, j, av);
        if (L.lamx != 0.0) exact_bubble_add(L.lamx, x0 - T::XW, x0, x0 + T::XW, T::XW * T::XH, av);
#pragma unroll
        for (int k = 0; k < 10; ++k) rs[k * T::RW * T::RH + t] = is_active(k, i, j, L.n) ? (bpre[k] - av[k]) : 0.0;
    }
    __syncthreads();
    if (t >= 5 * CSX * CSY) return;
    const int c = t % (CSX * CSY), grp = t / (CSX * CSY);
    const int cy = c / CSX, cx = c - cy * CSX;
    const int I = I0 + cx, J = J0 + cy;
    if (I > nc || J > nc) return;
    const double* r00 = rs + (2 * cy + 2) * T::RW + (2 * cx + 2);
    const int64_t planec = (int64_t)(nc + 1) * pitchc;
    const int64_t o = (int64_t)J * pitchc + I;
#define RF(cdI, cdJ, di, dj, kf) r00[(kf) * (T::RW * T::RH) + (-2 * (cdJ) + (dj)) * T::RW + (-2 * (cdI) + (di))]
#define MG_T(cdI, cdJ, di, dj, kf, w) acc = fma(w, RF(cdI, cdJ, di, dj, kf), acc);
#define OUT(k)                                                       \
    {                                                                \
        double acc = 0.0;                                            \
        MG_RESTRICT_##k(MG_T) bc[k * planec + o] = is_active(k, I, J, nc) ? acc : 0.0; \
    }
    switch (grp) {
        case 0: OUT(0) OUT(1) break;
        case 1: OUT(2) OUT(3) break;
        case 2: OUT(4) OUT(5) break;
        case 3: OUT(6) OUT(7) break;
        default: OUT(8) OUT(9) break;
    }
#undef OUT
#undef MG_T
#undef RF
}

template <int MODE, bool HET, int TX = CX, int TY = CY>
__global__ void __launch_bounds__(CTile<TX, TY>::NT, 2) restrict_kernel(const LevelParams L, int nc, int pitchc,
                                                          const double* __restrict__ x,
                                                          const double* __restrict__ br,
                                                          double* __restrict__ bc) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ double sm[];
    if (*L.stop) return;
    restrict_tile<MODE, HET, TX, TY, true>(L, nc, pitchc, x, br, bc, blockIdx.x, blockIdx.y, threadIdx.x, sm, true);
}

// ------------------------------------------------------------------------------------------
// prolongation x_f += P e_c: one thread per coarse cell writes its 4 fine indices
// EARLY (the latency-bound coarse levels): the stop flag, the 20 fine pairs and the 20 coarse values are
// all read before the flag is tested -- one round trip instead of three; the bandwidth-bound large
// levels keep the stop test first (fewer registers in flight, more CTAs per SM).  Same arithmetic.
template <bool EARLY>
__global__ void __launch_bounds__(256) prolong_kernel(int nf, int pitchf, int nc, int pitchc,
                                                      const double* __restrict__ e, double* __restrict__ x,
                                                      const int* __restrict__ stop) {
    pdl_wait();
    pdl_trigger();
    if (!EARLY && *stop) return;
    const int stopv = EARLY ? *stop : 0;
    const int I = blockIdx.x * 32 + (threadIdx.x & 31), J = blockIdx.y * 8 + (threadIdx.x >> 5);
    if (I >= nc || J >= nc) return;
    const int64_t planec = (int64_t)(nc + 1) * pitchc, planef = (int64_t)(nf + 1) * pitchf;
    const double* e0 = e + (int64_t)J * pitchc + I;
    const int fi = 2 * I, fj = 2 * J;
    double* x0 = x + (int64_t)fj * pitchf + fi;   // fi even, rows 256-B aligned: 16-B aligned pairs
    // the two fine columns 2I, 2I+1 of a fine row move as one 16-byte load / store (a warp covers
    // 512 contiguous bytes per instruction); all 20 pairs are loaded before the first store (a
    // load after a store to the same array cannot be hoisted by the compiler: 20 serial round trips)
    double2 xq[20];
#pragma unroll
    for (int q = 0; q < 20; ++q) xq[q] = *reinterpret_cast<const double2*>(x0 + (q >> 1) * planef + (q & 1) * pitchf);
    double pe[20];
    if (EARLY) {
#define PL(dI, dJ, pl) pe[pslot20(dI, dJ, pl)] = __ldg(e0 + (pl) * planec + (dJ) * pitchc + (dI));
        PL(0, 0, 0) PL(0, 0, 1) PL(0, 0, 2) PL(0, 0, 3) PL(0, 0, 4) PL(0, 1, 0) PL(0, 1, 1)
        PL(0, 1, 2) PL(1, 0, 0) PL(1, 0, 1) PL(1, 0, 3) PL(1, 1, 0) PL(1, 1, 1)
        PL(0, 0, 5) PL(0, 0, 6) PL(0, 0, 7) PL(0, 0, 8) PL(0, 0, 9) PL(0, 1, 5) PL(1, 0, 6)
#undef PL
        if (stopv) return;
    }
#define MG_Q(dI, dJ, pl, w) v = fma(w, EARLY ? pe[pslot20(dI, dJ, pl)] : __ldg(e0 + (pl) * planec + (dJ) * pitchc + (dI)), v);
#define PROL2(dj, kf)                                                                   \
    {                                                                                   \
        double v = 0.0;                                                                 \
        MG_PROLONG_0_##dj##_##kf(MG_Q) const double v0 = v;                             \
        v = 0.0;                                                                        \
        MG_PROLONG_1_##dj##_##kf(MG_Q) const double v1 = v;                             \
        double2 xv = xq[2 * kf + dj];                                                   \
        if (is_active(kf, fi, fj + dj, nf)) xv.x += v0;                                 \
        if (is_active(kf, fi + 1, fj + dj, nf)) xv.y += v1;                             \
        *reinterpret_cast<double2*>(x0 + kf * planef + dj * pitchf) = xv;               \
    }
#define PROL4(kf) PROL2(0, kf) PROL2(1, kf)
    PROL4(0) PROL4(1) PROL4(2) PROL4(3) PROL4(4) PROL4(5) PROL4(6) PROL4(7) PROL4(8) PROL4(9)
#undef PROL4
#undef PROL2
#undef MG_Q
}

// Bandwidth-bound levels (nf > 256): the same chains with the ten fine planes split over blockIdx.z
// (two planes per thread: 4 fine pairs in flight, ~40 registers, full occupancy; prolong_kernel<false>
// holds all 20 pairs in 136 registers -> one 256-thread CTA per SM, 2.4 TB/s at 2048^2).  Bitwise
// prolong_kernel: every output is the same FMA chain in table order.
__global__ void __launch_bounds__(256) prolong_planes_kernel(int nf, int pitchf, int nc, int pitchc,
                                                             const double* __restrict__ e, double* __restrict__ x,
                                                             const int* __restrict__ stop) {
    pdl_wait();
    pdl_trigger();
    if (*stop) return;
    const int I = blockIdx.x * 32 + (threadIdx.x & 31), J = blockIdx.y * 8 + (threadIdx.x >> 5);
    if (I >= nc || J >= nc) return;
    const int64_t planec = (int64_t)(nc + 1) * pitchc, planef = (int64_t)(nf + 1) * pitchf;
    const double* e0 = e + (int64_t)J * pitchc + I;
    const int fi = 2 * I, fj = 2 * J;
    double* x0 = x + (int64_t)fj * pitchf + fi;
    const int ka = 2 * blockIdx.z;   // planes ka, ka + 1
    double2 xq[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) xq[q] = *reinterpret_cast<const double2*>(x0 + (ka + (q >> 1)) * planef + (q & 1) * pitchf);
#define MG_Q(dI, dJ, pl, w) v = fma(w, __ldg(e0 + (pl) * planec + (dJ) * pitchc + (dI)), v);
#define PROL2(dj, kf, slot)                                                             \
    {                                                                                   \
        double v = 0.0;                                                                 \
        MG_PROLONG_0_##dj##_##kf(MG_Q) const double v0 = v;                             \
        v = 0.0;                                                                        \
        MG_PROLONG_1_##dj##_##kf(MG_Q) const double v1 = v;                             \
        double2 xv = xq[slot];                                                          \
        if (is_active(kf, fi, fj + dj, nf)) xv.x += v0;                                 \
        if (is_active(kf, fi + 1, fj + dj, nf)) xv.y += v1;                             \
        *reinterpret_cast<double2*>(x0 + kf * planef + dj * pitchf) = xv;               \
    }
#define PROL8(ka_, kb_) PROL2(0, ka_, 0) PROL2(1, ka_, 1) PROL2(0, kb_, 2) PROL2(1, kb_, 3)
    switch (blockIdx.z) {
        case 0: PROL8(0, 1) break;
        case 1: PROL8(2, 3) break;
        case 2: PROL8(4, 5) break;
        case 3: PROL8(6, 7) break;
        default: PROL8(8, 9) break;
    }
#undef PROL8
#undef PROL2
#undef MG_Q
}

// ------------------------------------------------------------------------------------------
// Bottom of the V-cycle in ONE CTA (Vanka, levels with n <= 32 down to the coarsest): the same tile
// functions as the per-level kernels, run by 16 virtual blocks of 64 threads over the tiles of a
// level in rounds, with CTA barriers between the steps instead of kernel boundaries.  Loads are
// plain (not read-only path): the kernel reads what it wrote.  Bitwise the per-level sequence.
constexpr int BOT_VB = 8, BOT_NT = BOT_VB * 64;
constexpr int BOT_VSM = VTile<VSX, VSY>::SMEM > CTile<CSX, CSY>::SMEM_FUSED ? VTile<VSX, VSY>::SMEM
                                                                           : CTile<CSX, CSY>::SMEM_FUSED;
constexpr int BOT_SMEM = BOT_VB * BOT_VSM;
static_assert(VTile<VSX, VSY>::NT == 64 && CTile<CSX, CSY>::NT == 64, "virtual blocks of 64 threads");
static_assert(BOT_SMEM <= 227 * 1024, "bottom kernel shared memory");

__global__ void __launch_bounds__(BOT_NT, 1) bottom_kernel(const __grid_constant__ BottomArgs A) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ double sm[];
    if (*A.stop) return;
    // grid-wide when launched cooperatively over several CTAs (gridDim.x > 1), one CTA otherwise
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    auto gsync = [&]() {
        if (gridDim.x > 1) grid.sync();
        else __syncthreads();
    };
    const int vb = threadIdx.x >> 6, t = threadIdx.x & 63;
    const int gvb = blockIdx.x * BOT_VB + vb, nvb = gridDim.x * BOT_VB;   // global virtual block
    double* vsm = sm + vb * (BOT_VSM / 8);
    auto relax = [&](int l, const double* xin, double* xo, bool xzero) {
        const VankaParams& P = A.vp[l];
        const int n = P.L.n, tx = (n + VSX) / VSX, ntiles = tx * ((n + VSY) / VSY);
        for (int r0 = 0; r0 < ntiles; r0 += nvb) {   // rounds: uniform over the grid
            const int tile = r0 + gvb;
            const bool act = tile < ntiles;
            const int bx = act ? tile % tx : 0, by = act ? tile / tx : 0;
            if (xzero) vanka_tile<true, VSX, VSY, false>(P, xin, A.b[l], xo, bx, by, t, vsm, act);
            else vanka_tile<false, VSX, VSY, false>(P, xin, A.b[l], xo, bx, by, t, vsm, act);
            __syncthreads();
        }
        gsync();
    };
    auto restrict_ = [&](int l, const double* xl) {
        const LevelParams& L = A.vp[l].L;
        const int nc = L.n / 2, tx = (nc + CSX) / CSX, ntiles = tx * ((nc + CSY) / CSY);
        for (int r0 = 0; r0 < ntiles; r0 += nvb) {
            const int tile = r0 + gvb;
            const bool act = tile < ntiles;
            const int bx = act ? tile % tx : 0, by = act ? tile / tx : 0;
            restrict_tile<1, false, CSX, CSY, false>(L, nc, A.pitch[l + 1], xl, A.b[l], A.b[l + 1], bx, by, t, vsm, act);
            __syncthreads();
        }
        gsync();
    };
    // x_f += P e_c on level l from e on level l + 1 (prolong_kernel's arithmetic, L2 loads)
    auto prolong_ = [&](int l, const double* e, double* x) {
        const int nf = A.vp[l].L.n, pitchf = A.vp[l].L.pitch, nc = nf / 2, pitchc = A.pitch[l + 1];
        const int64_t planec = (int64_t)(nc + 1) * pitchc, planef = (int64_t)(nf + 1) * pitchf;
        for (int cell = blockIdx.x * BOT_NT + threadIdx.x; cell < nc * nc; cell += gridDim.x * BOT_NT) {
            const int I = cell % nc, J = cell / nc;
            const double* e0 = e + (int64_t)J * pitchc + I;
#define EC(dI, dJ, pl) __ldcg(e0 + (pl) * planec + (dJ) * pitchc + (dI))
#define MG_Q(dI, dJ, pl, w) v = fma(w, EC(dI, dJ, pl), v);
            const int fi = 2 * I, fj = 2 * J;
            double* x0 = x + (int64_t)fj * pitchf + fi;
#define PROL2(dj, kf)                                                                   \
    {                                                                                   \
        double v = 0.0;                                                                 \
        MG_PROLONG_0_##dj##_##kf(MG_Q) const double v0 = v;                             \
        v = 0.0;                                                                        \
        MG_PROLONG_1_##dj##_##kf(MG_Q) const double v1 = v;                             \
        double2* p2 = reinterpret_cast<double2*>(x0 + kf * planef + dj * pitchf);       \
        double2 xv = __ldcg(p2);                                                        \
        if (is_active(kf, fi, fj + dj, nf)) xv.x += v0;                                 \
        if (is_active(kf, fi + 1, fj + dj, nf)) xv.y += v1;                             \
        *p2 = xv;                                                                       \
    }
#define PROL4(kf) PROL2(0, kf) PROL2(1, kf)
            PROL4(0) PROL4(1) PROL4(2) PROL4(3) PROL4(4) PROL4(5) PROL4(6) PROL4(7) PROL4(8) PROL4(9)
#undef PROL4
#undef PROL2
#undef MG_Q
#undef EC
        }
        gsync();
    };
    const int nl = A.nl;
    double* cur[BOT_MAXL + 1];
    for (int l = 0; l < nl; ++l) {
        double* a = A.x[l];
        double* tt = A.t[l];
        for (int k = 0; k < A.nu1; ++k) {
            relax(l, a, tt, k == 0);
            double* sw = a; a = tt; tt = sw;
        }
        restrict_(l, a);
        cur[l] = a;
    }
    // coarsest: x_c[slots] = G b_c[slots] (coarse_kernel's arithmetic), by CTA 0
    if (blockIdx.x == 0) {
        double* rb = sm;
        for (int k = threadIdx.x; k < A.N; k += BOT_NT) rb[k] = __ldcg(A.b[nl] + A.slots[k]);
        __syncthreads();
        for (int row = threadIdx.x; row < A.N; row += BOT_NT) {
            double acc = 0.0;
            for (int k = 0; k < A.N; ++k) acc = fma(__ldg(A.G + (int64_t)k * A.N + row), rb[k], acc);
            A.x[nl][A.slots[row]] = acc;
        }
    }
    gsync();
    cur[nl] = A.x[nl];
    for (int l = nl - 1; l >= 0; --l) {
        prolong_(l, cur[l + 1], cur[l]);
        double* a = cur[l];
        double* tt = (a == A.x[l]) ? A.t[l] : A.x[l];
        for (int k = 0; k < A.nu2; ++k) {
            relax(l, a, tt, false);
            double* sw = a; a = tt; tt = sw;
        }
        cur[l] = a;
    }
}

// ------------------------------------------------------------------------------------------
// coarsest solve: x[slots] = Ginv b[slots] (Ginv column major, deflation folded in)
__global__ void __launch_bounds__(256) coarse_kernel(int N, const double* __restrict__ G,
                                                     const int64_t* __restrict__ slots,
                                                     const double* __restrict__ b, double* __restrict__ x,
                                                     const int* __restrict__ stop) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ double rb[];
    if (*stop) return;
    for (int k = threadIdx.x; k < N; k += blockDim.x) rb[k] = __ldg(b + slots[k]);
    __syncthreads();
    for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < N; row += gridDim.x * blockDim.x) {
        // one FMA chain per row in k order; unrolled so the column loads of G are issued 16 ahead
        // instead of exposing one L2 round trip per k (the kernel is a 130-long latency chain)
        double acc = 0.0;
        int k = 0;
        for (; k + 16 <= N; k += 16) {
            double g[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) g[q] = __ldg(G + (int64_t)(k + q) * N + row);
#pragma unroll
            for (int q = 0; q < 16; ++q) acc = fma(g[q], rb[k + q], acc);
        }
        for (; k < N; ++k) acc = fma(__ldg(G + (int64_t)k * N + row), rb[k], acc);
        x[slots[row]] = acc;
    }
}

// small coarsest systems (N <= CS_MAXN): G staged in shared memory by cp.async while the right-hand side
// is gathered, then the same per-row FMA chains in k order (bitwise coarse_kernel) read from shared memory
constexpr int CS_MAXN = 160;
__global__ void __launch_bounds__(256) coarse_smem_kernel(int N, const double* __restrict__ G,
                                                          const int64_t* __restrict__ slots,
                                                          const double* __restrict__ b, double* __restrict__ x,
                                                          const int* __restrict__ stop) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(16) double csm[];
    double* gs = csm;                       // [N][N] column major (as G)
    double* rb = csm + ((N * N + 1) & ~1);  // [N]
    const int stopv = *stop;
    const int NN = N * N;
    for (int q = threadIdx.x; 2 * q + 1 < NN; q += blockDim.x)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(gs + 2 * q)), "l"(G + 2 * q) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    if ((NN & 1) && threadIdx.x == 0) gs[NN - 1] = __ldg(G + NN - 1);
    for (int k = threadIdx.x; k < N; k += blockDim.x) rb[k] = __ldg(b + slots[k]);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    if (stopv) return;
    for (int row = threadIdx.x; row < N; row += blockDim.x) {
        double acc = 0.0;
#pragma unroll 8
        for (int k = 0; k < N; ++k) acc = fma(gs[k * N + row], rb[k], acc);
        x[slots[row]] = acc;
    }
}

// ------------------------------------------------------------------------------------------
// inexact Braess-Sarazin
constexpr int BTX = 32, BTY = 8, BANT = 416, BBNT = 352;   // one position per thread in every phase

__device__ __forceinline__ void patch_apply8(const DispParams& U, int cls, const double rr[8], double* out, int os) {
    if (cls == 0) {
        double hp[3], hm[5];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            hp[q] = rr[2 + 2 * q] - rr[3 + 2 * q];
            hm[2 + q] = rr[2 + 2 * q] + rr[3 + 2 * q];
        }
        hm[0] = rr[0];
        hm[1] = rr[1];
        double yp[3] = {0, 0, 0}, ym[5] = {0, 0, 0, 0, 0};
#pragma unroll
        for (int c = 0; c < 5; ++c) {
#pragma unroll
            for (int a = 0; a < 5; ++a) ym[a] = fma(U.umT[c][a], hm[c], ym[a]);
            if (c < 3) {
#pragma unroll
                for (int a = 0; a < 3; ++a) yp[a] = fma(U.upT[c][a], hp[c], yp[a]);
            }
        }
        out[0] = ym[0];
        out[os] = ym[1];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            out[(2 + 2 * q) * os] = ym[2 + q] + yp[q];
            out[(3 + 2 * q) * os] = ym[2 + q] - yp[q];
        }
    } else {
        const double* G = U.ubnd + cls * 64;
#pragma unroll 1
        for (int a = 0; a < 8; ++a) {
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < 8; ++c) s = fma(__ldg(G + a * 8 + c), rr[c], s);
            out[a * os] = s;
        }
    }
}

template <int RW, int RH>
__device__ __forceinline__ void gather8(const double* r00, double rr[8]) {
#define RR(dx, dy, pl) r00[(pl) * (RW * RH) + (dy) * RW + (dx)]
    rr[0] = RR(0, 0, 0);  rr[1] = RR(0, 0, 1);
    rr[2] = RR(0, 0, 2);  rr[3] = RR(-1, 0, 2); rr[4] = RR(0, 0, 3); rr[5] = RR(0, -1, 3);
    rr[6] = RR(-1, 0, 4); rr[7] = RR(0, -1, 4);
#undef RR
}

// D_w(e) = mu_f h^2 sum_{T ni e} K_T^{-1} (M_w1)_T[e][e] for the RT0 DoF of plane k at index (i, j)
template <bool HET>
__device__ __forceinline__ double Dw_at(const LevelParams& L, int k, int i, int j) {
    double d = 0.0;
#define MG_I(kk, cdx, cdy, sh, q) d = fma(L.mw1d[sh][(q) - 9], kinv_at<HET>(L, i + (cdx), j + (cdy), sh), d);
    if (k == 5) { MG_INCIDENT_5(MG_I) }
    else if (k == 6) { MG_INCIDENT_6(MG_I) }
    else { MG_INCIDENT_7(MG_I) }
#undef MG_I
    return d;
}

// active-edge flags of the local edges of triangle sh in cell (i, j)
__device__ __forceinline__ void tri_edges_active(int sh, int i, int j, int n, bool act[3]) {
    if (sh == 0) {
        act[0] = is_active(5, i, j, n);
        act[1] = is_active(6, i, j, n);
        act[2] = true;
    } else {
        act[0] = is_active(5, i, j + 1, n);
        act[1] = is_active(6, i + 1, j, n);
        act[2] = true;
    }
}

// D_w of the local edges of triangle sh in cell (i, j)
template <bool HET>
__device__ __forceinline__ void tri_Dw(const LevelParams& L, int sh, int i, int j, double dw[3]) {
    if (sh == 0) {
        dw[0] = Dw_at<HET>(L, 5, i, j);
        dw[1] = Dw_at<HET>(L, 6, i, j);
    } else {
        dw[0] = Dw_at<HET>(L, 5, i, j + 1);
        dw[1] = Dw_at<HET>(L, 6, i + 1, j);
    }
    dw[2] = Dw_at<HET>(L, 7, i, j);
}

// diag(S)_T = s0 |T| + tau sum_{e in T active} Bw_T[e]^2 / D_w(e)
template <bool HET>
__device__ __forceinline__ double diagS(const LevelParams& L, int sh, int i, int j) {
    double dw[3];
    bool act[3];
    tri_Dw<HET>(L, sh, i, j, dw);
    tri_edges_active(sh, i, j, L.n, act);
    double s = L.s0h2;
#pragma unroll
    for (int e = 0; e < 3; ++e)
        if (act[e]) s += L.tau * L.bw[sh][e] * L.bw[sh][e] / dw[e];
    return s;
}

// stage A: r, z_u = F_u^{-1} r_u, z_w = (tau D_w)^{-1} r_w, g = alpha B_u z_u + tau B_w z_w - r_p,
// first Jacobi sweep dp = omega_J g / diag(S)
constexpr int BA_XW = BTX + 5, BA_XH = BTY + 5, BA_RW = BTX + 3, BA_RH = BTY + 3;
constexpr int BA_ZW = BTX + 2, BA_ZH = BTY + 2, BA_UW = BTX + 1, BA_UH = BTY + 1;
constexpr int BA_XSZ = 10 * BA_XW * BA_XH, BA_ZSZ = 8 * BA_ZW * BA_ZH + 5 * BA_UW * BA_UH;
constexpr int BA_USZ = BA_XSZ > BA_ZSZ ? BA_XSZ : BA_ZSZ;
constexpr int BA_SMEM = (BA_USZ + 10 * BA_RW * BA_RH) * 8;

// stage-A tile geometry for TX x TY owned cells (small tiles on the latency-bound coarse levels)
template <int TX, int TY>
struct BATile {
    static constexpr int XW = TX + 5, XH = TY + 5, RW = TX + 3, RH = TY + 3, ZW = TX + 2, ZH = TY + 2;
    static constexpr int UW = TX + 1, UH = TY + 1;
    static constexpr int XSZ = 10 * XW * XH, ZSZ = 8 * ZW * ZH + 5 * UW * UH, USZ = XSZ > ZSZ ? XSZ : ZSZ;
    static constexpr int SMEM = (USZ + 10 * RW * RH) * 8;
    static constexpr int NT = ((RW * RH + 31) / 32) * 32;
};
template <bool HET, bool XZERO, int TX = BTX, int TY = BTY>
__global__ void __launch_bounds__(BATile<TX, TY>::NT, 2) bsr_a_kernel(const LevelParams L, const DispParams U, double omJ,
                                                       const double* __restrict__ x, const double* __restrict__ b,
                                                       double* __restrict__ g, double* __restrict__ dp, NormSink S) {
    pdl_wait();
    pdl_trigger();
    using T = BATile<TX, TY>;
    extern __shared__ double sm[];
    double* xs = sm;
    double* zs = sm;                              // disp patch outputs, overlays xs
    double* zu = sm + 8 * T::ZW * T::ZH;          // z_u on owned + high ring
    double* rs = sm + T::USZ;
    if (*L.stop) return;
    const int n = L.n, pitch = L.pitch;
    const int64_t plane = L.plane;
    const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
    if (!XZERO) {
        // b of this thread's residual position travels with the x tile (one round trip instead of two)
        constexpr bool PRE = TX <= 8;   // small (latency-bound) tiles only
        double bp[10];
        if (PRE) {
            const int t = threadIdx.x, ly = t / T::RW, lx = t - ly * T::RW;
            load_b10(L, b, i0 - 1 + lx, j0 - 1 + ly, t < T::RW * T::RH, bp);
        }
        load_tile<T::XW, T::XH, 10>(xs, x, i0 - 2, j0 - 2, n, pitch, plane);
        __syncthreads();
        if (const int t = threadIdx.x; t < T::RW * T::RH) {
            const int ly = t / T::RW, lx = t - ly * T::RW;
            double rv[10];
            if (PRE) residual_at_b<T::XW, T::XH, HET>(L, xs, lx + 1, ly + 1, i0 - 1 + lx, j0 - 1 + ly, bp, rv);
            else residual_at<T::XW, T::XH, HET>(L, xs, lx + 1, ly + 1, i0 - 1 + lx, j0 - 1 + ly, b, rv);
#pragma unroll
            for (int k = 0; k < 10; ++k) rs[k * T::RW * T::RH + t] = rv[k];
        }
    } else {
        load_tile<T::RW, T::RH, 10>(rs, b, i0 - 1, j0 - 1, n, pitch, plane);
    }
    __syncthreads();
    // displacement patches at vertices [i0, i0+TX+1] x [j0, j0+TY+1]
    if (const int t = threadIdx.x; t < T::ZW * T::ZH) {
        const int py = t / T::ZW, px = t - py * T::ZW;
        const int a = i0 + px, bb = j0 + py;
        if (a <= n && bb <= n) {
            double rr[8];
            gather8<T::RW, T::RH>(rs + (py + 1) * T::RW + (px + 1), rr);
            patch_apply8(U, vertex_class(a, bb, n), rr, zs + t, T::ZW * T::ZH);
        } else {
#pragma unroll
            for (int s = 0; s < 8; ++s) zs[s * T::ZW * T::ZH + t] = 0.0;
        }
    }
    __syncthreads();
    // z_u on indices [i0, i0+TX] x [j0, j0+TY]
    if (const int t = threadIdx.x; t < T::UW * T::UH) {
        const int ly = t / T::UW, lx = t - ly * T::UW;
        const double* c00 = zs + ly * T::ZW + lx;
#define CC(s, dx, dy) c00[(s) * (T::ZW * T::ZH) + (dy) * T::ZW + (dx)]
        zu[0 * T::UW * T::UH + t] = CC(0, 0, 0);
        zu[1 * T::UW * T::UH + t] = CC(1, 0, 0);
        zu[2 * T::UW * T::UH + t] = CC(2, 0, 0) + CC(3, 1, 0);
        zu[3 * T::UW * T::UH + t] = CC(4, 0, 0) + CC(5, 0, 1);
        zu[4 * T::UW * T::UH + t] = CC(6, 1, 0) + CC(7, 0, 1);
#undef CC
    }
    __syncthreads();
    const int lx = threadIdx.x % TX, ly = threadIdx.x / TX;
    const int i = i0 + lx, j = j0 + ly;
    double nrm = 0.0;
    if (threadIdx.x < TX * TY && i <= n && j <= n) {
        const double* r00 = rs + (ly + 1) * T::RW + (lx + 1);
        if (S.out || S.state) {
#pragma unroll
            for (int k = 0; k < 10; ++k) {
                const double rv = r00[k * T::RW * T::RH];
                nrm = fma(rv, rv, nrm);
            }
        }
        const int64_t o = (int64_t)j * pitch + i;
        if (i < n && j < n) {
            const double* u00 = zu + ly * T::UW + lx;
#pragma unroll
            for (int sh = 0; sh < 2; ++sh) {
                double dw[3];
                bool act[3];
                tri_Dw<HET>(L, sh, i, j, dw);
                tri_edges_active(sh, i, j, n, act);
                double gu = 0.0, gw = 0.0, ds = L.s0h2;
#define MG_L(s, q, dx, dy, pl)                                                              \
    if ((s) == sh) {                                                                        \
        if ((q) < 9) gu = fma(L.bu[s][(q) < 9 ? (q) : 0], u00[(pl) * (T::UW * T::UH) + (dy) * T::UW + (dx)], gu); \
        else if ((q) < 12) {                                                                \
            const int e = (q) < 12 ? (q) - 9 : 0;                                           \
            if (act[e]) {                                                                   \
                const double rw = r00[(pl) * (T::RW * T::RH) + (dy) * T::RW + (dx)];        \
                gw = fma(L.bw[s][e], rw / (L.tau * dw[e]), gw);                             \
                ds += L.tau * L.bw[s][e] * L.bw[s][e] / dw[e];                              \
            }                                                                               \
        }                                                                                   \
    }
                MG_LOCAL_0(MG_L)
                MG_LOCAL_1(MG_L)
#undef MG_L
                const double rp = r00[(8 + sh) * (T::RW * T::RH)];
                const double gv = L.alpha * gu + L.tau * gw - rp;
                g[sh * plane + o] = gv;
                dp[sh * plane + o] = omJ * gv / ds;
            }
        } else {
            g[o] = 0.0;
            g[plane + o] = 0.0;
            dp[o] = 0.0;
            dp[plane + o] = 0.0;
        }
    }
    if (S.out || S.state) norm_finish<T::NT>(S, nrm);
}

// Jacobi sweep on S dp = g: dp' = dp + omega_J (g - S dp) / diag(S)
template <bool HET>
__global__ void __launch_bounds__(256) bsr_jacobi_kernel(const LevelParams L, double omJ,
                                                         const double* __restrict__ g,
                                                         const double* __restrict__ dpi, double* __restrict__ dpo) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * 32 + (threadIdx.x & 31), j = blockIdx.y * 8 + (threadIdx.x >> 5);
    const int n = L.n;
    if (i > n || j > n || *L.stop) return;
    const int64_t plane = L.plane, pitch = L.pitch;
    const int64_t o = (int64_t)j * pitch + i;
    if (i == n || j == n) {
        dpo[o] = 0.0;
        dpo[plane + o] = 0.0;
        return;
    }
    // neighbours: LL(i,j) -- e0 H(i,j): UR(i,j-1); e1 V(i,j): UR(i-1,j); e2 D: UR(i,j)
    //             UR(i,j) -- e0 H(i,j+1): LL(i,j+1); e1 V(i+1,j): LL(i+1,j); e2 D: LL(i,j)
#pragma unroll
    for (int sh = 0; sh < 2; ++sh) {
        double dw[3];
        bool act[3];
        tri_Dw<HET>(L, sh, i, j, dw);
        tri_edges_active(sh, i, j, n, act);
        const double dself = __ldg(dpi + sh * plane + o);
        double ds = L.s0h2, off = 0.0;
#pragma unroll
        for (int e = 0; e < 3; ++e) {
            if (!act[e]) continue;
            const double c = L.tau * L.bw[sh][e] / dw[e];
            ds += c * L.bw[sh][e];
            int ni, nj;
            if (sh == 0) { ni = e == 1 ? i - 1 : i; nj = e == 0 ? j - 1 : j; }
            else         { ni = e == 1 ? i + 1 : i; nj = e == 0 ? j + 1 : j; }
            const double dn = __ldg(dpi + (1 - sh) * plane + (int64_t)nj * pitch + ni);
            off = fma(c * L.bw[1 - sh][e], dn, off);
        }
        const double sd = fma(ds, dself, off);
        dpo[sh * plane + o] = dself + omJ * (__ldg(g + sh * plane + o) - sd) / ds;
    }
}

// Per-level Jacobi table: tau / D_w(e) of the three RT0 edges owned by index
// (i, j) (0 if inactive) and 1 / diag(S) of its two triangles -- fixed by K^{-1}, formed once at
// setup so the Jacobi sweeps need neither the K^{-1} gathers nor divisions.  5 planes.
template <bool HET>
__global__ void __launch_bounds__(256) jtable_kernel(const LevelParams L, double* __restrict__ tab) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * 32 + (threadIdx.x & 31), j = blockIdx.y * 8 + (threadIdx.x >> 5);
    const int n = L.n;
    if (i > n || j > n) return;
    const int64_t plane = L.plane, o = (int64_t)j * L.pitch + i;
#pragma unroll
    for (int e = 0; e < 3; ++e)
        tab[e * plane + o] = is_active(5 + e, i, j, n) ? L.tau / Dw_at<HET>(L, 5 + e, i, j) : 0.0;
#pragma unroll
    for (int sh = 0; sh < 2; ++sh) {
        double v = 0.0;
        if (i < n && j < n) {
            double dw[3];
            bool act[3];
            tri_Dw<HET>(L, sh, i, j, dw);
            tri_edges_active(sh, i, j, n, act);
            double ds = L.s0h2;
#pragma unroll
            for (int e = 0; e < 3; ++e)
                if (act[e]) ds += L.tau * L.bw[sh][e] * L.bw[sh][e] / dw[e];
            v = 1.0 / ds;
        }
        tab[(3 + sh) * plane + o] = v;
    }
}

// Jacobi sweep with the table: dp' = dp + omega_J (g / diag S - dp - (S dp - diag(S) dp) / diag S)
template <int DUMMY = 0>
__global__ void __launch_bounds__(256) bsr_jacobi_t_kernel(const LevelParams L, double omJ,
                                                           const double* __restrict__ g,
                                                           const double* __restrict__ tab,
                                                           const double* __restrict__ dpi, double* __restrict__ dpo) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * 32 + (threadIdx.x & 31), j = blockIdx.y * 8 + (threadIdx.x >> 5);
    const int n = L.n;
    if (i > n || j > n || *L.stop) return;
    const int64_t plane = L.plane, pitch = L.pitch;
    const int64_t o = (int64_t)j * pitch + i;
    if (i == n || j == n) {
        dpo[o] = 0.0;
        dpo[plane + o] = 0.0;
        return;
    }
    // edge factors of the cell's triangles: LL -> H(i,j), V(i,j), D(i,j); UR -> H(i,j+1), V(i+1,j), D(i,j)
    const double tH0 = __ldg(tab + o), tV0 = __ldg(tab + plane + o), tD = __ldg(tab + 2 * plane + o);
    const double tH1 = __ldg(tab + o + pitch), tV1 = __ldg(tab + plane + o + 1);
#pragma unroll
    for (int sh = 0; sh < 2; ++sh) {
        const double te[3] = {sh == 0 ? tH0 : tH1, sh == 0 ? tV0 : tV1, tD};
        const double dself = __ldg(dpi + sh * plane + o);
        double off = 0.0;
#pragma unroll
        for (int e = 0; e < 3; ++e) {
            int ni, nj;
            if (sh == 0) { ni = e == 1 ? i - 1 : i; nj = e == 0 ? j - 1 : j; }
            else         { ni = e == 1 ? i + 1 : i; nj = e == 0 ? j + 1 : j; }
            if (te[e] != 0.0) {   // inactive edge: no coupling (and the neighbour may lie outside)
                const double dn = __ldg(dpi + (1 - sh) * plane + (int64_t)nj * pitch + ni);
                off = fma(te[e] * L.bw[sh][e] * L.bw[1 - sh][e], dn, off);
            }
        }
        const double ids = __ldg(tab + (3 + sh) * plane + o);
        dpo[sh * plane + o] = dself + omJ * (fma(__ldg(g + sh * plane + o), ids, -dself) - off * ids);
    }
}

// Two Jacobi sweeps with the table in one launch (round 2): a CTA owns 32 x 8 cells, runs the first sweep
// on the 34 x 10 cells around them into shared memory (the one-cell ring is recomputed, its inputs come
// from L2), then the second sweep on its own cells.  Each sweep is bsr_jacobi_t_kernel's expression, so
// the result is bitwise that of two launches; g, dp and the 5-plane table cross DRAM once instead of twice.
constexpr int J2_W = 34, J2_H = 10, J2_N = J2_W * J2_H;
__device__ __forceinline__ void jacobi_t_cell(const LevelParams& L, double omJ, const double* __restrict__ g,
                                              const double* __restrict__ tab, int i, int j, int64_t o,
                                              double dself0, double dself1, const double nb[2][3], double out[2]) {
    const int64_t plane = L.plane, pitch = L.pitch;
    const double tH0 = __ldg(tab + o), tV0 = __ldg(tab + plane + o), tD = __ldg(tab + 2 * plane + o);
    const double tH1 = __ldg(tab + o + pitch), tV1 = __ldg(tab + plane + o + 1);
#pragma unroll
    for (int sh = 0; sh < 2; ++sh) {
        const double te[3] = {sh == 0 ? tH0 : tH1, sh == 0 ? tV0 : tV1, tD};
        const double dself = sh == 0 ? dself0 : dself1;
        double off = 0.0;
#pragma unroll
        for (int e = 0; e < 3; ++e)
            if (te[e] != 0.0) off = fma(te[e] * L.bw[sh][e] * L.bw[1 - sh][e], nb[sh][e], off);
        const double ids = __ldg(tab + (3 + sh) * plane + o);
        out[sh] = dself + omJ * (fma(__ldg(g + sh * plane + o), ids, -dself) - off * ids);
    }
}

__global__ void __launch_bounds__(256) bsr_jacobi2_t_kernel(const LevelParams L, double omJ, const double* __restrict__ g,
                                                            const double* __restrict__ tab,
                                                            const double* __restrict__ dpi, double* __restrict__ dpo) {
    pdl_wait();
    pdl_trigger();
    __shared__ double d1[2 * J2_N];   // first-sweep dp of cells (i0 - 1 + lx, j0 - 1 + ly), [shape][ly][lx]
    const int n = L.n;
    if (*L.stop) return;
    const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 8;
    const int64_t plane = L.plane, pitch = L.pitch;
    // neighbours of LL(i,j): UR(i,j-1), UR(i-1,j), UR(i,j); of UR(i,j): LL(i,j+1), LL(i+1,j), LL(i,j)
    for (int c = threadIdx.x; c < J2_N; c += 256) {
        const int ly = c / J2_W, lx = c - ly * J2_W;
        const int i = i0 - 1 + lx, j = j0 - 1 + ly;
        double out[2] = {0.0, 0.0};
        if (i >= 0 && j >= 0 && i < n && j < n) {
            const int64_t o = (int64_t)j * pitch + i;
            const double tH0 = __ldg(tab + o), tV0 = __ldg(tab + plane + o), tD = __ldg(tab + 2 * plane + o);
            const double tH1 = __ldg(tab + o + pitch), tV1 = __ldg(tab + plane + o + 1);
            const double s0 = __ldg(dpi + o), s1 = __ldg(dpi + plane + o);
            double nb[2][3];
            nb[0][0] = tH0 != 0.0 ? __ldg(dpi + plane + o - pitch) : 0.0;
            nb[0][1] = tV0 != 0.0 ? __ldg(dpi + plane + o - 1) : 0.0;
            nb[0][2] = s1;
            nb[1][0] = tH1 != 0.0 ? __ldg(dpi + o + pitch) : 0.0;
            nb[1][1] = tV1 != 0.0 ? __ldg(dpi + o + 1) : 0.0;
            nb[1][2] = s0;
            jacobi_t_cell(L, omJ, g, tab, i, j, o, s0, s1, nb, out);
        }
        d1[c] = out[0];
        d1[J2_N + c] = out[1];
    }
    __syncthreads();
    const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;
    const int i = i0 + lx, j = j0 + ly;
    if (i > n || j > n) return;
    const int64_t o = (int64_t)j * pitch + i;
    if (i == n || j == n) {
        dpo[o] = 0.0;
        dpo[plane + o] = 0.0;
        return;
    }
    const double* c0 = d1 + (ly + 1) * J2_W + (lx + 1);   // LL plane at the cell
    const double* c1 = c0 + J2_N;                         // UR plane
    double nb[2][3];
    nb[0][0] = c1[-J2_W];
    nb[0][1] = c1[-1];
    nb[0][2] = c1[0];
    nb[1][0] = c0[J2_W];
    nb[1][1] = c0[1];
    nb[1][2] = c0[0];
    double out[2];
    jacobi_t_cell(L, omJ, g, tab, i, j, o, c0[0], c1[0], nb, out);
    dpo[o] = out[0];
    dpo[plane + o] = out[1];
}

// stage B: du = F_u^{-1}(r_u - alpha B_u^T dp), dw = (r_w - tau B_w^T dp)/(tau D_w),
// xout = x + omega (du, dw, dp)
constexpr int BB_XW = BTX + 4, BB_XH = BTY + 4, BB_RW = BTX + 2, BB_RH = BTY + 2;
constexpr int BB_PW = BTX + 1, BB_PH = BTY + 1, BB_DW = BTX + 3, BB_DH = BTY + 3;
constexpr int BB_XSZ = 10 * BB_XW * BB_XH, BB_ZSZ = 8 * BB_PW * BB_PH;
constexpr int BB_USZ = BB_XSZ > BB_ZSZ ? BB_XSZ : BB_ZSZ;
constexpr int BB_SMEM = (BB_USZ + 10 * BB_RW * BB_RH + 2 * BB_DW * BB_DH) * 8;

template <int TX, int TY>
struct BBTile {
    static constexpr int XW = TX + 4, XH = TY + 4, RW = TX + 2, RH = TY + 2, PW = TX + 1, PH = TY + 1;
    static constexpr int DW = TX + 3, DH = TY + 3;
    static constexpr int XSZ = 10 * XW * XH, ZSZ = 8 * PW * PH, USZ = XSZ > ZSZ ? XSZ : ZSZ;
    static constexpr int SMEM = (USZ + 10 * RW * RH + 2 * DW * DH) * 8;
    static constexpr int NT = ((RW * RH + 31) / 32) * 32;
};
template <bool HET, bool XZERO, int TX = BTX, int TY = BTY>
__global__ void __launch_bounds__(BBTile<TX, TY>::NT, 2) bsr_b_kernel(const LevelParams L, const DispParams U, double omega,
                                                       const double* __restrict__ x, const double* __restrict__ b,
                                                       const double* __restrict__ dp, double* __restrict__ xo,
                                                       const double* __restrict__ jg, const double* __restrict__ jtab,
                                                       double omJ) {
    pdl_wait();
    pdl_trigger();
    using T = BBTile<TX, TY>;
    extern __shared__ double sm[];
    double* xs = sm;
    double* zs = sm;
    double* rs = sm + T::USZ;
    double* ps = rs + 10 * T::RW * T::RH;   // dp on cells [i0-2, i0+TX] x [j0-2, j0+TY]
    if (*L.stop) return;
    const int n = L.n, pitch = L.pitch;
    const int64_t plane = L.plane;
    const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
    // this thread's owner x, the D_w of its RT0 DoFs and b of its residual position: issued with the first
    // round trip of the kernel instead of at their uses (latency-bound levels)
    // (small tiles only: the 32 x 8 tile runs at its 80-register cap and is bandwidth- rather than latency-bound)
    constexpr bool PRE = TX <= 8;
    double xown[10], dwown[3], bp[10];
    if (PRE) {
        const int olx = threadIdx.x % TX, oly = threadIdx.x / TX, oi = i0 + olx, oj = j0 + oly;
        const bool own = threadIdx.x < TX * TY && oi <= n && oj <= n;
        const int64_t oo = own ? (int64_t)oj * pitch + oi : 0;
#pragma unroll
        for (int k = 0; k < 10; ++k) xown[k] = (!XZERO && own) ? __ldg(x + k * plane + oo) : 0.0;
#pragma unroll
        for (int k = 5; k < 8; ++k) dwown[k - 5] = own ? Dw_at<HET>(L, k, oi, oj) : 1.0;
        const int t = threadIdx.x, ly = t / T::RW, lx = t - ly * T::RW;
        if (!XZERO) load_b10(L, b, i0 - 1 + lx, j0 - 1 + ly, t < T::RW * T::RH, bp);
    }
    if (jg) {
        // the last two table Jacobi sweeps fused in (latency-bound levels: one launch less per relaxation):
        // dp on the cells two rings further out, one sweep into q2, the second into ps -- each cell the
        // expression of bsr_jacobi_t_kernel, so ps is bitwise what two launches would have left in dp
        constexpr int W1 = T::DW + 4, H1 = T::DH + 4, W2 = T::DW + 2, H2 = T::DH + 2;
        static_assert(2 * W1 * H1 + 2 * W2 * H2 <= T::USZ, "Jacobi scratch aliases the x tile");
        double* q1 = sm;
        double* q2 = q1 + 2 * W1 * H1;
        for (int t = threadIdx.x; t < 2 * W1 * H1; t += T::NT) {
            const int sh = t / (W1 * H1), rem = t - sh * (W1 * H1);
            const int ly = rem / W1, lx = rem - ly * W1;
            const int ci = i0 - 4 + lx, cj = j0 - 4 + ly;
            q1[t] = (ci >= 0 && cj >= 0 && ci < n && cj < n) ? __ldg(dp + sh * plane + (int64_t)cj * pitch + ci) : 0.0;
        }
        __syncthreads();
        auto sweep = [&](const double* src, int WS, int HS, double* dst, int WD, int HD, int org) {
            // dst cell (lx, ly) = mesh cell (i0 - org + lx, j0 - org + ly) = src cell (lx + 1, ly + 1)
            for (int t = threadIdx.x; t < WD * HD; t += T::NT) {
                const int ly = t / WD, lx = t - ly * WD;
                const int ci = i0 - org + lx, cj = j0 - org + ly;
                double out[2] = {0.0, 0.0};
                if (ci >= 0 && cj >= 0 && ci < n && cj < n) {
                    const double* p0 = src + (ly + 1) * WS + (lx + 1);
                    const double* p1 = p0 + WS * HS;
                    double nb[2][3];
                    nb[0][0] = p1[-WS];
                    nb[0][1] = p1[-1];
                    nb[0][2] = p1[0];
                    nb[1][0] = p0[WS];
                    nb[1][1] = p0[1];
                    nb[1][2] = p0[0];
                    jacobi_t_cell(L, omJ, jg, jtab, ci, cj, (int64_t)cj * pitch + ci, p0[0], p1[0], nb, out);
                }
                dst[t] = out[0];
                dst[WD * HD + t] = out[1];
            }
        };
        sweep(q1, W1, H1, q2, W2, H2, 3);
        __syncthreads();
        sweep(q2, W2, H2, ps, T::DW, T::DH, 2);
        __syncthreads();   // q1 / q2 alias the x tile loaded next
    } else {
        for (int t = threadIdx.x; t < 2 * T::DW * T::DH; t += T::NT) {
            const int sh = t / (T::DW * T::DH), rem = t - sh * (T::DW * T::DH);
            const int ly = rem / T::DW, lx = rem - ly * T::DW;
            const int ci = i0 - 2 + lx, cj = j0 - 2 + ly;
            ps[t] = (ci >= 0 && cj >= 0 && ci < n && cj < n) ? __ldg(dp + sh * plane + (int64_t)cj * pitch + ci) : 0.0;
        }
    }
    if (!XZERO) {
        load_tile<T::XW, T::XH, 10>(xs, x, i0 - 2, j0 - 2, n, pitch, plane);
        __syncthreads();
        if (const int t = threadIdx.x; t < T::RW * T::RH) {
            const int ly = t / T::RW, lx = t - ly * T::RW;
            double rv[10];
            if (PRE) residual_at_b<T::XW, T::XH, HET>(L, xs, lx + 1, ly + 1, i0 - 1 + lx, j0 - 1 + ly, bp, rv);
            else residual_at<T::XW, T::XH, HET>(L, xs, lx + 1, ly + 1, i0 - 1 + lx, j0 - 1 + ly, b, rv);
#pragma unroll
            for (int k = 0; k < 8; ++k) rs[k * T::RW * T::RH + t] = rv[k];
        }
    } else {
        load_tile<T::RW, T::RH, 8>(rs, b, i0 - 1, j0 - 1, n, pitch, plane);
    }
    __syncthreads();
    // y_u = r_u - alpha B_u^T dp on the r tile (u planes, active DoFs)
    if (const int t = threadIdx.x; t < T::RW * T::RH) {
        const int ly = t / T::RW, lx = t - ly * T::RW;
        const int c = i0 - 1 + lx, d = j0 - 1 + ly;
        const double* p00 = ps + (ly + 1) * T::DW + (lx + 1);   // cell (c, d)
        double bt[5] = {0, 0, 0, 0, 0};
#define MG_I(k, cdx, cdy, sh, q) bt[k] = fma(L.bu[sh][q], p00[(sh) * (T::DW * T::DH) + (cdy) * T::DW + (cdx)], bt[k]);
        MG_INCIDENT_0(MG_I) MG_INCIDENT_1(MG_I) MG_INCIDENT_2(MG_I) MG_INCIDENT_3(MG_I) MG_INCIDENT_4(MG_I)
#undef MG_I
#pragma unroll
        for (int k = 0; k < 5; ++k)
            if (is_active(k, c, d, n)) rs[k * T::RW * T::RH + t] -= L.alpha * bt[k];
    }
    __syncthreads();
    if (const int t = threadIdx.x; t < T::PW * T::PH) {
        const int py = t / T::PW, px = t - py * T::PW;
        const int a = i0 + px, bb = j0 + py;
        if (a <= n && bb <= n) {
            double rr[8];
            gather8<T::RW, T::RH>(rs + (py + 1) * T::RW + (px + 1), rr);
            patch_apply8(U, vertex_class(a, bb, n), rr, zs + t, T::PW * T::PH);
        } else {
#pragma unroll
            for (int s = 0; s < 8; ++s) zs[s * T::PW * T::PH + t] = 0.0;
        }
    }
    __syncthreads();
    const int lx = threadIdx.x % TX, ly = threadIdx.x / TX;
    const int i = i0 + lx, j = j0 + ly;
    if (threadIdx.x >= TX * TY || i > n || j > n) return;
    const double* c00 = zs + ly * T::PW + lx;
#define CC(s, dx, dy) c00[(s) * (T::PW * T::PH) + (dy) * T::PW + (dx)]
    double d[10];
    d[0] = CC(0, 0, 0);
    d[1] = CC(1, 0, 0);
    d[2] = CC(2, 0, 0) + CC(3, 1, 0);
    d[3] = CC(4, 0, 0) + CC(5, 0, 1);
    d[4] = CC(6, 1, 0) + CC(7, 0, 1);
#undef CC
    const double* p00 = ps + (ly + 2) * T::DW + (lx + 2);   // cell (i, j)
    const double* r00 = rs + (ly + 1) * T::RW + (lx + 1);
    double bw[3] = {0, 0, 0};
#define MG_I(k, cdx, cdy, sh, q) bw[(k) - 5] = fma(L.bw[sh][(q) - 9], p00[(sh) * (T::DW * T::DH) + (cdy) * T::DW + (cdx)], bw[(k) - 5]);
    MG_INCIDENT_5(MG_I) MG_INCIDENT_6(MG_I) MG_INCIDENT_7(MG_I)
#undef MG_I
#pragma unroll
    for (int k = 5; k < 8; ++k) {
        const double dwk = PRE ? dwown[k - 5] : Dw_at<HET>(L, k, i, j);
        d[k] = is_active(k, i, j, n) ? (r00[k * T::RW * T::RH] - L.tau * bw[k - 5]) / (L.tau * dwk) : 0.0;
    }
    d[8] = p00[0];
    d[9] = p00[T::DW * T::DH];
    const int64_t o = (int64_t)j * pitch + i;
#pragma unroll
    for (int k = 0; k < 10; ++k) {
        const double xv = XZERO ? 0.0 : (PRE ? xown[k] : __ldg(x + k * plane + o));
        xo[k * plane + o] = is_active(k, i, j, n) ? fma(omega, d[k], xv) : 0.0;
    }
}

// ------------------------------------------------------------------------------------------
// K^{-1} pyramid (reading A11): level 0 from the user's K [shape][j][i] (n x n), then averages
__global__ void kinv_from_K_kernel(int n, int pitch, const double* __restrict__ K, double* __restrict__ kinv) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * 32 + (threadIdx.x & 31), j = blockIdx.y * 8 + (threadIdx.x >> 5);
    if (i >= n || j >= n) return;
    const int64_t plane = (int64_t)(n + 1) * pitch;
    for (int sh = 0; sh < 2; ++sh)
        kinv[sh * plane + (int64_t)j * pitch + i] = 1.0 / K[((int64_t)sh * n + j) * n + i];
}

__global__ void kinv_coarsen_kernel(int nf, int pitchf, const double* __restrict__ kf, int pitchc,
                                    double* __restrict__ kc) {
    pdl_wait();
    pdl_trigger();
    const int I = blockIdx.x * 32 + (threadIdx.x & 31), J = blockIdx.y * 8 + (threadIdx.x >> 5);
    const int nc = nf / 2;
    if (I >= nc || J >= nc) return;
    const int64_t pf = (int64_t)(nf + 1) * pitchf, pc = (int64_t)(nc + 1) * pitchc;
#define KF(sh, di, dj) kf[(sh) * pf + (int64_t)(2 * J + (dj)) * pitchf + 2 * I + (di)]
    // children in the oracle's accumulation order (shape-major, then j, then i)
    const double ll = ((KF(0, 0, 0) + KF(0, 1, 0)) + KF(0, 0, 1)) + KF(1, 0, 0);
    const double ur = ((KF(0, 1, 1) + KF(1, 1, 0)) + KF(1, 0, 1)) + KF(1, 1, 1);
#undef KF
    kc[(int64_t)J * pitchc + I] = ll / 4.0;
    kc[pc + (int64_t)J * pitchc + I] = ur / 4.0;
}

int g_carveout = cudaSharedmemCarveoutMaxShared;   // MG_CARVEOUT (-1: driver default)

// ------------------------------------------------------------------------------------------
// mbarrier / TMA helpers of the row-marching kernels
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// as mbar_wait, backing off between polls (a waiting warp then leaves the issue slots to others)
#ifndef MG_SLEEP_NS
#define MG_SLEEP_NS 64
#endif
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, unsigned parity) {
    unsigned ok;
    for (;;) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        __nanosleep(MG_SLEEP_NS);
    }
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// 3-D TMA box load (dims: column, row, plane) completing on `bar`
__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
            "r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// Every kernel of the cycle asks for the same L1 / shared-memory split (the maximum shared
// carveout): kernels with different preferred splits force the SM to drain and reconfigure between
// consecutive launches, which the latency-bound coarse levels pay on every kernel boundary.
template <typename F>
void carve(F* f) {
    cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, g_carveout);
}
template <typename F>
void set_smem(F* f, int bytes) {
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    carve(f);
}

}  // namespace

// ------------------------------------------------------------------------------------------
// Row-marching Vanka, row-granular rings (3 CTAs / SM): the level-0 hot kernel.  Same arithmetic as
// vanka_kernel (the 2-D tile sweep);
// x, b and the patch outputs live in modular rings of single rows (x: 10, b/r: 9, patches: 5
// rows), filled by one 3-D TMA box per row (32 columns x 1 row x 10 planes) and prefetched one
// step ahead, which cuts shared memory to 72 KB per CTA.
constexpr int M2T = 28, M2R = 4, M2W = M2T + 4, M2C = M2T + 1, M2NT = 128;
// MG_PATCH_MMA: the interior patch solves of a row run as two small GEMMs on the fp64 tensor cores
// (mma.sync m8n8k4: Y+ = G+ H+ (9 x 9 padded to 16 x 12) and Y- = G- H- (11 x 11 -> 16 x 12) over the
// warp's 32 patch columns), staged through the row's patch-correction ring slot, whose stride is then
// padded to 32 columns.  Replaces the 202 DFMA + ~101 constant loads per patch by 48 DMMA + fragment
// traffic per warp and row ("what was tried" for the measurement).
#ifndef MG_PATCH_MMA
#define MG_PATCH_MMA 0
#endif
constexpr int M2CS = MG_PATCH_MMA ? 32 : M2C;   // patch-correction ring stride (patch columns)
constexpr int M2XR = 10, M2BR = 9, M2CR = 5;
constexpr int M2ROW = 10 * M2W;                                  // doubles per x / b ring row
constexpr int M2SMEM = (M2XR * M2ROW + M2BR * M2ROW + M2CR * 20 * M2CS) * 8 + 64;
static_assert(M2T + 2 <= 32 && M2R * 32 == M2NT, "one warp per row, one residual position per thread");
static_assert(M2T % 2 == 0, "TMA box origins i0 - 2 must be even columns");


constexpr int M2NP = 2;   // producer warps of the fused-prolongation sweep (one per row parity of a group;
                          // measured: one warp for both 1.39 ms, two 1.36 ms at 4096^2)

// PROL: the sweep relaxes x + P e_H instead of x (the coarse-grid correction of the V-cycle fused
// into the first post-smoothing sweep): every x row is corrected in the ring right
// after its TMA box lands, with the same arithmetic as prolong_kernel (v = sum of w e_H in table
// order, x + v), so the result is bitwise that of prolong_kernel followed by the sweep, and x + P e_H
// never goes through HBM.
// PV (prolongation variant): 0 plain sweep; 1 fused prolongation by M2NP = 2 producer warps (each
// thread all 10 planes of one column pair of two rows); 2 fused prolongation by 4 producer warps
// (a warp-uniform half of the planes each) with warp-specialised register counts: the producer
// warpgroup drops to M2WS_PREG registers (setmaxnreg.dec) and the compute warpgroup takes them
// (setmaxnreg.inc to M2WS_CREG) -- the 6-warp variant runs every warp at the 96 registers 18 warps
// per SM allow, against 166 in the plain sweep.
#ifndef M2WS_PREG
#define M2WS_PREG 40
#endif
#ifndef M2WS_CREG
#define M2WS_CREG 120
#endif
// PV 3: one producer warp doing both tasks of a group (rows y, y+2 and y+1, y+3) with their coarse
// values double-buffered: 5 warps per CTA, 15 per SM, so the compute warps get 128 registers (4 warps
// per SM sub-partition) instead of the 96 of the 6-warp kernel
__host__ __device__ constexpr int m2np(int pv) { return pv == 2 ? 4 : (pv == 3 ? 1 : (pv == 1 ? M2NP : 0)); }
template <bool XZERO, int PV>
__global__ void __launch_bounds__(M2NT + 32 * m2np(PV), 3) vanka_march2_kernel(const __grid_constant__ CUtensorMap tmx,
                                                               const __grid_constant__ CUtensorMap tmb,
                                                               const VankaParams P, double* __restrict__ xo,
                                                               NormSink S, int MH, const ProlSrc E) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(128) double sm[];
    double* xr = sm;                        // [M2XR][10][M2W]
    double* br = xr + M2XR * M2ROW;         // [M2BR][10][M2W]   b, overwritten by r
    double* cr = br + M2BR * M2ROW;         // [M2CR][20][M2CS]  patch corrections
    uint64_t* bars = reinterpret_cast<uint64_t*>(cr + M2CR * 20 * M2CS);
    const LevelParams& L = P.L;
    constexpr bool PROL = PV != 0;
    constexpr int NPW = m2np(PV);            // producer warps
    if (*L.stop) return;
    // barrier of the four compute warps (the PROL producer warp never joins it)
    auto csync = [&]() {
        if (PROL) asm volatile("bar.sync 1, %0;" ::"n"(M2NT) : "memory");
        else __syncthreads();
    };
    const int n = L.n;
    const int i0 = blockIdx.x * M2T, j0 = blockIdx.y * MH;
    const int rows = min(MH, n + 1 - j0);
    const int nsteps = (rows + M2R - 1) / M2R;
    const int t = threadIdx.x;
    // ring slot of global row y (the offset keeps the argument non-negative down to j0 - 2 M2R)
    auto sx = [&](int y) { return (y - j0 + 2 * M2R) % M2XR; };
    auto sb = [&](int y) { return (y - j0 + 2 * M2R) % M2BR; };
    auto sc = [&](int y) { return (y - j0 + 2 * M2R) % M2CR; };
    // group g brings the rows first used by step g: x rows j0+gR+2 .. j0+gR+R+1 (g = -1: j0-R .. j0+1)
    // and b rows j0+gR+1 .. j0+gR+R
    auto issue = [&](int g) {
        if (g >= nsteps) return;
        uint64_t* bar = &bars[(g + 1) & 1];
        const int nx = XZERO ? 0 : (g < 0 ? M2R + 2 : M2R);
        mbar_expect_tx(bar, (nx + M2R) * M2ROW * 8);
        const int xfirst = g < 0 ? j0 - M2R : j0 + g * M2R + 2;
#pragma unroll 1
        for (int k = 0; k < nx; ++k) tma_load3(xr + sx(xfirst + k) * M2ROW, &tmx, i0 - 2, xfirst + k, 0, bar);
        const int bfirst = j0 + g * M2R + 1;
#pragma unroll 1
        for (int k = 0; k < M2R; ++k) tma_load3(br + sb(bfirst + k) * M2ROW, &tmb, i0 - 2, bfirst + k, 0, bar);
    };
    if (t == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_init(&bars[2], NPW);
        mbar_init(&bars[3], NPW);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // PROL: M2NP producer warps correct the x rows of group g (x += P e_H) as soon as their
    // TMA boxes land -- during step g - 1 of the four compute warps -- and arrive on ready[g]; the
    // compute warps wait on ready[] instead of the TMA barrier, so the prolongation runs on issue
    // slots the latency-bound sweep leaves idle.  Lanes 0-15 take the column pairs (2I, 2I+1) of row
    // y, lanes 16-31 those of row y + 2 (same parity: the table branch is warp uniform).
    // producer task k of a group part (y0, count): lanes 0-15 row y0 + k, lanes 16-31 row y0 + k + 2,
    // column pair (2I, 2I+1); pe[k][] holds the 20 coarse values of the task (pslot20)
    auto prol_task = [&](int y0, int count, int k, int& y, int& I, int& J) {
        const int lane = t & 31;
        const int rsel = (PV == 2 ? (k >> 1) : k) + 2 * (lane >> 4);
        y = y0 + rsel;
        I = (i0 >> 1) - 1 + (lane & 15);
        J = y >> 1;
        return rsel < count && I >= 0 && I < E.nc && J >= 0 && J < E.nc;
    };
    // producer warp k (= M2NT / 32 + k) takes task k of every group part
    const int kp = (t >> 5) - M2NT / 32;
    auto prol_load = [&](int y0, int count, double (&pe)[20], int k) {
        {
            int y, I, J;
            if (!prol_task(y0, count, k, y, I, J)) return;
            const double* e0 = E.e + (int64_t)J * E.pitchc + I;
#define PL(dI, dJ, pl) pe[pslot20(dI, dJ, pl)] = __ldg(e0 + (pl) * E.planec + (dJ) * E.pitchc + (dI));
            if (PV != 2 || (k & 1) == 0) {
                PL(0, 0, 0) PL(0, 0, 1) PL(0, 0, 2) PL(0, 0, 3) PL(0, 0, 4) PL(0, 1, 0) PL(0, 1, 1)
                PL(0, 1, 2) PL(1, 0, 0) PL(1, 0, 1) PL(1, 0, 3) PL(1, 1, 0) PL(1, 1, 1)
            }
            if (PV != 2 || (k & 1) == 1) {
                PL(0, 0, 5) PL(0, 0, 6) PL(0, 0, 7) PL(0, 0, 8) PL(0, 0, 9) PL(0, 1, 5) PL(1, 0, 6)
            }
#undef PL
        }
    };
    auto prol_apply = [&](int y0, int count, const double (&pe)[20], int k) {
#ifdef MG_PROL_NOOP
        return;   // diagnostic build: the pipeline without the arithmetic (wrong results)
#endif
        {
            int y, I, J;
            if (!prol_task(y0, count, k, y, I, J)) return;
            double* xrow = xr + sx(y) * M2ROW + 2 * (t & 15);
            const int fi = 2 * I;
            const unsigned m0 = active_mask(fi, y, n), m1 = active_mask(fi + 1, y, n);
#define PQ(dI, dJ, pl, wt) v = fma(wt, pe[pslot20(dI, dJ, pl)], v);
#define PX(dj, kf)                                                                    \
    {                                                                                 \
        double v = 0.0;                                                               \
        MG_PROLONG_0_##dj##_##kf(PQ) const double v0 = v;                             \
        v = 0.0;                                                                      \
        MG_PROLONG_1_##dj##_##kf(PQ) double2* x2 = reinterpret_cast<double2*>(xrow + (kf) * M2W); \
        double2 xv = *x2;                                                             \
        if (m0 & (1u << (kf))) xv.x += v0;                                            \
        if (m1 & (1u << (kf))) xv.y += v;                                             \
        *x2 = xv;                                                                     \
    }
            if (PV == 2) {   // warp-uniform plane half
                if ((k & 1) == 0) {
                    if (y & 1) { PX(1, 0) PX(1, 1) PX(1, 2) PX(1, 3) PX(1, 4) }
                    else { PX(0, 0) PX(0, 1) PX(0, 2) PX(0, 3) PX(0, 4) }
                } else {
                    if (y & 1) { PX(1, 5) PX(1, 6) PX(1, 7) PX(1, 8) PX(1, 9) }
                    else { PX(0, 5) PX(0, 6) PX(0, 7) PX(0, 8) PX(0, 9) }
                }
            } else {
                if (y & 1) { PX(1, 0) PX(1, 1) PX(1, 2) PX(1, 3) PX(1, 4) PX(1, 5) PX(1, 6) PX(1, 7) PX(1, 8) PX(1, 9) }
                else { PX(0, 0) PX(0, 1) PX(0, 2) PX(0, 3) PX(0, 4) PX(0, 5) PX(0, 6) PX(0, 7) PX(0, 8) PX(0, 9) }
            }
#undef PX
#undef PQ
        }
    };
    uint64_t* ready = bars + 2;
    if (PROL && t >= M2NT) {
        // ---- producer warp: the coarse values of a group are loaded before its TMA boxes are
        // awaited, so their latency overlaps the wait
        if (PV == 2) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(M2WS_PREG));
        double pe[20];
        auto publish = [&](int g) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // ring slots are refilled by TMA later
            __syncwarp();
            if ((t & 31) == 0) mbar_arrive(&ready[(g + 1) & 1]);
        };
        mbar_wait_sleep(&bars[0], 0);
        if (PV == 3) {
            double pe1[20];
#pragma unroll 1
            for (int part = 0; part < 2; ++part) {   // group -1: rows j0 - R .. j0 + 1
                const int y0 = part ? j0 : j0 - M2R, cnt = part ? 2 : M2R;
                prol_load(y0, cnt, pe, 0);
                prol_load(y0, cnt, pe1, 1);
                prol_apply(y0, cnt, pe, 0);
                prol_apply(y0, cnt, pe1, 1);
            }
            publish(-1);
#pragma unroll 1
            for (int g = 0; g < nsteps; ++g) {
                const int y0 = j0 + g * M2R + 2;
                prol_load(y0, M2R, pe, 0);
                prol_load(y0, M2R, pe1, 1);
                mbar_wait_sleep(&bars[(g + 1) & 1], ((g + 1) >> 1) & 1);
                prol_apply(y0, M2R, pe, 0);
                prol_apply(y0, M2R, pe1, 1);
                publish(g);
            }
        } else {
#pragma unroll 1
            for (int part = 0; part < 2; ++part) {   // group -1: rows j0 - R .. j0 + 1
                prol_load(part ? j0 : j0 - M2R, part ? 2 : M2R, pe, kp);
                prol_apply(part ? j0 : j0 - M2R, part ? 2 : M2R, pe, kp);
            }
            publish(-1);
#pragma unroll 1
            for (int g = 0; g < nsteps; ++g) {
                prol_load(j0 + g * M2R + 2, M2R, pe, kp);
                mbar_wait_sleep(&bars[(g + 1) & 1], ((g + 1) >> 1) & 1);
                prol_apply(j0 + g * M2R + 2, M2R, pe, kp);
                publish(g);
            }
        }
        if (S.out || S.state) norm_finish<M2NT + 32 * NPW>(S, 0.0);
        return;
    }
    if (PV == 2) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(M2WS_CREG));
#if MG_PATCH_MMA
    // A fragments of the interior +/- blocks (m8n8k4 row-major A: lane holds row l/4, column l%4 of
    // each 8 x 4 tile), zero padded; G+[r][c] = gpT[c][r]
    double mmaA_p[2][3], mmaA_m[2][3];
    {
        const int gq = (t & 31) >> 2, tg = t & 3;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int ks = 0; ks < 3; ++ks) {
                const int r = 8 * mt + gq, c = 4 * ks + tg;
                mmaA_p[mt][ks] = (r < 9 && c < 9) ? P.gpT[c][r] : 0.0;
                mmaA_m[mt][ks] = (r < 11 && c < 11) ? P.gmT[c][r] : 0.0;
            }
    }
#endif
    if (t == 0) {
        issue(-1);
        issue(0);
    }
    double nrm = 0.0;
    for (int s = -1; s < nsteps; ++s) {
        // ring slots of rows j0 + sR + d (0 <= d <= 5) from per-step bases (no modulo per access)
        const int bx0 = (s * M2R + 2 * M2R) % M2XR, bb0 = (s * M2R + 2 * M2R) % M2BR, bc0 = (s * M2R + 2 * M2R) % M2CR;
        auto sxs = [&](int d) { const int v = bx0 + d; return v >= M2XR ? v - M2XR : v; };
        auto sbs = [&](int d) { const int v = bb0 + d; return v >= M2BR ? v - M2BR : v; };
        auto scs = [&](int d) { const int v = bc0 + d; return v >= M2CR ? v - M2CR : v; };
        // TMA group s landed (and, PROL, its x rows were corrected by the producer warps)
        mbar_wait(PROL ? &ready[(s + 1) & 1] : &bars[(s + 1) & 1], ((s + 1) >> 1) & 1);
        // ---- residual rows y = j0 + s R + 1 + q
        // one warp per row (lanes beyond the row idle): no bank conflicts from rows wrapping in a warp
        if ((t & 31) < M2T + 2) {
            const int q = t >> 5, lx = t & 31;
            const int y = j0 + s * M2R + 1 + q, i = i0 - 1 + lx;
            double* bp = br + sbs(1 + q) * M2ROW + (lx + 1);
            const bool own = lx >= 1 && lx <= M2T && i <= n && y >= j0 && y < j0 + rows;
            double rv[10];
            if (!XZERO) {
                const double* xm = xr + sxs(q) * M2ROW + (lx + 1);
                const double* x0 = xr + sxs(1 + q) * M2ROW + (lx + 1);
                const double* xp = xr + sxs(2 + q) * M2ROW + (lx + 1);
                double av[10];
                apply_rows<M2W, false>(L, xm, x0, xp, i, y, av);
#pragma unroll
                for (int k = 0; k < 10; ++k) rv[k] = is_active(k, i, y, n) ? bp[k * M2W] - av[k] : 0.0;
#pragma unroll
                for (int k = 0; k < 10; ++k) bp[k * M2W] = rv[k];
            } else {
#pragma unroll
                for (int k = 0; k < 10; ++k) rv[k] = bp[k * M2W];
            }
            if (own) {
#pragma unroll
                for (int k = 0; k < 10; ++k) nrm = fma(rv[k], rv[k], nrm);
            }
        }
        csync();
        // every warp is past the owner phase of step s - 1 (the last reader of the x and r ring rows
        // that group s + 1 replaces): refill them.  The owner phase of a step and the residual phase
        // of the next need no barrier between them (disjoint ring rows), so this is the only one.
        // (PROL keeps the end-of-step refill: its producer warps need the longer lead time)
        if (!PROL && t == 0 && s >= 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(s + 1);
        }
        // ---- patch solves at vertex rows bb = j0 + s R + 1 + q (r rows bb - 1 and bb)
#if MG_PATCH_MMA
        {
            const int q = t >> 5, px = t & 31;
            const int a = i0 + px, bb = j0 + s * M2R + 1 + q;
            double* col = cr + scs(1 + q) * (20 * M2CS);       // [20][32]: H, then Y, then the output
            const bool valid = px < M2C && a <= n && bb >= 0 && bb <= n;
            const int cls = valid ? vertex_class(a, bb, n) : 0;
            double rr[20];
            if (valid) {
                const double* r0 = br + sbs(1 + q) * M2ROW + (px + 2);
                const double* rm = br + sbs(q) * M2ROW + (px + 2);
#define RR(dx, dy, pl) ((dy) < 0 ? rm : r0)[(pl) * M2W + (dx)]
                rr[0] = RR(0, 0, 0);   rr[1] = RR(0, 0, 1);
                rr[2] = RR(0, 0, 2);   rr[3] = RR(-1, 0, 2);  rr[4] = RR(0, 0, 3);   rr[5] = RR(0, -1, 3);
                rr[6] = RR(-1, 0, 4);  rr[7] = RR(0, -1, 4);
                rr[8] = RR(0, 0, 5);   rr[9] = RR(-1, 0, 5);  rr[10] = RR(0, 0, 6);  rr[11] = RR(0, -1, 6);
                rr[12] = RR(-1, 0, 7); rr[13] = RR(0, -1, 7);
                rr[14] = RR(0, 0, 8);  rr[15] = RR(-1, -1, 9); rr[16] = RR(-1, 0, 8); rr[17] = RR(0, -1, 9);
                rr[18] = RR(-1, 0, 9); rr[19] = RR(0, -1, 8);
#undef RR
            } else {
#pragma unroll
                for (int k = 0; k < 20; ++k) rr[k] = 0.0;
            }
            // +/- inputs of the interior class (0 for boundary classes: their lanes take the dense path)
            {
                const bool mm = valid && cls == 0;
#pragma unroll
                for (int k = 0; k < 6; ++k) {
                    col[k * M2CS + px] = mm ? rr[2 + 2 * k] - rr[3 + 2 * k] : 0.0;            // hp[k]
                    col[(11 + k) * M2CS + px] = mm ? rr[2 + 2 * k] + rr[3 + 2 * k] : 0.0;     // hm[2 + k]
                }
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    col[(6 + k) * M2CS + px] = mm ? rr[14 + 2 * k] + rr[15 + 2 * k] : 0.0;    // hp[6 + k]
                    col[(17 + k) * M2CS + px] = mm ? rr[14 + 2 * k] - rr[15 + 2 * k] : 0.0;   // hm[8 + k]
                }
                col[9 * M2CS + px] = mm ? rr[0] : 0.0;                                        // hm[0]
                col[10 * M2CS + px] = mm ? rr[1] : 0.0;                                       // hm[1]
            }
            __syncwarp();
            const int gq = px >> 2, tg = px & 3;
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                double bp[3], bm[3];
#pragma unroll
                for (int ks = 0; ks < 3; ++ks) {
                    const int kp = 4 * ks + tg;
                    bp[ks] = kp < 9 ? col[kp * M2CS + 8 * nt + gq] : 0.0;
                    bm[ks] = kp < 11 ? col[(9 + kp) * M2CS + 8 * nt + gq] : 0.0;
                }
                double dp[2][2], dm[2][2];
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) {
                    dp[mt][0] = dp[mt][1] = dm[mt][0] = dm[mt][1] = 0.0;
#pragma unroll
                    for (int ks = 0; ks < 3; ++ks) {
                        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                                     : "+d"(dp[mt][0]), "+d"(dp[mt][1]) : "d"(mmaA_p[mt][ks]), "d"(bp[ks]));
                        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                                     : "+d"(dm[mt][0]), "+d"(dm[mt][1]) : "d"(mmaA_m[mt][ks]), "d"(bm[ks]));
                    }
                }
                __syncwarp();   // every lane has read its B fragments of these columns
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) {
                    const int r = 8 * mt + gq, c = 8 * nt + 2 * tg;
                    if (r < 9) {
                        col[r * M2CS + c] = dp[mt][0];
                        col[r * M2CS + c + 1] = dp[mt][1];
                    }
                    if (r < 11) {
                        col[(9 + r) * M2CS + c] = dm[mt][0];
                        col[(9 + r) * M2CS + c + 1] = dm[mt][1];
                    }
                }
            }
            __syncwarp();
            if (valid) {
                if (cls == 0) {   // back to the spoke basis, in place in the lane's own column
                    double yp[9], ym[11];
#pragma unroll
                    for (int k = 0; k < 9; ++k) yp[k] = col[k * M2CS + px];
#pragma unroll
                    for (int k = 0; k < 11; ++k) ym[k] = col[(9 + k) * M2CS + px];
                    double* out = col + px;
                    out[0] = ym[0];
                    out[M2CS] = ym[1];
#pragma unroll
                    for (int k = 0; k < 6; ++k) {
                        out[(2 + 2 * k) * M2CS] = ym[2 + k] + yp[k];
                        out[(3 + 2 * k) * M2CS] = ym[2 + k] - yp[k];
                    }
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        out[(14 + 2 * k) * M2CS] = yp[6 + k] + ym[8 + k];
                        out[(15 + 2 * k) * M2CS] = yp[6 + k] - ym[8 + k];
                    }
                } else {
                    patch_apply20(P, cls, rr, col + px, M2CS);
                }
            }
        }
#else
        if ((t & 31) < M2C) {
            const int q = t >> 5, px = t & 31;
            const int a = i0 + px, bb = j0 + s * M2R + 1 + q;
            double* out = cr + scs(1 + q) * (20 * M2CS) + px;
            if (a <= n && bb >= 0 && bb <= n) {
                const double* r0 = br + sbs(1 + q) * M2ROW + (px + 2);
                const double* rm = br + sbs(q) * M2ROW + (px + 2);
                double rr[20];
#define RR(dx, dy, pl) ((dy) < 0 ? rm : r0)[(pl) * M2W + (dx)]
                rr[0] = RR(0, 0, 0);   rr[1] = RR(0, 0, 1);
                rr[2] = RR(0, 0, 2);   rr[3] = RR(-1, 0, 2);  rr[4] = RR(0, 0, 3);   rr[5] = RR(0, -1, 3);
                rr[6] = RR(-1, 0, 4);  rr[7] = RR(0, -1, 4);
                rr[8] = RR(0, 0, 5);   rr[9] = RR(-1, 0, 5);  rr[10] = RR(0, 0, 6);  rr[11] = RR(0, -1, 6);
                rr[12] = RR(-1, 0, 7); rr[13] = RR(0, -1, 7);
                rr[14] = RR(0, 0, 8);  rr[15] = RR(-1, -1, 9); rr[16] = RR(-1, 0, 8); rr[17] = RR(0, -1, 9);
                rr[18] = RR(-1, 0, 9); rr[19] = RR(0, -1, 8);
#undef RR
                patch_apply20(P, vertex_class(a, bb, n), rr, out, M2CS);
            } else {
#pragma unroll
                for (int k = 0; k < 20; ++k) out[k * M2CS] = 0.0;
            }
        }
#endif
        csync();
        // ---- owners y = j0 + s R + q: patch rows y and y + 1
        if (s >= 0 && (t & 31) < M2T) {
            const int q = t >> 5, lx = t & 31;
            const int y = j0 + s * M2R + q, i = i0 + lx;
            if (i <= n && y < j0 + rows) {
                const double* c0 = cr + scs(q) * (20 * M2CS) + lx;
                const double* c1 = cr + scs(q + 1) * (20 * M2CS) + lx;
#define CC(sl, dx, dy) ((dy) > 0 ? c1 : c0)[(sl) * M2CS + (dx)]
                double d[10];
                d[0] = CC(0, 0, 0);
                d[1] = CC(1, 0, 0);
                d[2] = CC(2, 0, 0) + CC(3, 1, 0);
                d[3] = CC(4, 0, 0) + CC(5, 0, 1);
                d[4] = CC(6, 1, 0) + CC(7, 0, 1);
                d[5] = CC(8, 0, 0) + CC(9, 1, 0);
                d[6] = CC(10, 0, 0) + CC(11, 0, 1);
                d[7] = CC(12, 1, 0) + CC(13, 0, 1);
                d[8] = CC(14, 0, 0) + CC(16, 1, 0) + CC(19, 0, 1);
                d[9] = CC(15, 1, 1) + CC(17, 0, 1) + CC(18, 1, 0);
#undef CC
                const double* xv = xr + sxs(q) * M2ROW + (lx + 2);
                const int64_t o = (int64_t)y * L.pitch + i;
#pragma unroll
                for (int k = 0; k < 10; ++k) {
                    const double xk = XZERO ? 0.0 : xv[k * M2W];
                    xo[k * L.plane + o] = is_active(k, i, y, n) ? fma(P.omega, d[k], xk) : 0.0;
                }
            }
        }
        if (PROL) {
            csync();
            if (t == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(s + 2);
            }
        }
    }
    if (S.out || S.state) norm_finish<M2NT + 32 * NPW>(S, nrm);
}

// ------------------------------------------------------------------------------------------
// dense boundary-class patch solve out of line (the warp sweep's boundary lanes when no
// vanka_bnd_kernel runs): patch_apply20's boundary branch, same order, through local memory so the
// dense pass's coefficient loads never set the register budget of the interior path
__device__ __noinline__ void patch_bnd20(const double* __restrict__ gb, const double* rr, double* o) {
    const double2* G = reinterpret_cast<const double2*>(gb);
#pragma unroll 1
    for (int a = 0; a < 20; a += 4) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int c2 = 0; c2 < 10; ++c2) {
            const double2 g0 = __ldg(G + (a + 0) * 10 + c2), g1 = __ldg(G + (a + 1) * 10 + c2);
            const double2 g2 = __ldg(G + (a + 2) * 10 + c2), g3 = __ldg(G + (a + 3) * 10 + c2);
            s0 = fma(g0.x, rr[2 * c2], s0); s0 = fma(g0.y, rr[2 * c2 + 1], s0);
            s1 = fma(g1.x, rr[2 * c2], s1); s1 = fma(g1.y, rr[2 * c2 + 1], s1);
            s2 = fma(g2.x, rr[2 * c2], s2); s2 = fma(g2.y, rr[2 * c2 + 1], s2);
            s3 = fma(g3.x, rr[2 * c2], s3); s3 = fma(g3.y, rr[2 * c2 + 1], s3);
        }
        o[a + 0] = s0;
        o[a + 1] = s1;
        o[a + 2] = s2;
        o[a + 3] = s3;
    }
}

// patch_apply20 with the 20 outputs in registers (the warp-marching sweep moves them between lanes
// by shuffles instead of a shared-memory ring).  Same arithmetic and summation order as
// patch_apply20 (interior: +/- blocks; boundary class: dense table, four output rows per pass).
__device__ __forceinline__ void patch_apply20r(const VankaParams& P, int cls, const double rr[20], double o[20]) {
    if (cls == 0) {
        double hp[9], hm[11];
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            hp[q] = rr[2 + 2 * q] - rr[3 + 2 * q];
            hm[2 + q] = rr[2 + 2 * q] + rr[3 + 2 * q];
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            hp[6 + q] = rr[14 + 2 * q] + rr[15 + 2 * q];
            hm[8 + q] = rr[14 + 2 * q] - rr[15 + 2 * q];
        }
        hm[0] = rr[0];
        hm[1] = rr[1];
        double yp[9], ym[11];
#pragma unroll
        for (int a = 0; a < 9; ++a) yp[a] = 0.0;
#pragma unroll
        for (int a = 0; a < 11; ++a) ym[a] = 0.0;
#pragma unroll
        for (int c = 0; c < 11; ++c) {
#pragma unroll
            for (int a = 0; a < 11; ++a) ym[a] = fma(P.gmT[c][a], hm[c], ym[a]);
            if (c < 9) {
#pragma unroll
                for (int a = 0; a < 9; ++a) yp[a] = fma(P.gpT[c][a], hp[c], yp[a]);
            }
        }
        o[0] = ym[0];
        o[1] = ym[1];
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            o[2 + 2 * q] = ym[2 + q] + yp[q];
            o[3 + 2 * q] = ym[2 + q] - yp[q];
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            o[14 + 2 * q] = yp[6 + q] + ym[8 + q];
            o[15 + 2 * q] = yp[6 + q] - ym[8 + q];
        }
    } else {
        // boundary classes: vanka_bnd_kernel (the warp sweep never calls this with cls != 0)
#pragma unroll
        for (int k = 0; k < 20; ++k) o[k] = 0.0;
    }
}

// ------------------------------------------------------------------------------------------
// Boundary-vertex patch solves of the warp-marching sweep: one thread per boundary vertex (a or b in
// {0, n}; index bnd_index), the four residual positions of its patch from a per-thread 4 x 4 x 10
// x tile, the dense boundary-class inverse (patch_apply20, same order), the 20 outputs to
// P.bcorr[k * 4n + index].  The warp kernel reads them instead of running the dense path, so its
// interior path keeps its register budget.
__host__ __device__ __forceinline__ int bnd_count(int n) { return 4 * n; }
__device__ __forceinline__ int bnd_index(int a, int b, int n) {
    return b == 0 ? a : (b == n ? (n + 1) + a : (a == 0 ? 2 * (n + 1) + (b - 1) : 2 * (n + 1) + (n - 1) + (b - 1)));
}
constexpr int WB_NT = 64, WB_SMEM = WB_NT * 160 * 8;
// x(i, j) += P e_H (i, j) for one fine index, all ten planes (prolong_kernel's table chains, same order)
__device__ __forceinline__ void prol_point(const ProlSrc& E, int i, int j, int n, double xk[10]) {
    const int I = i >> 1, J = j >> 1;
    if (i < 0 || j < 0 || I >= E.nc || J >= E.nc) return;
    const double* e0 = E.e + (int64_t)J * E.pitchc + I;
    const unsigned m = active_mask(i, j, n);
#define EQ(dI, dJ, pl, wt) v = fma(wt, __ldg(e0 + (pl) * E.planec + (dJ) * E.pitchc + (dI)), v);
#define P1(di, dj, kf)                                   \
    {                                                    \
        double v = 0.0;                                  \
        MG_PROLONG_##di##_##dj##_##kf(EQ)                \
        if (m & (1u << (kf))) xk[kf] += v;               \
    }
#define P10(di, dj) P1(di, dj, 0) P1(di, dj, 1) P1(di, dj, 2) P1(di, dj, 3) P1(di, dj, 4) \
                    P1(di, dj, 5) P1(di, dj, 6) P1(di, dj, 7) P1(di, dj, 8) P1(di, dj, 9)
    switch ((i & 1) + 2 * (j & 1)) {
        case 0: P10(0, 0) break;
        case 1: P10(1, 0) break;
        case 2: P10(0, 1) break;
        default: P10(1, 1) break;
    }
#undef P10
#undef P1
#undef EQ
}

template <bool XZERO, bool PROL, bool HET = false>
__global__ void __launch_bounds__(WB_NT) vanka_bnd_kernel(const VankaParams P, const double* __restrict__ x,
                                                          const double* __restrict__ b, const ProlSrc E) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(16) double smb[];
    const LevelParams& L = P.L;
    if (*L.stop) return;
    const int n = L.n, nb = bnd_count(n);
    const int t = blockIdx.x * WB_NT + threadIdx.x;
    if (t >= nb) return;
    int a, bb;
    if (t <= n) { a = t; bb = 0; }
    else if (t <= 2 * n + 1) { a = t - (n + 1); bb = n; }
    else if (t < 2 * (n + 1) + (n - 1)) { a = 0; bb = t - 2 * (n + 1) + 1; }
    else { a = n; bb = t - 2 * (n + 1) - (n - 1) + 1; }
    // residuals at (a - 1 + px, bb - 1 + py), px, py in {0, 1}
    double r[2][2][10];
    if (XZERO) {
#pragma unroll
        for (int py = 0; py < 2; ++py)
#pragma unroll
            for (int px = 0; px < 2; ++px) {
                const int i = a - 1 + px, j = bb - 1 + py;
                const bool in = i >= 0 && j >= 0 && i <= n && j <= n;
#pragma unroll
                for (int k = 0; k < 10; ++k) r[py][px][k] = in ? __ldg(b + k * L.plane + (int64_t)j * L.pitch + i) : 0.0;
            }
    } else {
        double* tile = smb + threadIdx.x * 160;   // [10][4][4]: x at columns a-2 .. a+1, rows bb-2 .. bb+1
#pragma unroll
        for (int ry = 0; ry < 4; ++ry)
#pragma unroll
            for (int rx = 0; rx < 4; ++rx) {
                const int i = a - 2 + rx, j = bb - 2 + ry;
                const bool in = i >= 0 && j >= 0 && i <= n && j <= n;
                double xk[10];
#pragma unroll
                for (int k = 0; k < 10; ++k) xk[k] = in ? __ldg(x + k * L.plane + (int64_t)j * L.pitch + i) : 0.0;
                if (PROL && in) prol_point(E, i, j, n, xk);
#pragma unroll
                for (int k = 0; k < 10; ++k) tile[k * 16 + ry * 4 + rx] = xk[k];
            }
#pragma unroll
        for (int py = 0; py < 2; ++py)
#pragma unroll
            for (int px = 0; px < 2; ++px) {
                const int i = a - 1 + px, j = bb - 1 + py;
                const double* x0 = tile + (py + 1) * 4 + (px + 1);
                double av[10];
                apply_rows<16, HET>(L, x0 - 4, x0, x0 + 4, i, j, av);
                const unsigned m = active_mask(i, j, n);
                const int64_t o = (i >= 0 && j >= 0 && i <= n && j <= n) ? (int64_t)j * L.pitch + i : 0;
#pragma unroll
                for (int k = 0; k < 10; ++k) r[py][px][k] = ((m >> k) & 1u) ? __ldg(b + k * L.plane + o) - av[k] : 0.0;
            }
    }
    double rr[20];
#define RR(dx, dy, pl) r[1 + (dy)][1 + (dx)][pl]
    rr[0] = RR(0, 0, 0);   rr[1] = RR(0, 0, 1);
    rr[2] = RR(0, 0, 2);   rr[3] = RR(-1, 0, 2);  rr[4] = RR(0, 0, 3);   rr[5] = RR(0, -1, 3);
    rr[6] = RR(-1, 0, 4);  rr[7] = RR(0, -1, 4);
    rr[8] = RR(0, 0, 5);   rr[9] = RR(-1, 0, 5);  rr[10] = RR(0, 0, 6);  rr[11] = RR(0, -1, 6);
    rr[12] = RR(-1, 0, 7); rr[13] = RR(0, -1, 7);
    rr[14] = RR(0, 0, 8);  rr[15] = RR(-1, -1, 9); rr[16] = RR(-1, 0, 8); rr[17] = RR(0, -1, 9);
    rr[18] = RR(-1, 0, 9); rr[19] = RR(0, -1, 8);
#undef RR
    if (HET) patch_apply_het_t<false>(P, P.hv.cls + vertex_class(a, bb, n) * MG_HV_CLS, a, bb, rr, P.bcorr + t, nb);
    else patch_apply20(P, vertex_class(a, bb, n), rr, P.bcorr + t, nb);
}

// Cooperative version (the default): a CTA takes a run of 32 boundary vertices of one side, stages
// the x tile (with P e_H added, PROL) in shared memory once, computes each residual position once
// and splits the dense patch solves over 4 threads per vertex (5 outputs each, same order).
constexpr int WB2_T = 32, WB2_NT = 128, WB2_XS = 10 * 4 * 35, WB2_RS = 10 * 2 * 33;
template <bool XZERO, bool PROL, bool HET = false>
__global__ void __launch_bounds__(WB2_NT) vanka_bnd2_kernel(const VankaParams P, const double* __restrict__ x,
                                                            const double* __restrict__ b, const ProlSrc E) {
    pdl_wait();
    pdl_trigger();
    __shared__ double xt[WB2_XS];   // [10][PH + 2][PW + 2], plane stride 140
    __shared__ double rt[WB2_RS];   // [10][PH][PW], plane stride 66
    __shared__ __align__(16) double gt[3 * 400];   // the dense inverses of this side's (at most 3) vertex classes
    const LevelParams& L = P.L;
    // every global read of the kernel is issued before the stop flag is tested (one L2 round trip)
    const int stopv = *L.stop;
    const int n = L.n, nb = bnd_count(n), side = blockIdx.y, t = threadIdx.x;
    const bool horiz = side < 2;
    const int v0 = blockIdx.x * WB2_T;
    // vertex run: horizontal sides a = v0 .. v0 + 31 at b = 0 / n; vertical b = v0 .. v0 + 31 at a = 0 / n
    const int fixed = (side & 1) ? n : 0;
    const int PW = horiz ? WB2_T + 1 : 2, PH = horiz ? 2 : WB2_T + 1;
    const int pi0 = horiz ? v0 - 1 : fixed - 1, pj0 = horiz ? fixed - 1 : v0 - 1;   // residual origin
    const int XW = PW + 2;
    // classes: bottom 3, 4, 5; top 6, 7, 8; left 1; right 2 (vertex_class)
    const int c0 = side == 0 ? 3 : side == 1 ? 6 : side == 2 ? 1 : 2, ncls = horiz ? 3 : 1;
    // HET: the side's condensed class tables (MG_HV_CLS doubles each) instead of the dense inverses
    const double* gsrc = HET ? P.hv.cls + c0 * MG_HV_CLS : P.gbnd + c0 * 400;
    for (int q = t; q < ncls * (HET ? MG_HV_CLS / 2 : 200); q += WB2_NT)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(gt + 2 * q)), "l"(gsrc + 2 * q)
                     : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    double bpre[10];
    {
        const int ly = t / PW, lx = t - ly * PW;
        const int i = pi0 + lx, j = pj0 + ly;
        const bool in = t < PW * PH && i >= 0 && j >= 0 && i <= n && j <= n;
        const int64_t o = in ? (int64_t)j * L.pitch + i : 0;
#pragma unroll
        for (int k = 0; k < 10; ++k) bpre[k] = in ? __ldg(b + k * L.plane + o) : 0.0;
    }
    if (!XZERO) {
        for (int p = t; p < (PW + 2) * (PH + 2); p += WB2_NT) {
            const int ly = p / XW, lx = p - ly * XW;
            const int i = pi0 - 1 + lx, j = pj0 - 1 + ly;
            const bool in = i >= 0 && j >= 0 && i <= n && j <= n;
            double xk[10];
#pragma unroll
            for (int k = 0; k < 10; ++k) xk[k] = in ? __ldg(x + k * L.plane + (int64_t)j * L.pitch + i) : 0.0;
            if (PROL && in) prol_point(E, i, j, n, xk);
#pragma unroll
            for (int k = 0; k < 10; ++k) xt[k * 140 + p] = xk[k];
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    if (stopv) return;
    if (t < PW * PH) {
        const int p = t;
        const int ly = p / PW, lx = p - ly * PW;
        const int i = pi0 + lx, j = pj0 + ly;
        if (XZERO) {
#pragma unroll
            for (int k = 0; k < 10; ++k) rt[k * 66 + p] = bpre[k];
        } else {
            const double* x0 = xt + (ly + 1) * XW + (lx + 1);
            double av[10];
            apply_rows<140, HET>(L, x0 - XW, x0, x0 + XW, i, j, av);
            const unsigned m = active_mask(i, j, n);
#pragma unroll
            for (int k = 0; k < 10; ++k) rt[k * 66 + p] = ((m >> k) & 1u) ? bpre[k] - av[k] : 0.0;
        }
    }
    __syncthreads();
    // patches: vertex q = t / 4 of the run, outputs 5 (t % 4) .. 5 (t % 4) + 4
    // HET: one thread per vertex runs the condensed solve (class table in shared memory, S~^{-1} per vertex)
    const int q = HET ? t : t >> 2, part = t & 3;
    const int a = horiz ? v0 + q : fixed, bb = horiz ? fixed : v0 + q;
    const bool valid = (horiz ? (a <= n) : (bb >= 1 && bb <= n - 1)) && (!HET || t < WB2_T);
    if (!valid || (!horiz && n < 2)) return;
    // residual of (a + dx, bb + dy), dx, dy in {-1, 0}: tile position (a + dx - pi0, bb + dy - pj0)
    const double* r00 = rt + (bb - pj0) * PW + (a - pi0);
#define RR(dx, dy, pl) r00[(pl) * 66 + (dy) * PW + (dx)]
    double rr[20];
    rr[0] = RR(0, 0, 0);   rr[1] = RR(0, 0, 1);
    rr[2] = RR(0, 0, 2);   rr[3] = RR(-1, 0, 2);  rr[4] = RR(0, 0, 3);   rr[5] = RR(0, -1, 3);
    rr[6] = RR(-1, 0, 4);  rr[7] = RR(0, -1, 4);
    rr[8] = RR(0, 0, 5);   rr[9] = RR(-1, 0, 5);  rr[10] = RR(0, 0, 6);  rr[11] = RR(0, -1, 6);
    rr[12] = RR(-1, 0, 7); rr[13] = RR(0, -1, 7);
    rr[14] = RR(0, 0, 8);  rr[15] = RR(-1, -1, 9); rr[16] = RR(-1, 0, 8); rr[17] = RR(0, -1, 9);
    rr[18] = RR(-1, 0, 9); rr[19] = RR(0, -1, 8);
#undef RR
    double* out = P.bcorr + bnd_index(a, bb, n);
    if (HET) {
        patch_apply_het_t<true>(P, gt + (vertex_class(a, bb, n) - c0) * MG_HV_CLS, a, bb, rr, out, nb);
        return;
    }
    const double* G = gt + (vertex_class(a, bb, n) - c0) * 400;
#pragma unroll
    for (int u = 0; u < 5; ++u) {
        const int k = part * 5 + u;
        const double2* g = reinterpret_cast<const double2*>(G + k * 20);
        double sacc = 0.0;
#pragma unroll
        for (int c2 = 0; c2 < 10; ++c2) {
            const double2 gg = g[c2];
            sacc = fma(gg.x, rr[2 * c2], sacc);
            sacc = fma(gg.y, rr[2 * c2 + 1], sacc);
        }
        out[k * nb] = sacc;
    }
}

// ------------------------------------------------------------------------------------------
// Warp-marching Vanka sweep (the level-0 hot kernel when MG_WARP_MIN_N <= n).  Same arithmetic as
// vanka_march2_kernel / vanka_kernel (residual, 20-DoF patch solves, owner-computes update,
// PAPER.md:575-588), organised so that no CTA-wide barrier is needed: every WARP marches down its
// own strip of WT = 30 owned columns, one grid row per iteration --
//   residual row y  (lane l: index i = i0 - 1 + l, all 32 lanes useful),
//   patch row y     (lane l: vertex a = i0 - 1 + l; the residuals of the left neighbour arrive by
//                    __shfl_up, those of row y - 1 are carried in registers from the previous iteration),
//   owner row y - 1 (lane l: index i0 - 1 + l, 30 lanes own; the corrections of the right neighbour
//                    arrive by __shfl_down, those of patch row y - 1 are carried as partial sums in
//                    the owner's summation order).
// Only x (a 4-row ring of 34-column, 10-plane TMA boxes) and b (2-row ring of 32-column boxes) pass
// through shared memory, each row prefetched one iteration ahead on per-slot mbarriers: 16 KB per
// warp, 14 warps per SM, and the r / patch-correction rings of the CTA kernel (and both of its
// barriers per step) are gone.
constexpr int WT = 30, WXW = WT + 4, WBW = WT + 4, WXR = 4, WBR = 1;   // TMA box origins: even columns (16 B)
constexpr int WXROW = 10 * WXW, WBROW = 10 * WBW;
constexpr int WXSLOT = (WXROW + 15) / 16 * 16;   // ring slot strides: 128-byte aligned TMA destinations
constexpr int WBSLOT = (WBROW + 15) / 16 * 16;
// the patch-correction sums are carried in registers instead of a [10][32] shared row (MG_WARP_CDREG=1):
// 14 KB per warp, 16 warps per SM for the plain sweep (126 registers), 12 with the fused prolongation
#ifndef MG_WARP_CDREG
#define MG_WARP_CDREG 1
#endif
constexpr int W_WARP_BYTES = ((WXR * WXSLOT + WBR * WBSLOT + (MG_WARP_CDREG ? 0 : 10 * 32)) * 8 + 64 + 127) / 128 * 128;
// PROL (first post-sweep with the coarse-grid correction x + P e_H fused in): + a 3-row ring of coarse
// rows (20-column boxes from the even column at or below (i0 - 2) / 2, one TMA box per coarse row)
constexpr int WCC = 20, WCROW = 10 * WCC, WCSLOT = (WCROW + 15) / 16 * 16, WCR = 3;
constexpr int W_WARP_BYTES_P =
    ((WXR * WXSLOT + WBR * WBSLOT + (MG_WARP_CDREG ? 0 : 10 * 32) + WCR * WCSLOT) * 8 + 64 + 127) / 128 * 128;
#ifndef MG_WPC
#define MG_WPC (MG_WARP_CDREG ? 8 : 6)   // warps per CTA (2 CTAs per SM)
#endif
#ifndef MG_WPC_P
#define MG_WPC_P (MG_WARP_CDREG ? 6 : 5)
#endif
template <bool PROL> struct WGeom {
    static constexpr int NW = PROL ? MG_WPC_P : MG_WPC, BYTES = PROL ? W_WARP_BYTES_P : W_WARP_BYTES;
    static constexpr int NT = 32 * NW, SMEM = NW * BYTES;
};
constexpr int WPC = MG_WPC, W_NT = 32 * WPC, W_SMEM = WPC * W_WARP_BYTES;
static_assert(2 * (WGeom<false>::SMEM + 1024) <= 228 * 1024 && 2 * (WGeom<true>::SMEM + 1024) <= 228 * 1024,
              "two CTAs per SM");
static_assert((WXW * 8) % 16 == 0 && (WBW * 8) % 16 == 0 && (WXSLOT * 8) % 128 == 0 && (WBSLOT * 8) % 128 == 0,
              "TMA box rows and ring slots 16 / 128-byte aligned");

template <bool XZERO, bool PROL, bool BK>
__global__ void __launch_bounds__(WGeom<PROL>::NT, 2) vanka_warp_kernel(const __grid_constant__ CUtensorMap tmx,
                                                                        const __grid_constant__ CUtensorMap tmb,
                                                                        const __grid_constant__ CUtensorMap tmc,
                                                                        const VankaParams P, double* __restrict__ xo,
                                                                        NormSink S, int MH, int nstrips, int ntasks,
                                                                        const ProlSrc E) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(128) double sm[];
    const LevelParams& L = P.L;
    if (*L.stop) return;
    const int n = L.n;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int task = blockIdx.x * WGeom<PROL>::NW + w;
    double nrm = 0.0;
    if (task < ntasks) {
        double* xr = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + w * WGeom<PROL>::BYTES);   // [WXR][10][WXW] (slot stride WXSLOT)
        double* br = xr + WXR * WXSLOT;                                                              // [WBR][10][WBW]
        constexpr bool CDREG = MG_WARP_CDREG;
        double* cds = br + WBR * WBSLOT;                                                             // [10][32] (!CDREG)
        double* cr = cds + (CDREG ? 0 : 10 * 32);                                                    // PROL: [WCR][10][WCC]
        uint64_t* xbar = reinterpret_cast<uint64_t*>(cr + (PROL ? WCR * WCSLOT : 0));                // [WXR]
        uint64_t* bbar = xbar + WXR;                                                                 // [WBR]
        uint64_t* cbar = bbar + WBR;                                                                 // PROL: [WCR]
        // tasks of the two boundary strips first (their dense boundary patches make them the slowest;
        // started in the first wave they do not trail the grid), then seg-major over the inner strips
        int strip, seg;
        const int nseg = ntasks / nstrips;
        if (nstrips <= 2) {
            strip = task % nstrips;
            seg = task / nstrips;
        } else if (task < 2 * nseg) {
            strip = (task & 1) ? nstrips - 1 : 0;
            seg = task >> 1;
        } else {
            strip = 1 + (task - 2 * nseg) % (nstrips - 2);
            seg = (task - 2 * nseg) / (nstrips - 2);
        }
        const int i0 = strip * WT, j0 = seg * MH;
        const int rows = min(MH, n + 1 - j0);
        const int yend = j0 + rows;   // residual / patch rows j0 - 1 .. yend, owner rows j0 .. yend - 1
        const int i = i0 - 1 + lane;  // residual position, patch vertex and owner index of this lane
        // every residual position / owner of the strip strictly inside the domain (warp uniform)
        const bool inner = i0 - 1 >= 1 && i0 + WT <= n - 1;
        // x row y: load number q = y - (j0 - 2), slot q % WXR; b row y: q = y - (j0 - 1), slot q % WBR
        auto load_x = [&](int y) {
            const int q = y - (j0 - 2);
            uint64_t* bar = &xbar[q % WXR];
            mbar_expect_tx(bar, WXROW * 8);
            tma_load3(xr + (q % WXR) * WXSLOT, &tmx, i0 - 2, y, 0, bar);
        };
        auto load_b = [&](int y) {
            const int q = y - (j0 - 1);
            uint64_t* bar = &bbar[q % WBR];
            mbar_expect_tx(bar, WBROW * 8);
            tma_load3(br + (q % WBR) * WBSLOT, &tmb, i0 - 2, y, 0, bar);
        };
        auto wait_x = [&](int y) { const int q = y - (j0 - 2); mbar_wait(&xbar[q % WXR], (q / WXR) & 1); };
        auto wait_b = [&](int y) { const int q = y - (j0 - 1); mbar_wait(&bbar[q % WBR], (q / WBR) & 1); };
        auto xrow = [&](int y) { return xr + ((y - (j0 - 2)) % WXR) * WXSLOT; };
        // PROL: coarse row J (load number J - Jb, slot % WCR); fine row r needs coarse rows r >> 1, (r >> 1) + 1
        const int I0 = (i0 - 2) >> 1, Iorg = I0 & ~1, Jb = (j0 - 2) >> 1, Jmax = ((yend + 1) >> 1) + 1;
        auto load_c = [&](int J) {
            const int q = J - Jb;
            uint64_t* bar = &cbar[q % WCR];
            mbar_expect_tx(bar, WCROW * 8);
            tma_load3(cr + (q % WCR) * WCSLOT, &tmc, Iorg, J, 0, bar);
        };
        auto wait_c = [&](int J) { const int q = J - Jb; mbar_wait(&cbar[q % WCR], (q / WCR) & 1); };
        auto crow = [&](int J) { return cr + ((J - Jb) % WCR) * WCSLOT; };
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < WXR; ++k) mbar_init(&xbar[k], 1);
#pragma unroll
            for (int k = 0; k < WBR; ++k) mbar_init(&bbar[k], 1);
            if (PROL)
#pragma unroll
                for (int k = 0; k < WCR; ++k) mbar_init(&cbar[k], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        if (lane == 0) {
            if (PROL)
#pragma unroll
                for (int k = 0; k < WCR; ++k)
                    if (Jb + k <= Jmax) load_c(Jb + k);
            if (!XZERO)
#pragma unroll
                for (int k = 0; k < WXR; ++k) load_x(j0 - 2 + k);
#pragma unroll
            for (int k = 0; k < WBR; ++k) load_b(j0 - 1 + k);
        }
        // PROL: x row r += P e_H in the ring (lanes 0-16: the column pair (2I, 2I+1), I = I0 + lane, of
        // fine row r; the prolongation's table arithmetic in table order, bitwise prolong_kernel's)
        auto prol_row = [&](int r) {
            const int J = r >> 1;
            wait_c(J);
            wait_c(J + 1);
            const int I = I0 + lane;
            if (lane <= 16 && I >= 0 && I < E.nc && J >= 0 && J < E.nc) {
                const double* c0 = crow(J) + (I - Iorg);
                const double* c1 = crow(J + 1) + (I - Iorg);
                double pe[20];
#define PL(dI, dJ, pl) pe[pslot20(dI, dJ, pl)] = ((dJ) ? c1 : c0)[(pl) * WCC + (dI)];
                PL(0, 0, 0) PL(0, 0, 1) PL(0, 0, 2) PL(0, 0, 3) PL(0, 0, 4) PL(0, 1, 0) PL(0, 1, 1)
                PL(0, 1, 2) PL(1, 0, 0) PL(1, 0, 1) PL(1, 0, 3) PL(1, 1, 0) PL(1, 1, 1)
                PL(0, 0, 5) PL(0, 0, 6) PL(0, 0, 7) PL(0, 0, 8) PL(0, 0, 9) PL(0, 1, 5) PL(1, 0, 6)
#undef PL
                double* xrw = xrow(r) + 2 * lane;
                const int fi = 2 * I;
                const unsigned m0 = active_mask(fi, r, n), m1 = active_mask(fi + 1, r, n);
#define PQ(dI, dJ, pl, wt) v = fma(wt, pe[pslot20(dI, dJ, pl)], v);
#define PX(dj, kf)                                                                    \
    {                                                                                 \
        double v = 0.0;                                                               \
        MG_PROLONG_0_##dj##_##kf(PQ) const double v0 = v;                             \
        v = 0.0;                                                                      \
        MG_PROLONG_1_##dj##_##kf(PQ) double2* x2 = reinterpret_cast<double2*>(xrw + (kf) * WXW); \
        double2 xv = *x2;                                                             \
        if (m0 & (1u << (kf))) xv.x += v0;                                            \
        if (m1 & (1u << (kf))) xv.y += v;                                             \
        *x2 = xv;                                                                     \
    }
#define PXF(dj, kf)                                                                   \
    {                                                                                 \
        double v = 0.0;                                                               \
        MG_PROLONG_0_##dj##_##kf(PQ) const double v0 = v;                             \
        v = 0.0;                                                                      \
        MG_PROLONG_1_##dj##_##kf(PQ) double2* x2 = reinterpret_cast<double2*>(xrw + (kf) * WXW); \
        double2 xv = *x2;                                                             \
        xv.x += v0;                                                                   \
        xv.y += v;                                                                    \
        *x2 = xv;                                                                     \
    }
                // warp-uniform: every fine index of the row active (inner strip, inner row) -> no masks
                if (I0 >= 1 && r >= 1 && r <= n - 1) {
                    if (r & 1) { PXF(1, 0) PXF(1, 1) PXF(1, 2) PXF(1, 3) PXF(1, 4) PXF(1, 5) PXF(1, 6) PXF(1, 7) PXF(1, 8) PXF(1, 9) }
                    else { PXF(0, 0) PXF(0, 1) PXF(0, 2) PXF(0, 3) PXF(0, 4) PXF(0, 5) PXF(0, 6) PXF(0, 7) PXF(0, 8) PXF(0, 9) }
                } else {
                    if (r & 1) { PX(1, 0) PX(1, 1) PX(1, 2) PX(1, 3) PX(1, 4) PX(1, 5) PX(1, 6) PX(1, 7) PX(1, 8) PX(1, 9) }
                    else { PX(0, 0) PX(0, 1) PX(0, 2) PX(0, 3) PX(0, 4) PX(0, 5) PX(0, 6) PX(0, 7) PX(0, 8) PX(0, 9) }
                }
#undef PXF
#undef PX
#undef PQ
            }
            __syncwarp();
            // after an odd fine row, coarse row J is dead: its slot takes J + WCR
            if ((r & 1) && lane == 0 && J + WCR <= Jmax) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                load_c(J + WCR);
            }
        };
        if (!XZERO) {
            wait_x(j0 - 2);
            wait_x(j0 - 1);
            if (PROL) {
                prol_row(j0 - 2);
                prol_row(j0 - 1);
            }
        }
        // carried from the previous iteration: r of row y - 1 (the planes the patch reads there), the
        // left neighbour's plane-9 residual of row y - 1, the dy = 0 corrections of patch row y - 1
        // (the corrections in shared memory, one column per lane: cds[k][lane], slot 9 = c18)
        double rp3 = 0, rp4 = 0, rp6 = 0, rp7 = 0, rp8 = 0, rp9 = 0, rpl9 = 0;
        double* cdl = cds + lane;
        double cdr[10];
#pragma unroll
        for (int k = 0; k < 10; ++k) cdr[k] = 0.0;
#define CD(k) (*(CDREG ? &cdr[k] : &cdl[32 * (k)]))
#pragma unroll 1
        for (int y = j0 - 1; y <= yend; ++y) {
            // ---- residual row y
            if (!XZERO) wait_x(y + 1);
            if (PROL) prol_row(y + 1);
            wait_b(y);
            double rv[10];
            {
                const double* bp = br + ((y - (j0 - 1)) % WBR) * WBSLOT + (lane + 1);
                if (!XZERO) {
                    const double* x0 = xrow(y) + (lane + 1);
                    double av[10];
                    apply_rows<WXW, false>(L, xrow(y - 1) + (lane + 1), x0, xrow(y + 1) + (lane + 1), i, y, av);
                    if (inner && y >= 1 && y <= n - 1) {   // warp-uniform: every position fully active
#pragma unroll
                        for (int k = 0; k < 10; ++k) rv[k] = bp[k * WBW] - av[k];
                    } else {
                        const unsigned m = active_mask(i, y, n);
#pragma unroll
                        for (int k = 0; k < 10; ++k) rv[k] = ((m >> k) & 1u) ? bp[k * WBW] - av[k] : 0.0;
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 10; ++k) rv[k] = bp[k * WBW];
                }
            }
            __syncwarp();
            // b row y consumed: its slot takes row y + WBR (one iteration ahead)
            if (lane == 0 && y + WBR <= yend) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                load_b(y + WBR);
            }
            if (lane >= 1 && lane <= WT && i <= n && y >= j0 && y < yend) {
#pragma unroll
                for (int k = 0; k < 10; ++k) nrm = fma(rv[k], rv[k], nrm);
            }
            // ---- patch row y (vertex (i, y)); left neighbour's residuals by shuffle
            const double l2 = __shfl_up_sync(0xffffffffu, rv[2], 1), l4 = __shfl_up_sync(0xffffffffu, rv[4], 1);
            const double l5 = __shfl_up_sync(0xffffffffu, rv[5], 1), l7 = __shfl_up_sync(0xffffffffu, rv[7], 1);
            const double l8 = __shfl_up_sync(0xffffffffu, rv[8], 1), l9 = __shfl_up_sync(0xffffffffu, rv[9], 1);
            double o[20];
            if (y >= j0 && lane >= 1 && i <= n && y <= n) {
                double rr[20];
                rr[0] = rv[0]; rr[1] = rv[1];
                rr[2] = rv[2]; rr[3] = l2;   rr[4] = rv[3]; rr[5] = rp3;
                rr[6] = l4;    rr[7] = rp4;
                rr[8] = rv[5]; rr[9] = l5;   rr[10] = rv[6]; rr[11] = rp6;
                rr[12] = l7;   rr[13] = rp7;
                rr[14] = rv[8]; rr[15] = rpl9; rr[16] = l8; rr[17] = rp9;
                rr[18] = l9;   rr[19] = rp8;
                if (i > 0 && i < n && y > 0 && y < n) {
                    patch_apply20r(P, 0, rr, o);
                } else if (BK) {   // boundary vertex: its outputs were computed by vanka_bnd_kernel
                    const int nb = bnd_count(n), bi = bnd_index(i, y, n);
#pragma unroll
                    for (int k = 0; k < 20; ++k) o[k] = __ldg(P.bcorr + k * nb + bi);
                } else {           // boundary vertex: dense class inverse, out of line
                    double rb[20], ob[20];
#pragma unroll
                    for (int k = 0; k < 20; ++k) rb[k] = rr[k];
                    patch_bnd20(P.gbnd + vertex_class(i, y, n) * 400, rb, ob);
#pragma unroll
                    for (int k = 0; k < 20; ++k) o[k] = ob[k];
                }
            } else {
#pragma unroll
                for (int k = 0; k < 20; ++k) o[k] = 0.0;
            }
            rp3 = rv[3]; rp4 = rv[4]; rp6 = rv[6]; rp7 = rv[7]; rp8 = rv[8]; rp9 = rv[9]; rpl9 = l9;
            // ---- owner row y - 1: carried dy = 0 sums + the dy = 1 corrections of patch row y
            const double r15 = __shfl_down_sync(0xffffffffu, o[15], 1);
            if (y >= j0 + 1) {
                const int yo = y - 1;
                if (lane >= 1 && lane <= WT && i <= n) {
                    double d[10];
                    d[0] = CD(0);
                    d[1] = CD(1);
                    d[2] = CD(2);
                    d[3] = CD(3) + o[5];
                    d[4] = CD(4) + o[7];
                    d[5] = CD(5);
                    d[6] = CD(6) + o[11];
                    d[7] = CD(7) + o[13];
                    d[8] = CD(8) + o[19];
                    d[9] = (r15 + o[17]) + CD(9);
                    const double* xv = xrow(yo) + (lane + 1);
                    const int64_t off = (int64_t)yo * L.pitch + i;
                    if (inner && yo >= 1 && yo <= n - 1) {   // warp-uniform: every owner fully active
#pragma unroll
                        for (int k = 0; k < 10; ++k) xo[k * L.plane + off] = fma(P.omega, d[k], XZERO ? 0.0 : xv[k * WXW]);
                    } else {
                        const unsigned m = active_mask(i, yo, n);
#pragma unroll
                        for (int k = 0; k < 10; ++k) {
                            const double xk = XZERO ? 0.0 : xv[k * WXW];
                            xo[k * L.plane + off] = ((m >> k) & 1u) ? fma(P.omega, d[k], xk) : 0.0;
                        }
                    }
                }
            }
            // dy = 0 corrections of patch row y, summed in the owner's order (right neighbour by shuffle)
            {
                const double s3 = __shfl_down_sync(0xffffffffu, o[3], 1), s6 = __shfl_down_sync(0xffffffffu, o[6], 1);
                const double s9 = __shfl_down_sync(0xffffffffu, o[9], 1), s12 = __shfl_down_sync(0xffffffffu, o[12], 1);
                const double s16 = __shfl_down_sync(0xffffffffu, o[16], 1), s18 = __shfl_down_sync(0xffffffffu, o[18], 1);
                CD(0) = o[0];
                CD(1) = o[1];
                CD(2) = o[2] + s3;
                CD(3) = o[4];
                CD(4) = s6;
                CD(5) = o[8] + s9;
                CD(6) = o[10];
                CD(7) = s12;
                CD(8) = o[14] + s16;
                CD(9) = s18;
            }
            // x row y - 1 is dead (last read: residual row y, owner row y - 1): its slot takes row y + 3
            if (!XZERO) {
                __syncwarp();
                if (lane == 0 && y + 3 <= yend + 1) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    load_x(y + 3);
                }
            }
        }
    }
#undef CD
    if (S.out || S.state) norm_finish<WGeom<PROL>::NT>(S, nrm);
}

// ------------------------------------------------------------------------------------------
// Warp-marching heterogeneous-K Vanka sweep (round 2; K-field levels with n >= MG_HET_WARP_N): the
// organisation of vanka_warp_kernel (one warp per 30-column strip, one row per iteration, residuals and
// corrections moved by shuffles, no CTA barrier) with the arithmetic of vanka_het_kernel -- the residual
// reads K^{-1} from a 4-row TMA ring of the two K^{-1} planes (apply_rows_kr), interior patches run the
// condensed +/- solve with the per-vertex S~^{-1} (patch_apply_het_pm, 21 coalesced loads per row), the
// boundary vertices' outputs come from vanka_bnd2_kernel<.., HET> (MG_HW_BK=2: vanka_bnd_kernel<.., HET>).  Same
// summation order in the owner phase:
// bitwise vanka_het_kernel.
constexpr int HW_KR = 4, HW_KROW = 2 * WXW, HW_KSLOT = (HW_KROW + 15) / 16 * 16;
constexpr int HW_BYTES = ((WXR * WXSLOT + WBR * WBSLOT + HW_KR * HW_KSLOT) * 8 + 128 + 127) / 128 * 128;
#ifndef MG_HW_NW
#define MG_HW_NW 6
#endif
#ifndef MG_HW_EARLY
#define MG_HW_EARLY 0   // 1: S~^{-1} of the row's vertices loaded into registers before the residual phase
#endif
constexpr int HW_NW = MG_HW_NW, HW_NT = 32 * HW_NW, HW_SMEM = HW_NW * HW_BYTES;
static_assert(2 * (HW_SMEM + 1024) <= 228 * 1024, "two CTAs per SM");

template <bool XZERO>
__global__ void __launch_bounds__(HW_NT, 2) vanka_hwarp_kernel(const __grid_constant__ CUtensorMap tmx,
                                                               const __grid_constant__ CUtensorMap tmb,
                                                               const __grid_constant__ CUtensorMap tmk,
                                                               const VankaParams P, const __grid_constant__ HvInterior Ti,
                                                               double* __restrict__ xo, NormSink S, int MH, int nstrips,
                                                               int ntasks, int pf) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(128) double sm[];
    const LevelParams& L = P.L;
    if (*L.stop) return;
    const int n = L.n;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int task = blockIdx.x * HW_NW + w;
    double nrm = 0.0;
    if (task < ntasks) {
        double* xr = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + w * HW_BYTES);   // [WXR][10][WXW]
        double* br = xr + WXR * WXSLOT;                                                      // [WBR][10][WBW]
        double* kr = br + WBR * WBSLOT;                                                      // [HW_KR][2][WXW]
        uint64_t* xbar = reinterpret_cast<uint64_t*>(kr + HW_KR * HW_KSLOT);                 // [WXR]
        uint64_t* bbar = xbar + WXR;                                                         // [WBR]
        uint64_t* kbar = bbar + WBR;                                                         // [HW_KR]
        int strip, seg;
        const int nseg = ntasks / nstrips;
        if (nstrips <= 2) {
            strip = task % nstrips;
            seg = task / nstrips;
        } else if (task < 2 * nseg) {
            strip = (task & 1) ? nstrips - 1 : 0;
            seg = task >> 1;
        } else {
            strip = 1 + (task - 2 * nseg) % (nstrips - 2);
            seg = (task - 2 * nseg) / (nstrips - 2);
        }
        const int i0 = strip * WT, j0 = seg * MH;
        const int rows = min(MH, n + 1 - j0);
        const int yend = j0 + rows;
        const int i = i0 - 1 + lane;
        const bool inner = i0 - 1 >= 1 && i0 + WT <= n - 1;
        auto load_x = [&](int y) {
            const int q = y - (j0 - 2);
            uint64_t* bar = &xbar[q % WXR];
            mbar_expect_tx(bar, WXROW * 8);
            tma_load3(xr + (q % WXR) * WXSLOT, &tmx, i0 - 2, y, 0, bar);
        };
        auto load_b = [&](int y) {
            const int q = y - (j0 - 1);
            uint64_t* bar = &bbar[q % WBR];
            mbar_expect_tx(bar, WBROW * 8);
            tma_load3(br + (q % WBR) * WBSLOT, &tmb, i0 - 2, y, 0, bar);
        };
        // K^{-1} cell row y (cells (., y)): load number q = y - (j0 - 2), slot q % HW_KR
        auto load_k = [&](int y) {
            const int q = y - (j0 - 2);
            uint64_t* bar = &kbar[q % HW_KR];
            mbar_expect_tx(bar, HW_KROW * 8);
            tma_load3(kr + (q % HW_KR) * HW_KSLOT, &tmk, i0 - 2, y, 0, bar);
        };
        auto wait_x = [&](int y) { const int q = y - (j0 - 2); mbar_wait(&xbar[q % WXR], (q / WXR) & 1); };
        auto wait_b = [&](int y) { const int q = y - (j0 - 1); mbar_wait(&bbar[q % WBR], (q / WBR) & 1); };
        auto wait_k = [&](int y) { const int q = y - (j0 - 2); mbar_wait(&kbar[q % HW_KR], (q / HW_KR) & 1); };
        auto xrow = [&](int y) { return xr + ((y - (j0 - 2)) % WXR) * WXSLOT; };
        auto krow = [&](int y) { return kr + ((y - (j0 - 2)) % HW_KR) * HW_KSLOT; };
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < WXR; ++k) mbar_init(&xbar[k], 1);
#pragma unroll
            for (int k = 0; k < WBR; ++k) mbar_init(&bbar[k], 1);
#pragma unroll
            for (int k = 0; k < HW_KR; ++k) mbar_init(&kbar[k], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        if (lane == 0) {
            if (!XZERO) {
#pragma unroll
                for (int k = 0; k < WXR; ++k) load_x(j0 - 2 + k);
                // K rows j0 - 2 .. j0 (the end of iteration y loads row y + 2 into the slot of row y - 2)
#pragma unroll
                for (int k = 0; k < HW_KR - 1; ++k)
                    if (j0 - 2 + k <= yend) load_k(j0 - 2 + k);
            }
#pragma unroll
            for (int k = 0; k < WBR; ++k) load_b(j0 - 1 + k);
        }
        if (!XZERO) {
            wait_x(j0 - 2);
            wait_x(j0 - 1);
            wait_k(j0 - 2);
        }
        double rp3 = 0, rp4 = 0, rp6 = 0, rp7 = 0, rp8 = 0, rp9 = 0, rpl9 = 0;
        double cdr[10];
#pragma unroll
        for (int k = 0; k < 10; ++k) cdr[k] = 0.0;
#pragma unroll 1
        for (int y = j0 - 1; y <= yend; ++y) {
            // S~^{-1} of vertex row y + 2 towards the SM (lane k: plane k, the up to 3 lines of the strip's 32 columns)
            if (pf && lane < MG_HV_NSINV && y + 2 >= 1 && y + 2 <= n - 1) {
                const double* pa = P.hv.sinv + lane * L.plane + (int64_t)(y + 2) * L.pitch + max(i0 - 1, 0);
                if (pf == 1) {
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(pa));
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(pa + 16));
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(pa + 31));
                } else {
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(pa));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(pa + 16));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(pa + 31));
                }
            }
#if MG_HW_EARLY
            // the S~^{-1} entries of this lane's vertex (i, y), issued before the residual phase
            double sq[MG_HV_NSINV];
            {
                const bool vin = y >= j0 && lane >= 1 && i > 0 && i < n && y > 0 && y < n;
                const double* si = P.hv.sinv + (vin ? (int64_t)y * L.pitch + i : 0);
#pragma unroll
                for (int q = 0; q < MG_HV_NSINV; ++q) sq[q] = vin ? __ldg(si + q * L.plane) : 0.0;
            }
#endif
            // ---- residual row y
            if (!XZERO) {
                wait_x(y + 1);
                wait_k(y);
            }
            wait_b(y);
            double rv[10];
            {
                const double* bp = br + ((y - (j0 - 1)) % WBR) * WBSLOT + (lane + 1);
                if (!XZERO) {
                    const double* x0 = xrow(y) + (lane + 1);
                    double av[10];
                    apply_rows_kr<WXW, WXW>(L, xrow(y - 1) + (lane + 1), x0, xrow(y + 1) + (lane + 1),
                                            krow(y - 1) + (lane + 1), krow(y) + (lane + 1), av);
                    if (inner && y >= 1 && y <= n - 1) {
#pragma unroll
                        for (int k = 0; k < 10; ++k) rv[k] = bp[k * WBW] - av[k];
                    } else {
                        const unsigned m = active_mask(i, y, n);
#pragma unroll
                        for (int k = 0; k < 10; ++k) rv[k] = ((m >> k) & 1u) ? bp[k * WBW] - av[k] : 0.0;
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 10; ++k) rv[k] = bp[k * WBW];
                }
            }
            __syncwarp();
            if (lane == 0 && y + WBR <= yend) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                load_b(y + WBR);
            }
            if (lane >= 1 && lane <= WT && i <= n && y >= j0 && y < yend) {
#pragma unroll
                for (int k = 0; k < 10; ++k) nrm = fma(rv[k], rv[k], nrm);
            }
            // ---- patch row y (vertex (i, y)); left neighbour's residuals by shuffle
            const double l2 = __shfl_up_sync(0xffffffffu, rv[2], 1), l4 = __shfl_up_sync(0xffffffffu, rv[4], 1);
            const double l5 = __shfl_up_sync(0xffffffffu, rv[5], 1), l7 = __shfl_up_sync(0xffffffffu, rv[7], 1);
            const double l8 = __shfl_up_sync(0xffffffffu, rv[8], 1), l9 = __shfl_up_sync(0xffffffffu, rv[9], 1);
            double o[20];
            if (y >= j0 && lane >= 1 && i <= n && y <= n) {
                double rr[20];
                rr[0] = rv[0]; rr[1] = rv[1];
                rr[2] = rv[2]; rr[3] = l2;   rr[4] = rv[3]; rr[5] = rp3;
                rr[6] = l4;    rr[7] = rp4;
                rr[8] = rv[5]; rr[9] = l5;   rr[10] = rv[6]; rr[11] = rp6;
                rr[12] = l7;   rr[13] = rp7;
                rr[14] = rv[8]; rr[15] = rpl9; rr[16] = l8; rr[17] = rp9;
                rr[18] = l9;   rr[19] = rp8;
                if (i > 0 && i < n && y > 0 && y < n) {
#if MG_HW_EARLY
                    patch_apply_het_pm<true>(P, Ti.pm, i, y, rr, o, 1, sq);
#else
                    patch_apply_het_pm(P, Ti.pm, i, y, rr, o, 1);
#endif
                } else {   // boundary vertex: its outputs were computed by the boundary kernel (launch_vanka_hwarp)
                    const int nb = bnd_count(n), bi = bnd_index(i, y, n);
#pragma unroll
                    for (int k = 0; k < 20; ++k) o[k] = __ldg(P.bcorr + k * nb + bi);
                }
            } else {
#pragma unroll
                for (int k = 0; k < 20; ++k) o[k] = 0.0;
            }
            rp3 = rv[3]; rp4 = rv[4]; rp6 = rv[6]; rp7 = rv[7]; rp8 = rv[8]; rp9 = rv[9]; rpl9 = l9;
            // ---- owner row y - 1
            const double r15 = __shfl_down_sync(0xffffffffu, o[15], 1);
            if (y >= j0 + 1) {
                const int yo = y - 1;
                if (lane >= 1 && lane <= WT && i <= n) {
                    double d[10];
                    d[0] = cdr[0];
                    d[1] = cdr[1];
                    d[2] = cdr[2];
                    d[3] = cdr[3] + o[5];
                    d[4] = cdr[4] + o[7];
                    d[5] = cdr[5];
                    d[6] = cdr[6] + o[11];
                    d[7] = cdr[7] + o[13];
                    d[8] = cdr[8] + o[19];
                    d[9] = (r15 + o[17]) + cdr[9];
                    const double* xv = xrow(yo) + (lane + 1);
                    const int64_t off = (int64_t)yo * L.pitch + i;
                    if (inner && yo >= 1 && yo <= n - 1) {
#pragma unroll
                        for (int k = 0; k < 10; ++k) xo[k * L.plane + off] = fma(P.omega, d[k], XZERO ? 0.0 : xv[k * WXW]);
                    } else {
                        const unsigned m = active_mask(i, yo, n);
#pragma unroll
                        for (int k = 0; k < 10; ++k) {
                            const double xk = XZERO ? 0.0 : xv[k * WXW];
                            xo[k * L.plane + off] = ((m >> k) & 1u) ? fma(P.omega, d[k], xk) : 0.0;
                        }
                    }
                }
            }
            {
                const double s3 = __shfl_down_sync(0xffffffffu, o[3], 1), s6 = __shfl_down_sync(0xffffffffu, o[6], 1);
                const double s9 = __shfl_down_sync(0xffffffffu, o[9], 1), s12 = __shfl_down_sync(0xffffffffu, o[12], 1);
                const double s16 = __shfl_down_sync(0xffffffffu, o[16], 1), s18 = __shfl_down_sync(0xffffffffu, o[18], 1);
                cdr[0] = o[0];
                cdr[1] = o[1];
                cdr[2] = o[2] + s3;
                cdr[3] = o[4];
                cdr[4] = s6;
                cdr[5] = o[8] + s9;
                cdr[6] = o[10];
                cdr[7] = s12;
                cdr[8] = o[14] + s16;
                cdr[9] = s18;
            }
            // x row y - 1 and K row y - 2 are dead: their slots take rows y + 3 and y + 2
            if (!XZERO) {
                __syncwarp();
                if (lane == 0) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    if (y + 3 <= yend + 1) load_x(y + 3);
                    if (y + 2 <= yend) load_k(y + 2);
                }
            }
        }
    }
    if (S.out || S.state) norm_finish<HW_NT>(S, nrm);
}

// ------------------------------------------------------------------------------------------
// accumulator slot of coarse plane kc within its restriction group (MG_RESTRICT_G0..G3)
__host__ __device__ constexpr int rslot(int kc) {
    return kc >= 8 ? 1 : (kc <= 1 ? 0 : (kc <= 4 ? kc - 2 : kc - 5));
}

// Row-marching fused residual + restriction b_H = P^T (b - A x) with TMA row chunks.
// A CTA owns coarse columns [I0, I0+QT) and coarse rows [J0, J0+MH); step s produces coarse rows
// J0 + s QR .. J0 + (s+1) QR - 1 from the fine residual rows 2(J0 + s QR) - 2 .. 2(J0 + s QR) + 2QR - 1,
// of which the lowest two are carried from step s-1 (no recompute in y).
constexpr int QT = 15, QR = 2, QF = 2 * QR;                 // coarse cols, coarse rows per step, fine rows per step
constexpr int Q_RW = 2 * QT + 2, Q_XW = 2 * QT + 6;          // fine r columns, x box width (origin 2 I0 - 4)
constexpr int QNT = Q_RW * QF;                               // 128 threads
constexpr int Q_XCH = 10 * QF * Q_XW, Q_BCH = 10 * QF * Q_RW;
constexpr int Q_SMEM = (3 * Q_XCH + 3 * Q_BCH) * 8 + 64;
// K field (third session): the K^{-1} planes of the x chunks' rows as a third chunk ring (same rows and columns as
// the x chunk, 2 planes) instead of gathers from global memory inside the residual
constexpr int Q_KCH = 2 * QF * Q_XW;
constexpr int Q_SMEM_K = (3 * Q_XCH + 3 * Q_BCH + 3 * Q_KCH) * 8 + 64;
static_assert(3 * (Q_SMEM_K + 1024) <= 228 * 1024, "three CTAs per SM");
static_assert((Q_KCH * 8) % 128 == 0, "K chunk slots 128-byte aligned");

template <bool HET>
__global__ void __launch_bounds__(QNT, 3) restrict_march_kernel(const __grid_constant__ CUtensorMap tmx,
                                                                const __grid_constant__ CUtensorMap tmb,
                                                                const __grid_constant__ CUtensorMap tmk,
                                                                const LevelParams L, int nc, int pitchc,
                                                                double* __restrict__ bc, int MH) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(128) double sm[];
    double* xr = sm;                    // [3][10][QF][Q_XW]
    double* br = xr + 3 * Q_XCH;        // [3][10][QF][Q_RW]  (b, overwritten by r)
    double* kq = br + 3 * Q_BCH;        // HET: [3][2][QF][Q_XW]  K^{-1} of the x chunks' rows
    uint64_t* bars = reinterpret_cast<uint64_t*>(kq + (HET ? 3 * Q_KCH : 0));
    if (*L.stop) return;
    constexpr bool DI = !HET;   // de-interleaved r columns (see the residual phase)
    const int n = L.n;
    const int I0 = blockIdx.x * QT, J0 = blockIdx.y * MH;
    const int crow = min(MH, nc + 1 - J0);
    const int nsteps = (crow + QR - 1) / QR;
    const int F0 = 2 * J0;
    const int t = threadIdx.x;
    const int nxc = nsteps + 2, nbc = nsteps + 1;
    // x chunk c: fine rows [F0 + (c-1) QF - 1, F0 + c QF - 1); b chunk d: fine rows [F0 + (d-1) QF, F0 + d QF)
    auto issue_x = [&](int c) {
        if (c < nxc) {
            mbar_expect_tx(&bars[c % 3], (Q_XCH + (HET ? Q_KCH : 0)) * 8);
            tma_load3(xr + (c % 3) * Q_XCH, &tmx, 2 * I0 - 4, F0 + (c - 1) * QF - 1, 0, &bars[c % 3]);
            if (HET) tma_load3(kq + (c % 3) * Q_KCH, &tmk, 2 * I0 - 4, F0 + (c - 1) * QF - 1, 0, &bars[c % 3]);
        }
    };
    auto issue_b = [&](int d) {
        if (d < nbc) {
            mbar_expect_tx(&bars[3 + d % 3], Q_BCH * 8);
            tma_load3(br + (d % 3) * Q_BCH, &tmb, 2 * I0 - 2, F0 + (d - 1) * QF, 0, &bars[3 + d % 3]);
        }
    };
    if (t == 0) {
        for (int k = 0; k < 6; ++k) mbar_init(&bars[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (t == 0) {
        issue_x(0);
        issue_x(1);
        issue_x(2);
        issue_b(0);
        issue_b(1);
    }
    const int64_t planec = (int64_t)(nc + 1) * pitchc;
    for (int s = -1; s < nsteps; ++s) {
        const int bslot = (s + 1) % 3;
        mbar_wait(&bars[(s + 1) % 3], ((s + 1) / 3) & 1);
        mbar_wait(&bars[(s + 2) % 3], ((s + 2) / 3) & 1);
        mbar_wait(&bars[3 + bslot], ((s + 1) / 3) & 1);
        {
            // fine residual row y = F0 + s QF + q, column i = 2 I0 - 2 + lx
            const int q = t / Q_RW, lx = t - q * Q_RW;
            const int y = F0 + s * QF + q, i = 2 * I0 - 2 + lx;
            const int ym = q, y0 = q + 1, yp = q + 2;   // offsets from the first row of x chunk s+1
            const double* base1 = xr + ((s + 1) % 3) * Q_XCH + (lx + 2);
            const double* base2 = xr + ((s + 2) % 3) * Q_XCH + (lx + 2);
            const double* xm = (ym < QF ? base1 + ym * Q_XW : base2 + (ym - QF) * Q_XW);
            const double* x0 = (y0 < QF ? base1 + y0 * Q_XW : base2 + (y0 - QF) * Q_XW);
            const double* xp = (yp < QF ? base1 + yp * Q_XW : base2 + (yp - QF) * Q_XW);
            double av[10];
            if (HET) {
                // K^{-1} of the cell rows y - 1 and y: rows ym, y0 of the K chunks (cells outside the mesh: 0)
                const double* kb1 = kq + ((s + 1) % 3) * Q_KCH + (lx + 2);
                const double* kb2 = kq + ((s + 2) % 3) * Q_KCH + (lx + 2);
                const double* km = (ym < QF ? kb1 + ym * Q_XW : kb2 + (ym - QF) * Q_XW);
                const double* k0 = (y0 < QF ? kb1 + y0 * Q_XW : kb2 + (y0 - QF) * Q_XW);
                apply_rows_kr<QF * Q_XW, QF * Q_XW>(L, xm, x0, xp, km, k0, av);
            } else {
                apply_rows<QF * Q_XW, false>(L, xm, x0, xp, i, y, av);
            }
            const double* bp = br + bslot * Q_BCH + q * Q_RW + lx;
            double rv[10];
#pragma unroll
            for (int k = 0; k < 10; ++k) rv[k] = is_active(k, i, y, n) ? bp[k * QF * Q_RW] - av[k] : 0.0;
            // scalar K: r replaces b in the chunk with its columns de-interleaved (even columns
            // first, then odd) so the restriction's stride-2 column reads hit consecutive banks;
            // every b of the row is read before any r lands (measured: 0.545 -> 0.518 ms at 4096^2;
            // with a K field the extra barrier costs more than it saves: 0.189 -> 0.225 ms at 2048^2)
            if (DI) __syncthreads();
            double* rp = br + bslot * Q_BCH + q * Q_RW + (!DI ? lx : (lx & 1) ? Q_RW / 2 + (lx >> 1) : (lx >> 1));
#pragma unroll
            for (int k = 0; k < 10; ++k) rp[k * QF * Q_RW] = rv[k];
        }
        __syncthreads();
        // coarse rows J = J0 + s QR + q: fine rows 2J - 2 .. 2J + 1 = rows 2q - 2 .. 2q + 1 of this step
        // (negative: the carried rows of b/r chunk s).  Warp w takes coarse plane group w
        // (MG_RESTRICT_G0..G3: planes {0,8}, {1,9}, {2,3,4}, {5,6,7}, ~23 entries each); lanes 0-14
        // coarse row q = 0, lanes 16-30 row q = 1.
        if (s >= 0) {
            const int grp = t >> 5, q = (t >> 4) & 1, cx = t & 15;
            const int I = I0 + cx, J = J0 + s * QR + q;
            if (cx < QT && I <= nc && J < J0 + crow) {
                const double* cur = br + bslot * Q_BCH + (DI ? cx + 1 : 2 * cx + 2);
                const double* car = br + ((s % 3) * Q_BCH) + (DI ? cx + 1 : 2 * cx + 2);
                const int64_t o = (int64_t)J * pitchc + I;
                // row pointer for fine-row offset f = 2q - 2cdJ + dj in [-2, 3]
#define ROWP(f) ((f) < 0 ? car + (QF + (f)) * Q_RW : cur + (f) * Q_RW)
// fine column 2cx + 2 - 2 cdI + di: parity di, de-interleaved index cx + 1 - cdI (+ Q_RW / 2 if odd)
#define RF(cdI, cdJ, di, dj, kf) \
    ROWP(2 * q - 2 * (cdJ) + (dj))[(kf) * (QF * Q_RW) + (DI ? (di) * (Q_RW / 2) - (cdI) : -2 * (cdI) + (di))]
                double acc[3] = {0.0, 0.0, 0.0};
#define MG_UG(kc, cdI, cdJ, di, dj, kf, w) acc[rslot(kc)] = fma(w, RF(cdI, cdJ, di, dj, kf), acc[rslot(kc)]);
                auto put = [&](int k, double v) { bc[k * planec + o] = is_active(k, I, J, nc) ? v : 0.0; };
                switch (grp) {
                    case 0: MG_RESTRICT_IL_G0(MG_UG) put(0, acc[0]); put(8, acc[1]); break;
                    case 1: MG_RESTRICT_IL_G1(MG_UG) put(1, acc[0]); put(9, acc[1]); break;
                    case 2: MG_RESTRICT_IL_G2(MG_UG) put(2, acc[0]); put(3, acc[1]); put(4, acc[2]); break;
                    default: MG_RESTRICT_IL_G3(MG_UG) put(5, acc[0]); put(6, acc[1]); put(7, acc[2]); break;
                }
#undef MG_UG
#undef RF
#undef ROWP
            }
        }
        __syncthreads();
        if (t == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue_x(s + 4);
            issue_b(s + 3);
        }
    }
}

// ------------------------------------------------------------------------------------------
// Row-marching inexact Braess-Sarazin relaxation, the structure of
// vanka_march2_kernel: 128 threads, one warp per row, 4 rows per step, single-row TMA rings
// (x, b / r, and for a K field the two K^{-1} planes) refilled one step ahead, 3 CTAs / SM.
//
// Stage A (bsr_a_march_kernel): r = b - A x, z_u = F_u^{-1} r_u (8-DoF displacement patches),
// g = alpha B_u z_u + tau B_w (tau D_w)^{-1} r_w - r_p and the first Jacobi sweep dp = omega_J g /
// diag(S) on the cells of a strip of BQ_T columns.  Step s computes the residual and patch rows
// j0 + sR + 2 .. + 5, the z_u rows j0 + sR + 1 .. + 4 and the g / dp cell rows j0 + sR .. + 3
// (lower rows carried from step s - 1).  Stage B (bsr_b_march_kernel): r again, y_u = r_u -
// alpha B_u^T dp, du = F_u^{-1} y_u, dw = (r_w - tau B_w^T dp) / (tau D_w), x + omega (du, dw, dp),
// rows as in vanka_march2_kernel (dp and K^{-1} arrive as 2-plane TMA rows).
constexpr int BQ_R = 4, BQ_NT = 128, BQ_W = 32, BQ_ROW = 10 * BQ_W, BQ_KROW = 2 * BQ_W;
constexpr int BMA_T = 26;                              // stage A: owned cells / strip (x box i0-2 .. i0+29)
constexpr int BMA_XR = 10, BMA_BR = 10, BMA_KR = 11, BMA_PR = 5, BMA_ZR = 5;
constexpr int BMA_PC = BMA_T + 2, BMA_ZC = BMA_T + 1;     // patch vertices i0 .. i0+27, z_u i0 .. i0+26
constexpr int BMA_SMEM = (BMA_XR * BQ_ROW + BMA_BR * BQ_ROW + BMA_KR * BQ_KROW + BMA_PR * 8 * BMA_PC + BMA_ZR * 5 * BMA_ZC) * 8 + 64;
constexpr int BB_T = 28;                              // stage B: owned indices / strip
constexpr int BB2_XR = 10, BB2_BR = 9, BB2_DR = 10, BB2_PR = 5, BB2_PC = BB_T + 1;
constexpr int BB2_SMEM = (BB2_XR * BQ_ROW + BB2_BR * BQ_ROW + 2 * BB2_DR * BQ_KROW + BB2_PR * 8 * BB2_PC) * 8 + 64;
constexpr int BB2_SMEM_NX = BB2_SMEM - BB2_XR * BQ_ROW * 8;   // stage B without the x ring (MODE 1, 2)
static_assert(3 * (BMA_SMEM + 1024) <= 228 * 1024 && 3 * (BB2_SMEM + 1024) <= 228 * 1024, "three CTAs per SM");
static_assert(BMA_T % 2 == 0 && BB_T % 2 == 0, "TMA box origins i0 - 2 must be even columns");

// 8-DoF displacement-patch residuals of vertex (a, b) from two r rows (r0: row b, rm: row b - 1,
// both at the vertex column): gather8's slot order
#define MG_GATHER8(rr, r0, rm, PS)                                                                  \
    rr[0] = (r0)[0 * (PS)];  rr[1] = (r0)[1 * (PS)];                                                \
    rr[2] = (r0)[2 * (PS)];  rr[3] = (r0)[2 * (PS) - 1]; rr[4] = (r0)[3 * (PS)]; rr[5] = (rm)[3 * (PS)]; \
    rr[6] = (r0)[4 * (PS) - 1]; rr[7] = (rm)[4 * (PS)];

template <bool HET, bool XZERO>
__global__ void __launch_bounds__(BQ_NT, 3) bsr_a_march_kernel(const __grid_constant__ CUtensorMap tmx,
                                                               const __grid_constant__ CUtensorMap tmb,
                                                               const __grid_constant__ CUtensorMap tmk,
                                                               const LevelParams L, const DispParams U, double omJ,
                                                               double* __restrict__ g, double* __restrict__ dp,
                                                               NormSink S, int MH, const double* __restrict__ jtab,
                                                               double* __restrict__ rs) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(128) double sm[];
    double* xr = sm;                          // [BMA_XR][10][32]
    double* br = xr + BMA_XR * BQ_ROW;         // [BMA_BR][10][32]  b, overwritten by r
    double* kr = br + BMA_BR * BQ_ROW;         // [BMA_KR][2][32]   K^{-1} (HET)
    double* pr = kr + BMA_KR * BQ_KROW;        // [BMA_PR][8][BMA_PC] displacement patch outputs
    double* zr = pr + BMA_PR * 8 * BMA_PC;      // [BMA_ZR][5][BMA_ZC] z_u
    uint64_t* bars = reinterpret_cast<uint64_t*>(zr + BMA_ZR * 5 * BMA_ZC);
    if (*L.stop) return;
    const int n = L.n;
    const int i0 = blockIdx.x * BMA_T, j0 = blockIdx.y * MH;
    const int rows = min(MH, n + 1 - j0);
    const int nsteps = (rows + BQ_R - 1) / BQ_R;
    const int t = threadIdx.x;
    auto sx = [&](int y) { return (y - j0 + 2 * BQ_R) % BMA_XR; };
    auto sb = [&](int y) { return (y - j0 + 2 * BQ_R) % BMA_BR; };
    auto sk = [&](int y) { return (y - j0 + 2 * BQ_R) % BMA_KR; };
    auto sp = [&](int y) { return (y - j0 + 2 * BQ_R) % BMA_PR; };
    auto sz = [&](int y) { return (y - j0 + 2 * BQ_R) % BMA_ZR; };
    // group g: x rows j0+gR+3 .. +6 (g = -1: j0-3 .. j0+2), b rows j0+gR+2 .. +5, K rows j0+gR+2 .. +5
    // (g = -1: j0-3 .. j0+1)
    auto issue = [&](int g) {
        if (g >= nsteps) return;
        uint64_t* bar = &bars[(g + 1) & 1];
        const int nx = XZERO ? 0 : (g < 0 ? 6 : BQ_R);
        const int nk = HET ? (g < 0 ? 5 : BQ_R) : 0;
        mbar_expect_tx(bar, ((nx + BQ_R) * BQ_ROW + nk * BQ_KROW) * 8);
        const int xfirst = g < 0 ? j0 - 3 : j0 + g * BQ_R + 3;
#pragma unroll 1
        for (int k = 0; k < nx; ++k) tma_load3(xr + sx(xfirst + k) * BQ_ROW, &tmx, i0 - 2, xfirst + k, 0, bar);
#pragma unroll 1
        for (int k = 0; k < BQ_R; ++k) {
            const int y = j0 + g * BQ_R + 2 + k;
            tma_load3(br + sb(y) * BQ_ROW, &tmb, i0 - 2, y, 0, bar);
        }
        const int kfirst = g < 0 ? j0 - 3 : j0 + g * BQ_R + 2;
#pragma unroll 1
        for (int k = 0; k < nk; ++k) tma_load3(kr + sk(kfirst + k) * BQ_KROW, &tmk, i0 - 2, kfirst + k, 0, bar);
    };
    // K^{-1} of triangle sh of cell (ci, cj) (0 outside the mesh: TMA zero fill / zeroed pyramid)
    auto kinv = [&](int ci, int cj, int sh) -> double {
        if (!HET) return L.kinv;
        return kr[sk(cj) * BQ_KROW + sh * BQ_W + (ci - (i0 - 2))];
    };
    auto Dw = [&](int k, int i, int j) -> double {   // D_w of the RT0 DoF of plane k at index (i, j)
        double d = 0.0;
#define MG_I(kk, cdx, cdy, sh, q) d = fma(L.mw1d[sh][(q) - 9], kinv(i + (cdx), j + (cdy), sh), d);
        if (k == 5) { MG_INCIDENT_5(MG_I) }
        else if (k == 6) { MG_INCIDENT_6(MG_I) }
        else { MG_INCIDENT_7(MG_I) }
#undef MG_I
        return d;
    };
    if (t == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (t == 0) {
        issue(-1);
        issue(0);
    }
    const int64_t plane = L.plane;
    double nrm = 0.0;
    for (int s = -1; s < nsteps; ++s) {
        // the Jacobi table entries of this thread's cell (g phase), issued a whole step ahead of their use
        double tpre[7];
        {
            const int yc = j0 + s * BQ_R + (t >> 5), ic = i0 + (t & 31);
            const bool ok = s >= 0 && (t & 31) < BMA_T && ic < n && yc < n && yc < j0 + rows;
            const double* tb = jtab + (ok ? (int64_t)yc * L.pitch + ic : 0);
            tpre[0] = ok ? __ldg(tb) : 0.0;
            tpre[1] = ok ? __ldg(tb + plane) : 0.0;
            tpre[2] = ok ? __ldg(tb + 2 * plane) : 0.0;
            tpre[3] = ok ? __ldg(tb + L.pitch) : 0.0;
            tpre[4] = ok ? __ldg(tb + plane + 1) : 0.0;
            tpre[5] = ok ? __ldg(tb + 3 * plane) : 0.0;
            tpre[6] = ok ? __ldg(tb + 4 * plane) : 0.0;
        }
        mbar_wait(&bars[(s + 1) & 1], ((s + 1) >> 1) & 1);
        const int q = t >> 5, lane = t & 31;
        // ---- residual rows y = j0 + sR + 2 + q at columns i0-1 .. i0+27
        if (lane < BMA_T + 3) {
            const int y = j0 + s * BQ_R + 2 + q, i = i0 - 1 + lane;
            double* bp = br + sb(y) * BQ_ROW + (lane + 1);
            double rv[10];
            if (!XZERO) {
                const double* xm = xr + sx(y - 1) * BQ_ROW + (lane + 1);
                const double* x0 = xr + sx(y) * BQ_ROW + (lane + 1);
                const double* xp = xr + sx(y + 1) * BQ_ROW + (lane + 1);
                double av[10];
                if (HET) apply_rows_kr<BQ_W, BQ_W>(L, xm, x0, xp, kr + sk(y - 1) * BQ_KROW + (lane + 1),
                                                   kr + sk(y) * BQ_KROW + (lane + 1), av);
                else apply_rows<BQ_W, false>(L, xm, x0, xp, i, y, av);
#pragma unroll
                for (int k = 0; k < 10; ++k) rv[k] = is_active(k, i, y, n) ? bp[k * BQ_W] - av[k] : 0.0;
#pragma unroll
                for (int k = 0; k < 10; ++k) bp[k * BQ_W] = rv[k];
            } else {
#pragma unroll
                for (int k = 0; k < 10; ++k) rv[k] = bp[k * BQ_W];
            }
            if (lane >= 1 && lane <= BMA_T && i <= n && y >= j0 && y < j0 + rows) {
#pragma unroll
                for (int k = 0; k < 10; ++k) nrm = fma(rv[k], rv[k], nrm);
                // r_u, r_w of the owned positions for stage B (bsr_b_march_kernel<.., 2> reads them
                // instead of evaluating the residual a second time)
                if (!XZERO && rs) {
                    const int64_t o = (int64_t)y * L.pitch + i;
#pragma unroll
                    for (int k = 0; k < 8; ++k) rs[k * L.plane + o] = rv[k];
                }
            }
        }
        __syncthreads();
        // ---- displacement patches at vertex rows bb = j0 + sR + 2 + q, vertices i0 .. i0+27
        if (lane < BMA_PC) {
            const int a = i0 + lane, bb = j0 + s * BQ_R + 2 + q;
            double* out = pr + sp(bb) * (8 * BMA_PC) + lane;
            if (a <= n && bb >= 0 && bb <= n) {
                const double* r0 = br + sb(bb) * BQ_ROW + (lane + 2);
                const double* rm = br + sb(bb - 1) * BQ_ROW + (lane + 2);
                double rr[8];
                MG_GATHER8(rr, r0, rm, BQ_W)
                patch_apply8(U, vertex_class(a, bb, n), rr, out, BMA_PC);
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) out[k * BMA_PC] = 0.0;
            }
        }
        __syncthreads();
        // ---- z_u rows y = j0 + sR + 1 + q at columns i0 .. i0+26 (patch rows y, y + 1)
        if (lane < BMA_ZC) {
            const int y = j0 + s * BQ_R + 1 + q;
            const double* c0 = pr + sp(y) * (8 * BMA_PC) + lane;
            const double* c1 = pr + sp(y + 1) * (8 * BMA_PC) + lane;
            double* zo = zr + sz(y) * (5 * BMA_ZC) + lane;
#define CC(sl, dx, dy) ((dy) > 0 ? c1 : c0)[(sl) * BMA_PC + (dx)]
            zo[0 * BMA_ZC] = CC(0, 0, 0);
            zo[1 * BMA_ZC] = CC(1, 0, 0);
            zo[2 * BMA_ZC] = CC(2, 0, 0) + CC(3, 1, 0);
            zo[3 * BMA_ZC] = CC(4, 0, 0) + CC(5, 0, 1);
            zo[4 * BMA_ZC] = CC(6, 1, 0) + CC(7, 0, 1);
#undef CC
        }
        __syncthreads();
        // ---- g and the first Jacobi sweep on the cells of rows y = j0 + sR + q, columns i0 .. i0+25
        if (s >= 0 && lane < BMA_T) {
            const int y = j0 + s * BQ_R + q, i = i0 + lane;
            if (i <= n && y < j0 + rows) {
                const int64_t o = (int64_t)y * L.pitch + i;
                if (i < n && y < n) {
                    const double* z0 = zr + sz(y) * (5 * BMA_ZC) + lane;
                    const double* z1 = zr + sz(y + 1) * (5 * BMA_ZC) + lane;
                    const double* r0 = br + sb(y) * BQ_ROW + (lane + 2);
                    const double* r1 = br + sb(y + 1) * BQ_ROW + (lane + 2);
                    // tau / D_w of the five edges of the cell (H(i,y), V(i,y), D(i,y), H(i,y+1),
                    // V(i+1,y); 0 if inactive) and 1 / diag S of its triangles: the Jacobi table
                    const double tH0 = tpre[0], tV0 = tpre[1], tD = tpre[2];
                    const double tH1 = tpre[3], tV1 = tpre[4];
                    const double itau2 = 1.0 / (L.tau * L.tau);
#pragma unroll
                    for (int sh = 0; sh < 2; ++sh) {
                        const double te[3] = {sh == 0 ? tH0 : tH1, sh == 0 ? tV0 : tV1, tD};
                        double gu = 0.0, gw = 0.0;
#define MG_L(s_, q_, dx, dy, pl)                                                                  \
    if ((s_) == sh) {                                                                             \
        if ((q_) < 9) gu = fma(L.bu[s_][(q_) < 9 ? (q_) : 0], ((dy) ? z1 : z0)[(pl) * BMA_ZC + (dx)], gu); \
        else if ((q_) < 12) {                                                                     \
            const int e = (q_) < 12 ? (q_) - 9 : 0;                                               \
            const double rw = ((dy) ? r1 : r0)[(pl) * BQ_W + (dx)];                               \
            gw = fma(L.bw[s_][e], rw * te[e] * itau2, gw);                                        \
        }                                                                                         \
    }
                        MG_LOCAL_0(MG_L)
                        MG_LOCAL_1(MG_L)
#undef MG_L
                        const double rp = r0[(8 + sh) * BQ_W];
                        const double gv = L.alpha * gu + L.tau * gw - rp;
                        g[sh * plane + o] = gv;
                        dp[sh * plane + o] = omJ * gv * tpre[5 + sh];
                    }
                } else {
                    g[o] = 0.0;
                    g[plane + o] = 0.0;
                    dp[o] = 0.0;
                    dp[plane + o] = 0.0;
                }
            }
        }
        __syncthreads();
        if (t == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(s + 2);
        }
    }
    if (S.out || S.state) norm_finish<BQ_NT>(S, nrm);
}

// MODE 0: r = b - A x evaluated here; 1: x = 0 (r = b); 2: r_u, r_w read from the vector stage A wrote (the
// "b" map points at it, 8 planes), x read at the owners only -- no x ring, no second residual
template <bool HET, int MODE>
__global__ void __launch_bounds__(BQ_NT, 3) bsr_b_march_kernel(const __grid_constant__ CUtensorMap tmx,
                                                               const __grid_constant__ CUtensorMap tmb,
                                                               const __grid_constant__ CUtensorMap tmd,
                                                               const __grid_constant__ CUtensorMap tmk,
                                                               const LevelParams L, const DispParams U, double omega,
                                                               double* __restrict__ xo, int MH,
                                                               const double* __restrict__ xin) {
    constexpr bool XZERO = MODE != 0;                       // no x ring, r taken from the b rows
    constexpr int XR = MODE == 0 ? BB2_XR : 0;              // x ring rows
    constexpr int BROWB = (MODE == 2 ? 8 * BQ_W : BQ_ROW);  // doubles per b / r box row
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(128) double sm[];
    double* xr = sm;                          // [BB2_XR][10][32]
    double* br = xr + XR * BQ_ROW;            // [BB2_BR][10][32]  b, overwritten by (y_u, r_w)
    double* dr = br + BB2_BR * BQ_ROW;        // [BB2_DR][2][32]   dp
    double* kr = dr + BB2_DR * BQ_KROW;       // [BB2_DR][2][32]   K^{-1} (HET)
    double* pr = kr + BB2_DR * BQ_KROW;       // [BB2_PR][8][BB2_PC]
    uint64_t* bars = reinterpret_cast<uint64_t*>(pr + BB2_PR * 8 * BB2_PC);
    if (*L.stop) return;
    const int n = L.n;
    const int i0 = blockIdx.x * BB_T, j0 = blockIdx.y * MH;
    const int rows = min(MH, n + 1 - j0);
    const int nsteps = (rows + BQ_R - 1) / BQ_R;
    const int t = threadIdx.x;
    auto sx = [&](int y) { return (y - j0 + 2 * BQ_R) % (XR ? XR : 1); };
    auto sb = [&](int y) { return (y - j0 + 2 * BQ_R) % BB2_BR; };
    auto sd = [&](int y) { return (y - j0 + 2 * BQ_R) % BB2_DR; };
    auto sp = [&](int y) { return (y - j0 + 2 * BQ_R) % BB2_PR; };
    // group g: x rows j0+gR+2 .. +5 (g = -1: j0-R .. j0+1), b rows j0+gR+1 .. +4, dp and K rows
    // j0+gR+1 .. +4 (g = -1: j0-4 .. j0)
    auto issue = [&](int g) {
        if (g >= nsteps) return;
        uint64_t* bar = &bars[(g + 1) & 1];
        const int nx = XZERO ? 0 : (g < 0 ? BQ_R + 2 : BQ_R);
        const int nd = g < 0 ? 5 : BQ_R;
        mbar_expect_tx(bar, (nx * BQ_ROW + BQ_R * BROWB + (HET ? 2 : 1) * nd * BQ_KROW) * 8);
        const int xfirst = g < 0 ? j0 - BQ_R : j0 + g * BQ_R + 2;
#pragma unroll 1
        for (int k = 0; k < nx; ++k) tma_load3(xr + sx(xfirst + k) * BQ_ROW, &tmx, i0 - 2, xfirst + k, 0, bar);
#pragma unroll 1
        for (int k = 0; k < BQ_R; ++k) {
            const int y = j0 + g * BQ_R + 1 + k;
            tma_load3(br + sb(y) * BQ_ROW, &tmb, i0 - 2, y, 0, bar);
        }
        const int dfirst = g < 0 ? j0 - 4 : j0 + g * BQ_R + 1;
#pragma unroll 1
        for (int k = 0; k < nd; ++k) {
            tma_load3(dr + sd(dfirst + k) * BQ_KROW, &tmd, i0 - 2, dfirst + k, 0, bar);
            if (HET) tma_load3(kr + sd(dfirst + k) * BQ_KROW, &tmk, i0 - 2, dfirst + k, 0, bar);
        }
    };
    auto kinv = [&](int ci, int cj, int sh) -> double {
        if (!HET) return L.kinv;
        return kr[sd(cj) * BQ_KROW + sh * BQ_W + (ci - (i0 - 2))];
    };
    auto dpc = [&](int ci, int cj, int sh) -> double { return dr[sd(cj) * BQ_KROW + sh * BQ_W + (ci - (i0 - 2))]; };
    if (t == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (t == 0) {
        issue(-1);
        issue(0);
    }
    for (int s = -1; s < nsteps; ++s) {
        // MODE 2: x of this thread's owner position, issued a whole step ahead of its use
        double xpre[10];
        if (MODE == 2) {
            const int yo = j0 + s * BQ_R + (t >> 5), io = i0 + (t & 31);
            const bool ok = s >= 0 && (t & 31) < BB_T && io <= n && yo < j0 + rows;
            const int64_t oo = ok ? (int64_t)yo * L.pitch + io : 0;
#pragma unroll
            for (int k = 0; k < 10; ++k) xpre[k] = ok ? __ldg(xin + k * L.plane + oo) : 0.0;
        }
        mbar_wait(&bars[(s + 1) & 1], ((s + 1) >> 1) & 1);
        const int q = t >> 5, lane = t & 31;
        // ---- rows y = j0 + sR + 1 + q at columns i0-1 .. i0+28: r, then y_u = r_u - alpha B_u^T dp
        if (lane < BB_T + 2) {
            const int y = j0 + s * BQ_R + 1 + q, i = i0 - 1 + lane;
            double* bp = br + sb(y) * BQ_ROW + (lane + 1);
            double rv[8];
            if (!XZERO) {
                const double* xm = xr + sx(y - 1) * BQ_ROW + (lane + 1);
                const double* x0 = xr + sx(y) * BQ_ROW + (lane + 1);
                const double* xp = xr + sx(y + 1) * BQ_ROW + (lane + 1);
                double av[10];
                if (HET) apply_rows_kr<BQ_W, BQ_W>(L, xm, x0, xp, kr + sd(y - 1) * BQ_KROW + (lane + 1),
                                                   kr + sd(y) * BQ_KROW + (lane + 1), av);
                else apply_rows<BQ_W, false>(L, xm, x0, xp, i, y, av);
#pragma unroll
                for (int k = 0; k < 8; ++k) rv[k] = is_active(k, i, y, n) ? bp[k * BQ_W] - av[k] : 0.0;
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) rv[k] = bp[k * BQ_W];
            }
            double bt[5] = {0, 0, 0, 0, 0};
#define MG_I(k, cdx, cdy, sh, qq) bt[k] = fma(L.bu[sh][qq], dpc(i + (cdx), y + (cdy), sh), bt[k]);
            MG_INCIDENT_0(MG_I) MG_INCIDENT_1(MG_I) MG_INCIDENT_2(MG_I) MG_INCIDENT_3(MG_I) MG_INCIDENT_4(MG_I)
#undef MG_I
#pragma unroll
            for (int k = 0; k < 5; ++k) bp[k * BQ_W] = is_active(k, i, y, n) ? rv[k] - L.alpha * bt[k] : rv[k];
#pragma unroll
            for (int k = 5; k < 8; ++k) bp[k * BQ_W] = rv[k];
        }
        __syncthreads();
        // ---- displacement patches at vertex rows bb = j0 + sR + 1 + q, vertices i0 .. i0+28
        if (lane < BB2_PC) {
            const int a = i0 + lane, bb = j0 + s * BQ_R + 1 + q;
            double* out = pr + sp(bb) * (8 * BB2_PC) + lane;
            if (a <= n && bb >= 0 && bb <= n) {
                const double* r0 = br + sb(bb) * BQ_ROW + (lane + 2);
                const double* rm = br + sb(bb - 1) * BQ_ROW + (lane + 2);
                double rr[8];
                MG_GATHER8(rr, r0, rm, BQ_W)
                patch_apply8(U, vertex_class(a, bb, n), rr, out, BB2_PC);
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) out[k * BB2_PC] = 0.0;
            }
        }
        __syncthreads();
        // ---- owners y = j0 + sR + q: x + omega (du, dw, dp)
        if (s >= 0 && lane < BB_T) {
            const int y = j0 + s * BQ_R + q, i = i0 + lane;
            if (i <= n && y < j0 + rows) {
                const double* c0 = pr + sp(y) * (8 * BB2_PC) + lane;
                const double* c1 = pr + sp(y + 1) * (8 * BB2_PC) + lane;
#define CC(sl, dx, dy) ((dy) > 0 ? c1 : c0)[(sl) * BB2_PC + (dx)]
                double d[10];
                d[0] = CC(0, 0, 0);
                d[1] = CC(1, 0, 0);
                d[2] = CC(2, 0, 0) + CC(3, 1, 0);
                d[3] = CC(4, 0, 0) + CC(5, 0, 1);
                d[4] = CC(6, 1, 0) + CC(7, 0, 1);
#undef CC
                double bw[3] = {0, 0, 0};
#define MG_I(k, cdx, cdy, sh, qq) bw[(k) - 5] = fma(L.bw[sh][(qq) - 9], dpc(i + (cdx), y + (cdy), sh), bw[(k) - 5]);
                MG_INCIDENT_5(MG_I) MG_INCIDENT_6(MG_I) MG_INCIDENT_7(MG_I)
#undef MG_I
                const double* rw = br + sb(y) * BQ_ROW + (lane + 2);
#pragma unroll
                for (int k = 5; k < 8; ++k) {
                    double dwk = 0.0;
#define MG_I(kk, cdx, cdy, sh, qq) dwk = fma(L.mw1d[sh][(qq) - 9], kinv(i + (cdx), y + (cdy), sh), dwk);
                    if (k == 5) { MG_INCIDENT_5(MG_I) }
                    else if (k == 6) { MG_INCIDENT_6(MG_I) }
                    else { MG_INCIDENT_7(MG_I) }
#undef MG_I
                    d[k] = is_active(k, i, y, n) ? (rw[k * BQ_W] - L.tau * bw[k - 5]) / (L.tau * dwk) : 0.0;
                }
                d[8] = dpc(i, y, 0);
                d[9] = dpc(i, y, 1);
                const double* xv = xr + sx(y) * BQ_ROW + (lane + 2);
                const int64_t o = (int64_t)y * L.pitch + i;
#pragma unroll
                for (int k = 0; k < 10; ++k) {
                    const double xk = MODE == 1 ? 0.0 : (MODE == 2 ? xpre[k] : xv[k * BQ_W]);
                    xo[k * L.plane + o] = is_active(k, i, y, n) ? fma(omega, d[k], xk) : 0.0;
                }
            }
        }
        __syncthreads();
        if (t == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(s + 2);
        }
    }
}
// ------------------------------------------------------------------------------------------
// patch_apply8 with the 8 outputs in registers (same arithmetic and order)
__device__ __forceinline__ void patch_apply8r(const DispParams& U, int cls, const double rr[8], double o[8]) {
    if (cls == 0) {
        double hp[3], hm[5];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            hp[q] = rr[2 + 2 * q] - rr[3 + 2 * q];
            hm[2 + q] = rr[2 + 2 * q] + rr[3 + 2 * q];
        }
        hm[0] = rr[0];
        hm[1] = rr[1];
        double yp[3] = {0, 0, 0}, ym[5] = {0, 0, 0, 0, 0};
#pragma unroll
        for (int c = 0; c < 5; ++c) {
#pragma unroll
            for (int a = 0; a < 5; ++a) ym[a] = fma(U.umT[c][a], hm[c], ym[a]);
            if (c < 3) {
#pragma unroll
                for (int a = 0; a < 3; ++a) yp[a] = fma(U.upT[c][a], hp[c], yp[a]);
            }
        }
        o[0] = ym[0];
        o[1] = ym[1];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            o[2 + 2 * q] = ym[2 + q] + yp[q];
            o[3 + 2 * q] = ym[2 + q] - yp[q];
        }
    } else {
        // boundary classes: one output row of coefficient loads in flight -- the next row's address
        // depends on this row's sum through an opaque (never taken) NaN test, so ptxas cannot hoist all
        // 64 loads and spill the interior path (a NaN sum only ever meets NaN sums)
        const double* G = U.ubnd + cls * 64;
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            double sacc = 0.0;
#pragma unroll
            for (int c = 0; c < 8; ++c) sacc = fma(__ldg(G + a * 8 + c), rr[c], sacc);
            o[a] = sacc;
            int dep;
            asm volatile("{\n\t.reg .pred p;\n\tsetp.nan.f64 p, %1, %1;\n\tselp.s32 %0, 1, 0, p;\n\t}" : "=r"(dep) : "d"(sacc));
            G += dep;
        }
    }
}

// Warp-marching BSR stage B (round 2; levels with n >= MG_WARP_MIN_N): the arithmetic of
// bsr_b_march_kernel (r, y_u = r_u - alpha B_u^T dp, F_u^{-1} by 8-DoF displacement patches,
// dw = D_w^{-1}(r_w - tau B_w^T dp), x + omega (du, dw, dp)) organised like
// vanka_warp_kernel: one warp per 30-column strip, one row per iteration -- residual and y_u row y,
// patch row y (left neighbour's y_u by shuffle, row y - 1's carried), owner row y - 1 (right
// neighbour's corrections by shuffle, patch row y - 1's dy = 0 sums carried, r_w of row y - 1
// carried).  x (4 rows), b (1), dp and K^{-1} (4 rows, 2 planes) arrive by TMA one iteration ahead.
constexpr int WQ_DROW = 2 * WXW, WQ_DSLOT = (WQ_DROW + 15) / 16 * 16, WQ_DR = 4;
template <bool HET> struct WQGeom {
    static constexpr int BYTES = ((WXR * WXSLOT + WBSLOT + (HET ? 2 : 1) * WQ_DR * WQ_DSLOT) * 8 + 128 + 127) / 128 * 128;
    static constexpr int NW = 232448 / BYTES > 12 ? 12 : 232448 / BYTES;   // one CTA per SM, <= 168 registers
    static constexpr int NT = 32 * NW, SMEM = NW * BYTES;
};
template <bool HET, bool XZERO>
__global__ void __launch_bounds__(WQGeom<HET>::NT, 1) bsr_b_warp_kernel(const __grid_constant__ CUtensorMap tmx,
                                                                       const __grid_constant__ CUtensorMap tmb,
                                                                       const __grid_constant__ CUtensorMap tmd,
                                                                       const __grid_constant__ CUtensorMap tmk,
                                                                       const LevelParams L, const DispParams U,
                                                                       double omega, double* __restrict__ xo, int MH,
                                                                       int nstrips, int ntasks) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(128) double sm[];
    if (*L.stop) return;
    const int n = L.n;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int task = blockIdx.x * WQGeom<HET>::NW + w;
    if (task >= ntasks) return;
    double* xr = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + w * WQGeom<HET>::BYTES);
    double* br = xr + WXR * WXSLOT;
    double* dr = br + WBSLOT;                          // [WQ_DR][2][WXW] dp
    double* kr = dr + WQ_DR * WQ_DSLOT;                // [WQ_DR][2][WXW] K^{-1} (HET)
    uint64_t* xbar = reinterpret_cast<uint64_t*>(kr + (HET ? WQ_DR * WQ_DSLOT : 0));
    uint64_t* bbar = xbar + WXR;
    uint64_t* dbar = bbar + 1;
    const int i0 = (task % nstrips) * WT, j0 = (task / nstrips) * MH;
    const int rows = min(MH, n + 1 - j0);
    const int yend = j0 + rows;
    const int i = i0 - 1 + lane;
    // x rows j0 - 2 .. yend + 1 (q = y - j0 + 2), b rows j0 - 1 .. yend (q = y - j0 + 1), dp / K rows
    // j0 - 2 .. yend (q = y - j0 + 2)
    auto load_x = [&](int y) {
        const int q = y - (j0 - 2);
        mbar_expect_tx(&xbar[q % WXR], WXROW * 8);
        tma_load3(xr + (q % WXR) * WXSLOT, &tmx, i0 - 2, y, 0, &xbar[q % WXR]);
    };
    auto load_b = [&](int y) {
        mbar_expect_tx(bbar, WBROW * 8);
        tma_load3(br, &tmb, i0 - 2, y, 0, bbar);
    };
    auto load_d = [&](int y) {
        const int q = y - (j0 - 2);
        mbar_expect_tx(&dbar[q % WQ_DR], (HET ? 2 : 1) * WQ_DROW * 8);
        tma_load3(dr + (q % WQ_DR) * WQ_DSLOT, &tmd, i0 - 2, y, 0, &dbar[q % WQ_DR]);
        if (HET) tma_load3(kr + (q % WQ_DR) * WQ_DSLOT, &tmk, i0 - 2, y, 0, &dbar[q % WQ_DR]);
    };
    auto wait_x = [&](int y) { const int q = y - (j0 - 2); mbar_wait(&xbar[q % WXR], (q / WXR) & 1); };
    auto wait_b = [&](int y) { const int q = y - (j0 - 1); mbar_wait(bbar, q & 1); };
    auto wait_d = [&](int y) { const int q = y - (j0 - 2); mbar_wait(&dbar[q % WQ_DR], (q / WQ_DR) & 1); };
    auto xrow = [&](int y) { return xr + ((y - (j0 - 2)) % WXR) * WXSLOT; };
    auto drow = [&](int y) { return dr + ((y - (j0 - 2)) % WQ_DR) * WQ_DSLOT; };
    auto krow = [&](int y) { return kr + ((y - (j0 - 2)) % WQ_DR) * WQ_DSLOT; };
    // dp / K^{-1} of triangle sh of cell (ci, cj) (cj one of the rows in the ring)
    auto dpc = [&](int ci, int cj, int sh) { return drow(cj)[sh * WXW + (ci - (i0 - 2))]; };
    auto kinv = [&](int ci, int cj, int sh) -> double {
        if (!HET) return L.kinv;
        return krow(cj)[sh * WXW + (ci - (i0 - 2))];
    };
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < WXR; ++k) mbar_init(&xbar[k], 1);
        mbar_init(bbar, 1);
#pragma unroll
        for (int k = 0; k < WQ_DR; ++k) mbar_init(&dbar[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    if (lane == 0) {
        if (!XZERO)
#pragma unroll
            for (int k = 0; k < WXR; ++k) load_x(j0 - 2 + k);
        load_b(j0 - 1);
        // dp / K rows j0 - 2 .. j0 (the end of iteration y loads row y + 2 into the slot of row y - 2)
#pragma unroll
        for (int k = 0; k < WQ_DR - 1; ++k)
            if (j0 - 2 + k <= yend) load_d(j0 - 2 + k);
    }
    if (!XZERO) {
        wait_x(j0 - 2);
        wait_x(j0 - 1);
    }
    wait_d(j0 - 2);
    // carried: y_u of row y - 1 (planes 3, 4), the left neighbour's plane-4 y_u of row y - 1 is not
    // needed (gather8 reads (a-1, b) only in the current row), r_w of row y - 1, the dy = 0 sums
    double yp3 = 0, yp4 = 0, rw5 = 0, rw6 = 0, rw7 = 0;
    double cd0 = 0, cd1 = 0, cd2 = 0, cd3 = 0, cd4 = 0;
#pragma unroll 1
    for (int y = j0 - 1; y <= yend; ++y) {
        if (!XZERO) wait_x(y + 1);
        wait_b(y);
        wait_d(y);
        // ---- r and y_u, row y
        double rv[8];
        {
            const double* bp = br + (lane + 1);
            if (!XZERO) {
                const double* x0 = xrow(y) + (lane + 1);
                double av[10];
                if (HET) apply_rows_kr<WXW, WXW>(L, xrow(y - 1) + (lane + 1), x0, xrow(y + 1) + (lane + 1),
                                                 krow(y - 1) + (lane + 1), krow(y) + (lane + 1), av);
                else apply_rows<WXW, false>(L, xrow(y - 1) + (lane + 1), x0, xrow(y + 1) + (lane + 1), i, y, av);
#pragma unroll
                for (int k = 0; k < 8; ++k) rv[k] = is_active(k, i, y, n) ? bp[k * WBW] - av[k] : 0.0;
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) rv[k] = bp[k * WBW];
            }
        }
        __syncwarp();
        if (lane == 0 && y + 1 <= yend) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            load_b(y + 1);
        }
        double yu[5];
        {
            double bt[5] = {0, 0, 0, 0, 0};
#define MG_I(k, cdx, cdy, sh, qq) bt[k] = fma(L.bu[sh][qq], dpc(i + (cdx), y + (cdy), sh), bt[k]);
            MG_INCIDENT_0(MG_I) MG_INCIDENT_1(MG_I) MG_INCIDENT_2(MG_I) MG_INCIDENT_3(MG_I) MG_INCIDENT_4(MG_I)
#undef MG_I
#pragma unroll
            for (int k = 0; k < 5; ++k) yu[k] = is_active(k, i, y, n) ? rv[k] - L.alpha * bt[k] : rv[k];
        }
        // ---- patch row y (vertex (i, y)); gather8: (a, b) own, (a - 1, b) by shuffle, (a, b - 1) carried
        const double l2 = __shfl_up_sync(0xffffffffu, yu[2], 1), l4 = __shfl_up_sync(0xffffffffu, yu[4], 1);
        double o[8];
        if (y >= j0 && lane >= 1 && i <= n && y <= n) {
            double rr[8];
            rr[0] = yu[0]; rr[1] = yu[1]; rr[2] = yu[2]; rr[3] = l2; rr[4] = yu[3]; rr[5] = yp3; rr[6] = l4; rr[7] = yp4;
            patch_apply8r(U, vertex_class(i, y, n), rr, o);
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) o[k] = 0.0;
        }
        yp3 = yu[3];
        yp4 = yu[4];
        // ---- owner row y - 1
        if (y >= j0 + 1 && lane >= 1 && lane <= WT && i <= n) {
            const int yo = y - 1;
            double d[10];
            d[0] = cd0;
            d[1] = cd1;
            d[2] = cd2;
            d[3] = cd3 + o[5];
            d[4] = cd4 + o[7];
            double bw[3] = {0, 0, 0};
#define MG_I(k, cdx, cdy, sh, qq) bw[(k) - 5] = fma(L.bw[sh][(qq) - 9], dpc(i + (cdx), yo + (cdy), sh), bw[(k) - 5]);
            MG_INCIDENT_5(MG_I) MG_INCIDENT_6(MG_I) MG_INCIDENT_7(MG_I)
#undef MG_I
            const double rwv[3] = {rw5, rw6, rw7};
#pragma unroll
            for (int k = 5; k < 8; ++k) {
                double dwk = 0.0;
#define MG_I(kk, cdx, cdy, sh, qq) dwk = fma(L.mw1d[sh][(qq) - 9], kinv(i + (cdx), yo + (cdy), sh), dwk);
                if (k == 5) { MG_INCIDENT_5(MG_I) }
                else if (k == 6) { MG_INCIDENT_6(MG_I) }
                else { MG_INCIDENT_7(MG_I) }
#undef MG_I
                d[k] = is_active(k, i, yo, n) ? (rwv[k - 5] - L.tau * bw[k - 5]) / (L.tau * dwk) : 0.0;
            }
            d[8] = dpc(i, yo, 0);
            d[9] = dpc(i, yo, 1);
            const double* xv = xrow(yo) + (lane + 1);
            const int64_t off = (int64_t)yo * L.pitch + i;
#pragma unroll
            for (int k = 0; k < 10; ++k) {
                const double xk = XZERO ? 0.0 : xv[k * WXW];
                xo[k * L.plane + off] = is_active(k, i, yo, n) ? fma(omega, d[k], xk) : 0.0;
            }
        }
        rw5 = rv[5];
        rw6 = rv[6];
        rw7 = rv[7];
        {
            const double s3 = __shfl_down_sync(0xffffffffu, o[3], 1), s6 = __shfl_down_sync(0xffffffffu, o[6], 1);
            cd0 = o[0];
            cd1 = o[1];
            cd2 = o[2] + s3;
            cd3 = o[4];
            cd4 = s6;
        }
        // x row y - 1 and dp / K row y - 2 are dead: their slots take rows y + 3 and y + 2
        __syncwarp();
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (!XZERO && y + 3 <= yend + 1) load_x(y + 3);
            if (y + 2 <= yend) load_d(y + 2);
        }
    }
}

#undef MG_GATHER8

// ------------------------------------------------------------------------------------------
// Row-marching residual / operator application (levels with n >= 512, scalar K): x rows arrive as
// TMA boxes (32 columns x 1 row x 10 planes) in a 10-row ring one step ahead, one warp per row,
// 28 owned columns per strip; b is read straight from global (one coalesced pass).
// MODE 0: r = b - A x (+||r||^2), MODE 1: y = A x on the active slots (FGMRES), MODE 2: ||b - A x||^2.
constexpr int RM_T = 28, RM_R = 4, RM_NT = 128, RM_XR = 10, RM_W = 32, RM_ROW = 10 * RM_W;
constexpr int RM_SMEM = RM_XR * RM_ROW * 8 + 64;
// K field (third session): the two K^{-1} planes of the cell rows in a ring of their own (rows y - 1, y of residual
// row y; group g: rows j0+gR .. j0+gR+3, g = 0 also j0-1), read by apply_rows_kr
constexpr int RM_KROW = 2 * RM_W, RM_SMEM_K = (RM_XR * RM_ROW + RM_XR * RM_KROW) * 8 + 64;

template <int MODE, bool HET = false>
__global__ void __launch_bounds__(RM_NT) residual_march_kernel(const __grid_constant__ CUtensorMap tmx,
                                                               const __grid_constant__ CUtensorMap tmk,
                                                               const LevelParams L, const double* __restrict__ b,
                                                               double* __restrict__ r, NormSink S, int MH) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(128) double sm[];
    double* xr = sm;
    double* kr = xr + RM_XR * RM_ROW;   // HET: [RM_XR][2][RM_W]
    uint64_t* bars = reinterpret_cast<uint64_t*>(kr + (HET ? RM_XR * RM_KROW : 0));
    if (*L.stop) return;
    const int n = L.n;
    const int i0 = blockIdx.x * RM_T, j0 = blockIdx.y * MH;
    const int rows = min(MH, n + 1 - j0);
    const int nsteps = (rows + RM_R - 1) / RM_R;
    const int t = threadIdx.x;
    auto sx = [&](int y) { return (y - j0 + 2 * RM_R) % RM_XR; };
    // group g: x rows j0+gR+1 .. j0+gR+4 (g = 0: j0-1 .. j0+4)
    auto issue = [&](int g) {
        if (g >= nsteps) return;
        uint64_t* bar = &bars[g & 1];
        const int nx = g == 0 ? RM_R + 2 : RM_R;
        const int first = g == 0 ? j0 - 1 : j0 + g * RM_R + 1;
        const int nk = HET ? (g == 0 ? RM_R + 1 : RM_R) : 0;
        const int kfirst = g == 0 ? j0 - 1 : j0 + g * RM_R;
        mbar_expect_tx(bar, (nx * RM_ROW + nk * RM_KROW) * 8);
#pragma unroll 1
        for (int k = 0; k < nx; ++k) tma_load3(xr + sx(first + k) * RM_ROW, &tmx, i0 - 2, first + k, 0, bar);
#pragma unroll 1
        for (int k = 0; k < nk; ++k) tma_load3(kr + sx(kfirst + k) * RM_KROW, &tmk, i0 - 2, kfirst + k, 0, bar);
    };
    if (t == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (t == 0) {
        issue(0);
        issue(1);
    }
    double nrm = 0.0;
    const int q = t >> 5, lane = t & 31;
    for (int s = 0; s < nsteps; ++s) {
        mbar_wait(&bars[s & 1], (s >> 1) & 1);
        const int y = j0 + s * RM_R + q, i = i0 - 2 + lane;
        if (lane >= 2 && lane < RM_T + 2 && i <= n && y < j0 + rows) {
            const double* x0 = xr + sx(y) * RM_ROW + lane;
            double av[10];
            if (HET) apply_rows_kr<RM_W, RM_W>(L, xr + sx(y - 1) * RM_ROW + lane, x0, xr + sx(y + 1) * RM_ROW + lane,
                                               kr + sx(y - 1) * RM_KROW + lane, kr + sx(y) * RM_KROW + lane, av);
            else apply_rows<RM_W, false>(L, xr + sx(y - 1) * RM_ROW + lane, x0, xr + sx(y + 1) * RM_ROW + lane, i, y, av);
            const unsigned am = active_mask(i, y, n);
            const int64_t o = (int64_t)y * L.pitch + i;
#pragma unroll
            for (int k = 0; k < 10; ++k) {
                double v;
                if (MODE == 1) v = (am >> k) & 1u ? av[k] : 0.0;
                else v = (am >> k) & 1u ? __ldg(b + k * L.plane + o) - av[k] : 0.0;
                if (MODE != 2) r[k * L.plane + o] = v;
                nrm = fma(v, v, nrm);
            }
        }
        __syncthreads();
        if (t == 0) issue(s + 2);   // the rows group s + 2 replaces were last read by this step
    }
    if (S.out || S.state) norm_finish<RM_NT>(S, nrm);
}

// Rows marched by one CTA.  All CTAs of a marching launch carry equal work, so the number of row
// segments per strip is chosen to make the launch an (almost) whole number of waves of resident
// CTAs (SMs x CTAs per SM), with segments of about `target` rows: a fractional last wave left ~35% of
// the SM time idle at level 1 (profiles/r01_ncu_level1.txt); a single lock-step wave (all CTAs
// loading, then all computing) halved the throughput at level 0, so several waves are kept.
static int g_sms = 0;
static int sm_count() {
    if (!g_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || g_sms <= 0) g_sms = 148;
    }
    return g_sms;
}
// segment target of the marching relaxations: ~n/64 rows, at least 32; 16 below n = 2048 (more, shorter
// marches against the wave tail of the 2-3 wave grids there; MG_MARCH_SMALL overrides)
static int relax_target(int n) {
    static int small = -1;
    if (small < 0) {
        const char* v = getenv("MG_MARCH_SMALL");
        small = v ? atoi(v) : 16;
    }
    return n >= 2048 ? std::max(32, n / 64) : small;
}

static int march_height(int n, int tcols, int rstep, int ctas_per_sm, int target = 128) {
    if (const char* v = getenv("MG_MARCH_TARGET")) target = atoi(v);
    const long strips = (n + tcols) / tcols;
    const long slots = (long)sm_count() * ctas_per_sm;
    const long base = (n + target) / target;                            // segments of ~target rows
    const long waves = std::max(2L, (strips * base + slots / 2) / slots);
    const long segs = std::max(1L, waves * slots / strips);
    int mh = (int)((n + segs) / segs);                                   // ceil((n + 1) / segs)
    mh = ((mh + rstep - 1) / rstep) * rstep;
    return std::max(mh, rstep);
}

// ---- TMA descriptors (driver entry point fetched once through the runtime)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn g_encode = nullptr;

static int g_resid_march_n = 512;   // residual / apply on levels with n >= this: marching kernel (MG_RESID_MARCH_N)
void set_resid_march_n(int n) { g_resid_march_n = n; }
static int g_prol_ws = 0;   // fused-prolongation sweep: 1 warp-specialised (4 producer warps, setmaxnreg; measured: ptxas keeps the 80-register launch cap), 0 the 6-warp kernel (default)
void set_prol_ws(int on) { g_prol_ws = on; }
static int g_pdl = 0;   // programmatic dependent launch (MG_PDL=1; measured no gain on the cycle graph)
void set_pdl(int on) { g_pdl = on; }

template <typename... KArgs, typename... Args>
static cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = g_pdl;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

static cudaError_t encode_vec_map(CUtensorMap* m, const double* ptr, int n, int pitch, int64_t plane, int boxw,
                                  int boxh, int planes = 10) {
    if (!g_encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || !fn) return e != cudaSuccess ? e : cudaErrorNotSupported;
        g_encode = reinterpret_cast<EncodeTiledFn>(fn);
    }
    cuuint64_t dims[3] = {(cuuint64_t)(n + 1), (cuuint64_t)(n + 1), (cuuint64_t)planes};
    cuuint64_t strides[2] = {(cuuint64_t)pitch * 8, (cuuint64_t)plane * 8};
    cuuint32_t box[3] = {(cuuint32_t)boxw, (cuuint32_t)boxh, (cuuint32_t)planes};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(ptr), dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

static void carve_all();
void set_carveout(int pct) { g_carveout = pct; }
void kernels_init() {
    carve_all();
    {
        int ld[2][9][3];
        for (int sh = 0; sh < 2; ++sh)
            for (int q = 0; q < 9; ++q)
                for (int k = 0; k < 3; ++k) ld[sh][q][k] = LOCAL_DOF[sh][q][k];
        cudaMemcpyToSymbol(c_local_dof, ld, sizeof(ld));
    }
    set_smem(bottom_kernel, BOT_SMEM);
    set_smem(vanka_march2_kernel<false, 0>, M2SMEM);
    set_smem(vanka_march2_kernel<true, 0>, M2SMEM);
    set_smem(vanka_march2_kernel<false, 1>, M2SMEM);
    set_smem(vanka_march2_kernel<false, 2>, M2SMEM);
    set_smem(vanka_march2_kernel<false, 3>, M2SMEM);
    set_smem(vanka_warp_kernel<false, false, true>, WGeom<false>::SMEM);
    set_smem(vanka_warp_kernel<false, true, true>, WGeom<true>::SMEM);
    set_smem(vanka_warp_kernel<true, false, true>, WGeom<false>::SMEM);
    set_smem(vanka_warp_kernel<false, false, false>, WGeom<false>::SMEM);
    set_smem(vanka_warp_kernel<false, true, false>, WGeom<true>::SMEM);
    set_smem(vanka_warp_kernel<true, false, false>, WGeom<false>::SMEM);
    set_smem(vanka_hwarp_kernel<false>, HW_SMEM);
    set_smem(vanka_hwarp_kernel<true>, HW_SMEM);
    carve(vanka_bnd2_kernel<false, false, true>);
    carve(vanka_bnd2_kernel<true, false, true>);
    set_smem(vanka_bnd_kernel<false, false, true>, WB_SMEM);
    set_smem(vanka_bnd_kernel<true, false, true>, WB_SMEM);
    set_smem(bsr_b_warp_kernel<false, false>, WQGeom<false>::SMEM);
    set_smem(bsr_b_warp_kernel<false, true>, WQGeom<false>::SMEM);
    set_smem(bsr_b_warp_kernel<true, false>, WQGeom<true>::SMEM);
    set_smem(bsr_b_warp_kernel<true, true>, WQGeom<true>::SMEM);
    set_smem(vanka_bnd_kernel<false, false>, WB_SMEM);
    carve(vanka_bnd2_kernel<false, false>);
    carve(vanka_bnd2_kernel<false, true>);
    carve(vanka_bnd2_kernel<true, false>);
    set_smem(vanka_bnd_kernel<false, true>, WB_SMEM);
    set_smem(vanka_bnd_kernel<true, false>, WB_SMEM);
    set_smem(bsr_a_march_kernel<false, false>, BMA_SMEM);
    set_smem(bsr_a_march_kernel<false, true>, BMA_SMEM);
    set_smem(bsr_a_march_kernel<true, false>, BMA_SMEM);
    set_smem(bsr_a_march_kernel<true, true>, BMA_SMEM);
    set_smem(bsr_b_march_kernel<false, 0>, BB2_SMEM);
    set_smem(bsr_b_march_kernel<false, 1>, BB2_SMEM_NX);
    set_smem(bsr_b_march_kernel<false, 2>, BB2_SMEM_NX);
    set_smem(bsr_b_march_kernel<true, 0>, BB2_SMEM);
    set_smem(bsr_b_march_kernel<true, 1>, BB2_SMEM_NX);
    set_smem(bsr_b_march_kernel<true, 2>, BB2_SMEM_NX);
    set_smem(restrict_march_kernel<false>, Q_SMEM);
    set_smem(restrict_march_kernel<true>, Q_SMEM_K);
    set_smem(vanka_kernel<false>, V_SMEM);
    set_smem(vanka_kernel<true>, V_SMEM);
    set_smem(vanka_kernel<false, VSX, VSY>, VTile<VSX, VSY>::SMEM);
    set_smem(vanka_small_kernel<false>, VSmall::SMEM);
    set_smem(vanka_small_kernel<false, true>, VSmall::SMEM_P);
    set_smem(vanka_small4_kernel<false>, VSmall::SMEM);
    set_smem(vanka_small4_kernel<true>, VSmall::SMEM);
    set_smem(vanka_small4_kernel<false, true>, VSmall::SMEM_P);
    set_smem(vanka_small_kernel<true>, VSmall::SMEM);
    set_smem(vanka_kernel<true, VSX, VSY>, VTile<VSX, VSY>::SMEM);
    set_smem(vanka_het_kernel<false>, V_SMEM);
    set_smem(vanka_het_kernel<true>, V_SMEM);
    set_smem(vanka_het_kernel<false, VSX, VSY>, VTile<VSX, VSY>::SMEM);
    set_smem(vanka_het_kernel<true, VSX, VSY>, VTile<VSX, VSY>::SMEM);
    set_smem(restrict_kernel<0, false>, C_SMEM_PLAIN);
    set_smem(restrict_kernel<2, false>, C_SMEM_PLAIN);
    set_smem(restrict_kernel<1, false>, C_SMEM_FUSED);
    set_smem(restrict_kernel<1, true>, C_SMEM_FUSED);
    set_smem(restrict_kernel<1, false, CSX, CSY>, CTile<CSX, CSY>::SMEM_FUSED);
    set_smem(restrict_kernel<1, true, CSX, CSY>, CTile<CSX, CSY>::SMEM_FUSED);
    set_smem(restrict_small_kernel<false>, CTile<CSX, CSY>::SMEM_FUSED);
    set_smem(restrict_small_kernel<true>, CTile<CSX, CSY>::SMEM_FUSED);
    set_smem(coarse_kernel, 4096 * 8);
    set_smem(coarse_smem_kernel, (((CS_MAXN * CS_MAXN + 1) & ~1) + CS_MAXN) * 8);
    set_smem(bsr_a_kernel<false, false>, BA_SMEM);
    set_smem(bsr_a_kernel<false, true>, BA_SMEM);
    set_smem(bsr_a_kernel<true, false>, BA_SMEM);
    set_smem(bsr_a_kernel<true, true>, BA_SMEM);
    set_smem(bsr_b_kernel<false, false>, BB_SMEM);
    set_smem(bsr_b_kernel<false, true>, BB_SMEM);
    set_smem(bsr_b_kernel<true, false>, BB_SMEM);
    set_smem(bsr_b_kernel<true, true>, BB_SMEM);
}

static_assert(VNT >= V_RW * V_RH && VNT % 32 == 0, "one residual position per thread");
static_assert(CNT >= C_RW * C_RH && CNT >= 5 * CX * CY && CNT % 32 == 0, "restrict thread mapping");
static_assert(BANT >= BA_RW * BA_RH && BANT % 32 == 0, "bsr_a thread mapping");
static_assert(BBNT >= BB_RW * BB_RH && BBNT % 32 == 0, "bsr_b thread mapping");

int blocks_residual(int n) { return ((n + RTX) / RTX) * ((n + RTY) / RTY); }
int g_small_tile_n = 128;
int g_small_diet = 2;   // small-tile sweeps: 2 vanka_small4_kernel (4 threads per position), 1 vanka_small_kernel (all global
                        // reads in one round trip), 0 vanka_kernel + prolong_kernel (MG_SMALL_DIET)
void set_small_diet(int on) { g_small_diet = on; }
int small_tile_n() { return g_small_tile_n; }
int small_diet() { return g_small_diet; }   // levels with n <= this use the small 2-D tiles (mg_setup: MG_SMALL_TILE_N)
void set_small_tile_n(int n) { g_small_tile_n = n; }
int blocks_vanka(int n) {
    return n <= g_small_tile_n ? ((n + VSX) / VSX) * ((n + VSY) / VSY) : ((n + VTX) / VTX) * ((n + VTY) / VTY);
}
int blocks_bsr(int n) {
    return n <= g_small_tile_n ? ((n + VSX) / VSX) * ((n + VSY) / VSY) : ((n + BTX) / BTX) * ((n + BTY) / BTY);
}

static cudaError_t launch_residual_march(int mode, const LevelParams& L, const double* x, const double* b, double* r,
                                         NormSink S, cudaStream_t s) {
    CUtensorMap mx, mk;
    cudaError_t e = encode_vec_map(&mx, x, L.n, L.pitch, L.plane, RM_W, 1);
    if (e != cudaSuccess) return e;
    const bool het = L.kinv_field != nullptr;
    e = encode_vec_map(&mk, het ? L.kinv_field : x, L.n, L.pitch, L.plane, RM_W, 1, 2);
    if (e != cudaSuccess) return e;
    const int MH = march_height(L.n, RM_T, RM_R, 6, 64);
    dim3 grid((L.n + RM_T) / RM_T, (L.n + MH) / MH);
    if (het) {
        if (mode == 0) launch_k(residual_march_kernel<0, true>, grid, RM_NT, RM_SMEM_K, s, mx, mk, L, b, r, S, MH);
        else if (mode == 1) launch_k(residual_march_kernel<1, true>, grid, RM_NT, RM_SMEM_K, s, mx, mk, L, b, r, S, MH);
        else launch_k(residual_march_kernel<2, true>, grid, RM_NT, RM_SMEM_K, s, mx, mk, L, b, r, S, MH);
    } else if (mode == 0) launch_k(residual_march_kernel<0>, grid, RM_NT, RM_SMEM, s, mx, mk, L, b, r, S, MH);
    else if (mode == 1) launch_k(residual_march_kernel<1>, grid, RM_NT, RM_SMEM, s, mx, mk, L, b, r, S, MH);
    else launch_k(residual_march_kernel<2>, grid, RM_NT, RM_SMEM, s, mx, mk, L, b, r, S, MH);
    return cudaGetLastError();
}
int blocks_residual_march(int n) {
    const int MH = march_height(n, RM_T, RM_R, 6, 64);
    return ((n + RM_T) / RM_T) * ((n + MH) / MH);
}

cudaError_t launch_residual(const LevelParams& L, const double* x, const double* b, double* r, NormSink S,
                            cudaStream_t s) {
    if (L.lamx == 0.0 && L.n >= g_resid_march_n) return launch_residual_march(r ? 0 : 2, L, x, b, r, S, s);
    dim3 grid((L.n + RTX) / RTX, (L.n + RTY) / RTY);
    if (L.kinv_field) launch_k(residual_kernel<true, false>, grid, RNT, 0, s, L, x, b, r, S);
    else launch_k(residual_kernel<false, false>, grid, RNT, 0, s, L, x, b, r, S);
    return cudaGetLastError();
}

cudaError_t launch_apply(const LevelParams& L, const double* x, double* y, NormSink S, cudaStream_t s) {
    if (L.lamx == 0.0 && L.n >= g_resid_march_n) return launch_residual_march(1, L, x, nullptr, y, S, s);
    dim3 grid((L.n + RTX) / RTX, (L.n + RTY) / RTY);
    if (L.kinv_field) launch_k(residual_kernel<true, true>, grid, RNT, 0, s, L, x, nullptr, y, S);
    else launch_k(residual_kernel<false, true>, grid, RNT, 0, s, L, x, nullptr, y, S);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// Vector kernels of FGMRES over whole padded level vectors (inactive / padding slots are 0).
// Deterministic: fixed grid, per-block partials, summed in block order by the last block.
constexpr int DOT_BLOCKS = 296, DOT_NT = 256, VK = 8;

__global__ void __launch_bounds__(DOT_NT) vec_dots_kernel(const double* __restrict__ w, VecPtrs V, int k,
                                                          int64_t len, double* __restrict__ partials,
                                                          unsigned* __restrict__ counter, double* __restrict__ out) {
    pdl_wait();
    pdl_trigger();
    double acc[VK];
#pragma unroll
    for (int q = 0; q < VK; ++q) acc[q] = 0.0;
    const int64_t n2 = len / 2;
    const double2* w2 = reinterpret_cast<const double2*>(w);
    for (int64_t e = (int64_t)blockIdx.x * DOT_NT + threadIdx.x; e < n2; e += (int64_t)DOT_BLOCKS * DOT_NT) {
        const double2 a = __ldg(w2 + e);
#pragma unroll
        for (int q = 0; q < VK; ++q) {
            if (q < k) {
                const double2 v = __ldg(reinterpret_cast<const double2*>(V.p[q]) + e);
                acc[q] = fma(a.x, v.x, acc[q]);
                acc[q] = fma(a.y, v.y, acc[q]);
            }
        }
    }
    __shared__ double red[VK][DOT_NT / 32];
    __shared__ unsigned last;
#pragma unroll
    for (int q = 0; q < VK; ++q) {
        double v = acc[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0) red[q][threadIdx.x >> 5] = v;
    }
    __syncthreads();
    if (threadIdx.x < k) {
        double t = 0.0;
        for (int u = 0; u < DOT_NT / 32; ++u) t += red[threadIdx.x][u];
        partials[threadIdx.x * DOT_BLOCKS + blockIdx.x] = t;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(counter, 1u) == DOT_BLOCKS - 1);
    __syncthreads();
    if (last) {
        __threadfence();
        if (threadIdx.x < k) {
            double t = 0.0;
            for (int u = 0; u < DOT_BLOCKS; ++u) t += __ldcg(partials + threadIdx.x * DOT_BLOCKS + u);
            out[threadIdx.x] = t;
        }
        if (threadIdx.x == 0) *counter = 0u;
    }
}

// w = w - sum_q c[q] v_q   (c in device memory)
__global__ void __launch_bounds__(DOT_NT) vec_update_kernel(double* __restrict__ w, VecPtrs V, int k,
                                                            const double* __restrict__ c, int64_t len) {
    pdl_wait();
    pdl_trigger();
    const int64_t n2 = len / 2;
    double2* w2 = reinterpret_cast<double2*>(w);
    double cq[VK];
#pragma unroll
    for (int q = 0; q < VK; ++q) cq[q] = q < k ? c[q] : 0.0;
    for (int64_t e = (int64_t)blockIdx.x * DOT_NT + threadIdx.x; e < n2; e += (int64_t)gridDim.x * DOT_NT) {
        double2 a = w2[e];
#pragma unroll
        for (int q = 0; q < VK; ++q) {
            if (q < k) {
                const double2 v = __ldg(reinterpret_cast<const double2*>(V.p[q]) + e);
                a.x = fma(-cq[q], v.x, a.x);
                a.y = fma(-cq[q], v.y, a.y);
            }
        }
        w2[e] = a;
    }
}

// dst = src over a whole padded vector (len doubles, 16-B aligned), skipped when the solve's stop
// flag is raised: the level-0 copy-back of an odd sweep count must not run in the cycle that
// stops mg_solve (its pre-sweep already wrote the scratch vector past the recorded iterate)
__global__ void __launch_bounds__(DOT_NT) vec_copy_kernel(double* __restrict__ dst, const double* __restrict__ src,
                                                          int64_t len, const int* __restrict__ stop) {
    pdl_wait();
    pdl_trigger();
    if (*stop) return;
    const int64_t n2 = len / 2;
    for (int64_t e = (int64_t)blockIdx.x * DOT_NT + threadIdx.x; e < n2; e += (int64_t)gridDim.x * DOT_NT)
        reinterpret_cast<double2*>(dst)[e] = __ldg(reinterpret_cast<const double2*>(src) + e);
    if ((len & 1) && blockIdx.x == 0 && threadIdx.x == 0) dst[len - 1] = src[len - 1];
}

// y = s * x
__global__ void __launch_bounds__(DOT_NT) vec_scale_kernel(double* __restrict__ y, const double* __restrict__ x,
                                                           double s, int64_t len) {
    pdl_wait();
    pdl_trigger();
    const int64_t n2 = len / 2;
    for (int64_t e = (int64_t)blockIdx.x * DOT_NT + threadIdx.x; e < n2; e += (int64_t)gridDim.x * DOT_NT) {
        double2 a = __ldg(reinterpret_cast<const double2*>(x) + e);
        a.x *= s;
        a.y *= s;
        reinterpret_cast<double2*>(y)[e] = a;
    }
}

// fused Gram-Schmidt pass (see mg_kernels.cuh): KB >= k basis vectors (register accumulators sized
// to the bucket, so short bases keep occupancy high), two double2 element pairs per thread and step
// for memory-level parallelism
constexpr int GS_BLOCKS = 592, GS_NT = 256;
template <int MODE, int KB>
__global__ void __launch_bounds__(GS_NT) vec_gs_kernel(const double* __restrict__ w, double* wo, GsPtrs V, int k,
                                                       const double* __restrict__ c, const double* __restrict__ sc,
                                                       int64_t len, double* __restrict__ partials,
                                                       unsigned* __restrict__ counter, double* __restrict__ out) {
    pdl_wait();
    pdl_trigger();
    constexpr int NA = MODE == 0 || MODE == 1 ? KB + 1 : (MODE == 2 ? 1 : 0);
    double acc[NA > 0 ? NA : 1];
#pragma unroll
    for (int q = 0; q < (NA > 0 ? NA : 1); ++q) acc[q] = 0.0;
    __shared__ double cq[KB];   // update coefficients (broadcast reads)
    if (threadIdx.x < KB)
        cq[threadIdx.x] = (MODE != 0 && (int)threadIdx.x < k) ? c[threadIdx.x] * (sc ? sc[threadIdx.x] : 1.0) : 0.0;
    __syncthreads();
    const int64_t n2 = len / 2;
    const int64_t stride = (int64_t)gridDim.x * GS_NT;
    const double2* w2 = reinterpret_cast<const double2*>(w);
    if (MODE == 1 && KB <= 16) {
        // one element pair per thread and step with the k basis pairs held in registers: the update
        // and the dots of the updated pair read the basis once (re-reading it through L2 halved the
        // pass's bandwidth at k = 9-16)
        for (int64_t e0 = (int64_t)blockIdx.x * GS_NT + threadIdx.x; e0 < n2; e0 += stride) {
            double2 a0 = w2[e0];
            double2 vv[KB];
#pragma unroll
            for (int q = 0; q < KB; ++q)
                vv[q] = q < k ? __ldg(reinterpret_cast<const double2*>(V.p[q]) + e0) : make_double2(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < KB; ++q)
                if (q < k) {
                    a0.x = fma(-cq[q], vv[q].x, a0.x);
                    a0.y = fma(-cq[q], vv[q].y, a0.y);
                }
            reinterpret_cast<double2*>(wo)[e0] = a0;
#pragma unroll
            for (int q = 0; q < KB; ++q)
                if (q < k) {
                    acc[q] = fma(a0.x, vv[q].x, acc[q]);
                    acc[q] = fma(a0.y, vv[q].y, acc[q]);
                }
            acc[NA - 1] = fma(a0.x, a0.x, acc[NA - 1]);
            acc[NA - 1] = fma(a0.y, a0.y, acc[NA - 1]);
        }
    } else
    for (int64_t e0 = (int64_t)blockIdx.x * GS_NT + threadIdx.x; e0 < n2; e0 += 2 * stride) {
        const int64_t e1 = e0 + stride;
        const bool has1 = e1 < n2;
        double2 a0 = w2[e0], a1 = has1 ? w2[e1] : make_double2(0.0, 0.0);
        if (MODE == 0) {
#pragma unroll
            for (int q = 0; q < KB; ++q)
                if (q < k) {
                    const double2* vp = reinterpret_cast<const double2*>(V.p[q]);
                    const double2 v0 = __ldg(vp + e0), v1 = has1 ? __ldg(vp + e1) : make_double2(0.0, 0.0);
                    acc[q] = fma(a0.x, v0.x, acc[q]);
                    acc[q] = fma(a0.y, v0.y, acc[q]);
                    acc[q] = fma(a1.x, v1.x, acc[q]);
                    acc[q] = fma(a1.y, v1.y, acc[q]);
                }
        } else {
            // loads in groups of 4 vectors ahead of their FMAs (keeps 8 loads in flight per thread)
#pragma unroll
            for (int q0 = 0; q0 < KB; q0 += 4) {
                double2 v0[4], v1[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int q = q0 + u;
                    const double2* vp = reinterpret_cast<const double2*>(V.p[q]);
                    v0[u] = q < k ? __ldg(vp + e0) : make_double2(0.0, 0.0);
                    v1[u] = (q < k && has1) ? __ldg(vp + e1) : make_double2(0.0, 0.0);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int q = q0 + u;
                    if (q < k) {
                        a0.x = fma(-cq[q], v0[u].x, a0.x);
                        a0.y = fma(-cq[q], v0[u].y, a0.y);
                        a1.x = fma(-cq[q], v1[u].x, a1.x);
                        a1.y = fma(-cq[q], v1[u].y, a1.y);
                    }
                }
            }
            reinterpret_cast<double2*>(wo)[e0] = a0;
            if (has1) reinterpret_cast<double2*>(wo)[e1] = a1;
            if (MODE == 1) {
                // dots of the updated pairs with the basis (re-read: an L1 / L2 hit)
#pragma unroll
                for (int q = 0; q < KB; ++q)
                    if (q < k) {
                        const double2* vp = reinterpret_cast<const double2*>(V.p[q]);
                        const double2 v0 = __ldg(vp + e0), v1 = has1 ? __ldg(vp + e1) : make_double2(0.0, 0.0);
                        acc[q] = fma(a0.x, v0.x, acc[q]);
                        acc[q] = fma(a0.y, v0.y, acc[q]);
                        acc[q] = fma(a1.x, v1.x, acc[q]);
                        acc[q] = fma(a1.y, v1.y, acc[q]);
                    }
            }
        }
        if (MODE != 3) {
            acc[NA - 1] = fma(a0.x, a0.x, acc[NA - 1]);
            acc[NA - 1] = fma(a0.y, a0.y, acc[NA - 1]);
            acc[NA - 1] = fma(a1.x, a1.x, acc[NA - 1]);
            acc[NA - 1] = fma(a1.y, a1.y, acc[NA - 1]);
        }
    }
    if (NA == 0) return;
    __shared__ double red[NA > 0 ? NA : 1][GS_NT / 32];
    __shared__ unsigned last;
#pragma unroll
    for (int q = 0; q < (NA > 0 ? NA : 1); ++q) {
        double v = acc[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0) red[q][threadIdx.x >> 5] = v;
    }
    __syncthreads();
    const int nres = MODE == 2 ? 1 : k + 1;   // results: dots 0..k-1, norm at slot k (mode 2: slot 0)
    auto slot = [&](int r) { return MODE == 2 ? 0 : (r < k ? r : NA - 1); };
    for (int r = threadIdx.x; r < nres; r += GS_NT) {
        double t = 0.0;
        for (int u = 0; u < GS_NT / 32; ++u) t += red[slot(r)][u];
        partials[r * GS_BLOCKS + blockIdx.x] = t;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (last) {
        __threadfence();
        for (int r = threadIdx.x; r < nres; r += GS_NT) {
            double t = 0.0;
            for (int u = 0; u < (int)gridDim.x; ++u) t += __ldcg(partials + r * GS_BLOCKS + u);
            out[r] = t;
        }
        if (threadIdx.x == 0) *counter = 0u;
    }
}

// grid of a Gram-Schmidt pass: one wave of resident CTAs (the register-heavy buckets fit 2-3 CTAs per
// SM: a fixed 4 x 148 grid ran them in two partial waves at 3.6 TB/s), at most GS_BLOCKS
template <typename F>
static int gs_blocks(F* f) {
    int per = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, f, GS_NT, 0) != cudaSuccess || per <= 0) per = 1;
    return std::min(GS_BLOCKS, per * sm_count());
}
template <int KB>
static void launch_gs_kb(int mode, const double* w, double* wo, const GsPtrs& V, int k, const double* c,
                         const double* sc, int64_t len, double* partials, unsigned* counter, double* out, cudaStream_t s) {
    static const int nb[4] = {gs_blocks(vec_gs_kernel<0, KB>), gs_blocks(vec_gs_kernel<1, KB>),
                              gs_blocks(vec_gs_kernel<2, KB>), gs_blocks(vec_gs_kernel<3, KB>)};
    switch (mode) {
        case 0: launch_k(vec_gs_kernel<0, KB>, nb[0], GS_NT, 0, s, w, wo, V, k, c, sc, len, partials, counter, out); break;
        case 1: launch_k(vec_gs_kernel<1, KB>, nb[1], GS_NT, 0, s, w, wo, V, k, c, sc, len, partials, counter, out); break;
        case 2: launch_k(vec_gs_kernel<2, KB>, nb[2], GS_NT, 0, s, w, wo, V, k, c, sc, len, partials, counter, out); break;
        default: launch_k(vec_gs_kernel<3, KB>, nb[3], GS_NT, 0, s, w, wo, V, k, c, sc, len, partials, counter, out); break;
    }
}

cudaError_t launch_gs(int mode, const double* w, double* wo, const GsPtrs& V, int k, const double* c,
                      const double* sc, int64_t len, double* partials, unsigned* counter, double* out, cudaStream_t s) {
    if (k < 0 || k > GS_KMAX) return cudaErrorInvalidValue;
    if (k <= 4) launch_gs_kb<4>(mode, w, wo, V, k, c, sc, len, partials, counter, out, s);
    else if (k <= 8) launch_gs_kb<8>(mode, w, wo, V, k, c, sc, len, partials, counter, out, s);
    else if (k <= 16) launch_gs_kb<16>(mode, w, wo, V, k, c, sc, len, partials, counter, out, s);
    else launch_gs_kb<GS_KMAX>(mode, w, wo, V, k, c, sc, len, partials, counter, out, s);
    return cudaGetLastError();
}
int gs_partials_needed() { return (GS_KMAX + 1) * GS_BLOCKS; }

cudaError_t launch_dots(const double* w, const VecPtrs& V, int k, int64_t len, double* partials, unsigned* counter,
                        double* out, cudaStream_t s) {
    launch_k(vec_dots_kernel, DOT_BLOCKS, DOT_NT, 0, s, w, V, k, len, partials, counter, out);
    return cudaGetLastError();
}
cudaError_t launch_update(double* w, const VecPtrs& V, int k, const double* c, int64_t len, cudaStream_t s) {
    launch_k(vec_update_kernel, 2 * DOT_BLOCKS, DOT_NT, 0, s, w, V, k, c, len);
    return cudaGetLastError();
}
cudaError_t launch_scale(double* y, const double* x, double sc, int64_t len, cudaStream_t s) {
    launch_k(vec_scale_kernel, 2 * DOT_BLOCKS, DOT_NT, 0, s, y, x, sc, len);
    return cudaGetLastError();
}
// ------------------------------------------------------------------------------------------
// Exact BSR: S dp = g solved by Jacobi-preconditioned conjugate gradients on the
// two P0 planes, S = s0 M_p + tau B_w D_w^{-1} B_w^T applied from the per-level Jacobi table (tau / D_w
// per RT0 edge, 1 / diag S per triangle).  Two kernels per iteration with every scalar on the device
// (graph-capturable; each kernel returns at entry once the iteration has converged):
//   cg_a: p = z + beta p, q = S z + beta q (= S p), partial sums of p.q -> alpha = rz / pq
//   cg_b: dp += alpha p, r -= alpha q, z = r / diag S, partial sums of r.z -> beta, convergence
// CgState: [0] rz, [1] alpha, [2] beta, [3] rz0, [4] tol^2, [5] converged flag (as double), [6] its
constexpr int CG_NT = 256;
__device__ __forceinline__ double s_offdiag(const LevelParams& L, const double* __restrict__ tab,
                                            const double* __restrict__ v, int sh, int i, int j) {
    const int64_t plane = L.plane, pitch = L.pitch, o = (int64_t)j * pitch + i;
    const double te[3] = {sh == 0 ? __ldg(tab + o) : __ldg(tab + o + pitch),
                          sh == 0 ? __ldg(tab + plane + o) : __ldg(tab + plane + o + 1), __ldg(tab + 2 * plane + o)};
    double off = 0.0;
#pragma unroll
    for (int e = 0; e < 3; ++e) {
        int ni, nj;
        if (sh == 0) { ni = e == 1 ? i - 1 : i; nj = e == 0 ? j - 1 : j; }
        else         { ni = e == 1 ? i + 1 : i; nj = e == 0 ? j + 1 : j; }
        if (te[e] != 0.0) off = fma(te[e] * L.bw[sh][e] * L.bw[1 - sh][e], __ldg(v + (1 - sh) * plane + (int64_t)nj * pitch + ni), off);
    }
    return off;
}

// deterministic block sum + last-block finish (partials / counter private to the CG)
template <int MODE>
__device__ void cg_finish(double v, double* partials, unsigned* counter, double* st) {
    const int nb = gridDim.x * gridDim.y, bid = blockIdx.y * gridDim.x + blockIdx.x;
    const double t = block_sum<CG_NT>(v);
    __shared__ unsigned last;
    if (threadIdx.x == 0) {
        partials[bid] = t;
        __threadfence();
        last = atomicAdd(counter, 1u) == (unsigned)nb - 1u;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double acc = 0.0;
    for (int k = threadIdx.x; k < nb; k += CG_NT) acc += __ldcg(partials + k);
    const double tot = block_sum<CG_NT>(acc);
    if (threadIdx.x == 0) {
        if (MODE == 0) {          // tot = p.q
            st[1] = tot > 0.0 ? st[0] / tot : 0.0;
        } else if (MODE == 1) {   // tot = r.z (new)
            st[2] = st[0] > 0.0 ? tot / st[0] : 0.0;
            st[0] = tot;
            st[6] += 1.0;
            if (!(tot > st[4] * st[3])) st[5] = 1.0;
        } else {                  // MODE 2: initial r.z
            st[0] = tot;
            st[3] = tot;
            st[2] = 0.0;
            st[6] = 0.0;
            st[5] = tot > 0.0 ? 0.0 : 1.0;
        }
        *counter = 0u;
    }
}

// init: r = g (in place), z = r / diag S, dp = 0, p = q = 0, rz = r.z
__global__ void __launch_bounds__(CG_NT) cg_init_kernel(const LevelParams L, const double* __restrict__ tab, double* r,
                                                        double* z, double* dp, double* p, double* q, double* partials,
                                                        unsigned* counter, double* st) {
    const int i = blockIdx.x * 32 + (threadIdx.x & 31), j = blockIdx.y * 8 + (threadIdx.x >> 5);
    double v = 0.0;
    if (i <= L.n && j <= L.n && !*L.stop) {
        const int64_t o = (int64_t)j * L.pitch + i;
#pragma unroll
        for (int sh = 0; sh < 2; ++sh) {
            const int64_t k = sh * L.plane + o;
            const double zz = r[k] * __ldg(tab + (3 + sh) * L.plane + o);
            z[k] = zz;
            dp[k] = 0.0;
            p[k] = 0.0;
            q[k] = 0.0;
            v = fma(r[k], zz, v);
        }
    }
    cg_finish<2>(v, partials, counter, st);
}

__global__ void __launch_bounds__(CG_NT) cg_a_kernel(const LevelParams L, const double* __restrict__ tab,
                                                     const double* __restrict__ z, double* p, double* q,
                                                     double* partials, unsigned* counter, double* st) {
    if (st[5] != 0.0 || *L.stop) return;
    const int i = blockIdx.x * 32 + (threadIdx.x & 31), j = blockIdx.y * 8 + (threadIdx.x >> 5);
    const double beta = st[2];
    double v = 0.0;
    if (i < L.n && j < L.n) {
        const int64_t o = (int64_t)j * L.pitch + i;
#pragma unroll
        for (int sh = 0; sh < 2; ++sh) {
            const int64_t k = sh * L.plane + o;
            const double zk = z[k];
            const double sz = fma(zk, 1.0 / __ldg(tab + (3 + sh) * L.plane + o), s_offdiag(L, tab, z, sh, i, j));
            const double pk = fma(beta, p[k], zk), qk = fma(beta, q[k], sz);
            p[k] = pk;
            q[k] = qk;
            v = fma(pk, qk, v);
        }
    }
    cg_finish<0>(v, partials, counter, st);
}

__global__ void __launch_bounds__(CG_NT) cg_b_kernel(const LevelParams L, const double* __restrict__ tab,
                                                     const double* __restrict__ p, const double* __restrict__ q,
                                                     double* r, double* z, double* dp, double* partials,
                                                     unsigned* counter, double* st) {
    if (st[5] != 0.0 || *L.stop) return;
    const int i = blockIdx.x * 32 + (threadIdx.x & 31), j = blockIdx.y * 8 + (threadIdx.x >> 5);
    const double alpha = st[1];
    double v = 0.0;
    if (i < L.n && j < L.n) {
        const int64_t o = (int64_t)j * L.pitch + i;
#pragma unroll
        for (int sh = 0; sh < 2; ++sh) {
            const int64_t k = sh * L.plane + o;
            dp[k] = fma(alpha, p[k], dp[k]);
            const double rk = fma(-alpha, q[k], r[k]);
            r[k] = rk;
            const double zk = rk * __ldg(tab + (3 + sh) * L.plane + o);
            z[k] = zk;
            v = fma(rk, zk, v);
        }
    }
    cg_finish<1>(v, partials, counter, st);
}

cudaError_t launch_cg_exact(const LevelParams& L, const double* tab, double* g, double* dp, double* z, double* p,
                            double* q, double* partials, unsigned* counter, double* st, int max_iters,
                            cudaStream_t s) {
    dim3 grid((L.n + 32) / 32, (L.n + 8) / 8);
    cg_init_kernel<<<grid, CG_NT, 0, s>>>(L, tab, g, z, dp, p, q, partials, counter, st);
    for (int it = 0; it < max_iters; ++it) {
        cg_a_kernel<<<grid, CG_NT, 0, s>>>(L, tab, z, p, q, partials, counter, st);
        cg_b_kernel<<<grid, CG_NT, 0, s>>>(L, tab, p, q, g, z, dp, partials, counter, st);
    }
    return cudaGetLastError();
}
int cg_partials_needed(int n) { return ((n + 32) / 32) * ((n + 8) / 8); }

// Backward-Euler history term (eq. discrete3 scaled by -1): the pressure rows of
// b^m get -(1/M) M_p p^{m-1} + alpha B_u u^{m-1}, B_u u = -(div u, 1_T) of the 9 displacement DoFs
// of triangle T (L.bu = h REF_BU in LOCAL_DOF order), M_p = h^2/2.  One thread per cell.
__global__ void __launch_bounds__(256) step_rhs_kernel(const LevelParams L, double inv_M, double alpha,
                                                       const double* __restrict__ x, double* __restrict__ b) {
    const int i = blockIdx.x * 32 + (threadIdx.x & 31), j = blockIdx.y * 8 + (threadIdx.x >> 5);
    const int n = L.n;
    if (i >= n || j >= n) return;
    const double h = 1.0 / n;
#pragma unroll
    for (int sh = 0; sh < 2; ++sh) {
        double d = 0.0;
#pragma unroll
        for (int q = 0; q < 9; ++q) {
            const int ii = i + c_local_dof[sh][q][0], jj = j + c_local_dof[sh][q][1], p = c_local_dof[sh][q][2];
            d = fma(L.bu[sh][q], x[p * L.plane + (int64_t)jj * L.pitch + ii], d);
        }
        const int64_t o = (8 + sh) * L.plane + (int64_t)j * L.pitch + i;
        b[o] += fma(-inv_M * (h * h * 0.5), x[o], alpha * d);   // M_p = |T| = h^2/2 (REF_MP)
    }
}

cudaError_t launch_step_rhs(const LevelParams& L, double inv_M, double alpha, const double* x, double* b,
                            cudaStream_t s) {
    dim3 grid((L.n + 31) / 32, (L.n + 7) / 8);
    step_rhs_kernel<<<grid, 256, 0, s>>>(L, inv_M, alpha, x, b);
    return cudaGetLastError();
}

cudaError_t launch_hv_sinv(const LevelParams& L, const double* W, const double* C, double* sinv, cudaStream_t s) {
    dim3 grid((L.n + 32) / 32, (L.n + 8) / 8);
    hv_sinv_kernel<<<grid, 256, 0, s>>>(L, W, C, sinv);
    return cudaGetLastError();
}
cudaError_t launch_copy(double* dst, const double* src, int64_t len, const int* stop, cudaStream_t s) {
    launch_k(vec_copy_kernel, 2 * DOT_BLOCKS, DOT_NT, 0, s, dst, src, len, stop);
    return cudaGetLastError();
}
int dot_partials_needed() { return VK * DOT_BLOCKS; }

cudaError_t launch_vanka(const VankaParams& P, const double* x, const double* b, double* xo, bool x_zero,
                         NormSink S, cudaStream_t s, const HvInterior* Ti, const ProlSrc* E) {
    if (E && (P.hv.cls || P.L.n > g_small_tile_n || !g_small_diet || x_zero)) return cudaErrorInvalidValue;
    if (P.hv.cls) {   // heterogeneous K: condensed patch solves, K^{-1} field in the residual
        if (!Ti) return cudaErrorInvalidValue;
        if (P.L.n <= g_small_tile_n) {
            using T = VTile<VSX, VSY>;
            dim3 grid((P.L.n + VSX) / VSX, (P.L.n + VSY) / VSY);
            if (x_zero) launch_k(vanka_het_kernel<true, VSX, VSY>, grid, T::NT, T::SMEM, s, P, *Ti, x, b, xo, S);
            else launch_k(vanka_het_kernel<false, VSX, VSY>, grid, T::NT, T::SMEM, s, P, *Ti, x, b, xo, S);
            return cudaGetLastError();
        }
        dim3 grid((P.L.n + VTX) / VTX, (P.L.n + VTY) / VTY);
        if (x_zero) launch_k(vanka_het_kernel<true>, grid, VNT, V_SMEM, s, P, *Ti, x, b, xo, S);
        else launch_k(vanka_het_kernel<false>, grid, VNT, V_SMEM, s, P, *Ti, x, b, xo, S);
        return cudaGetLastError();
    }
    if (P.L.n <= g_small_tile_n) {
        using T = VTile<VSX, VSY>;
        dim3 grid((P.L.n + VSX) / VSX, (P.L.n + VSY) / VSY);
        const ProlSrc none{nullptr, 0, 0, 0};
        if (g_small_diet == 2) {
            if (x_zero) launch_k(vanka_small4_kernel<true>, grid, VS4_NT, VSmall::SMEM, s, P, x, b, xo, S, none);
            else if (E) launch_k(vanka_small4_kernel<false, true>, grid, VS4_NT, VSmall::SMEM_P, s, P, x, b, xo, S, *E);
            else launch_k(vanka_small4_kernel<false>, grid, VS4_NT, VSmall::SMEM, s, P, x, b, xo, S, none);
        } else if (g_small_diet) {
            if (x_zero) launch_k(vanka_small_kernel<true>, grid, T::NT, VSmall::SMEM, s, P, x, b, xo, S, none);
            else if (E) launch_k(vanka_small_kernel<false, true>, grid, T::NT, VSmall::SMEM_P, s, P, x, b, xo, S, *E);
            else launch_k(vanka_small_kernel<false>, grid, T::NT, VSmall::SMEM, s, P, x, b, xo, S, none);
        } else {
            if (x_zero) launch_k(vanka_kernel<true, VSX, VSY>, grid, T::NT, T::SMEM, s, P, x, b, xo, S);
            else launch_k(vanka_kernel<false, VSX, VSY>, grid, T::NT, T::SMEM, s, P, x, b, xo, S);
        }
        return cudaGetLastError();
    }
    dim3 grid((P.L.n + VTX) / VTX, (P.L.n + VTY) / VTY);
    if (x_zero) launch_k(vanka_kernel<true>, grid, VNT, V_SMEM, s, P, x, b, xo, S);
    else launch_k(vanka_kernel<false>, grid, VNT, V_SMEM, s, P, x, b, xo, S);
    return cudaGetLastError();
}

// warp-marching sweep (vanka_warp_kernel) on levels with n >= MG_WARP_MIN_N (0: off); its tasks are
// (strip of WT columns, segment of MH rows), one per warp, sized to whole waves of the 2 x WPC warps
// per SM with segments near MG_WARP_TARGET rows
static int g_warp_min_n = 512;
static int g_warp_prol = 1;
static int g_warp_bk = 1;     // boundary-vertex patches precomputed by 1: vanka_bnd2_kernel, 2: vanka_bnd_kernel; 0: out of line in the sweep
void set_warp_bk(int on) { g_warp_bk = on; }   // the fused-prolongation post-sweep through the warp kernel too (MG_WARP_PROL)
void set_warp_prol(int on) { g_warp_prol = on; }
static void warp_tasks_nw(int n, int slots_per_sm, int& MH, int& nstrips, int& ntasks);
static void warp_tasks(int n, int& MH, int& nstrips, int& ntasks, bool prol = false) {
    warp_tasks_nw(n, 2 * (prol ? WGeom<true>::NW : WGeom<false>::NW), MH, nstrips, ntasks);
}
static int g_warp_bsr = 0;   // BSR stage B through bsr_b_warp_kernel on the warp levels (MG_WARP_BSR; measured: no gain, off)
void set_warp_bsr(int on) { g_warp_bsr = on; }
static void warp_tasks_nw(int n, int slots_per_sm, int& MH, int& nstrips, int& ntasks) {
    static int target = -1;
    if (target < 0) {
        const char* v = getenv("MG_WARP_TARGET");
        target = v ? std::max(4, atoi(v)) : 128;
    }
    nstrips = (n + WT) / WT;   // ceil((n + 1) / WT)
    const long slots = (long)sm_count() * slots_per_sm;
    const long base = (n + target) / target;
    const long waves = std::max(1L, (nstrips * base + slots / 2) / slots);
    long nseg = std::max(1L, waves * slots / nstrips);
    static int minrows = -1;   // shortest segment (MG_WARP_MINROWS): the per-task prologue and pipeline fill
    if (minrows < 0) {
        const char* v = getenv("MG_WARP_MINROWS");
        minrows = v ? std::max(4, atoi(v)) : 4;   // 8 until the warp sweeps took over the 512^2 level: config 3 0.428 -> 0.418 ms
    }
    MH = std::max(minrows, (int)((n + nseg) / nseg));
    nseg = (n + MH) / MH;
    ntasks = (int)(nstrips * nseg);
}
void set_warp_min_n(int n) { g_warp_min_n = n; }

cudaError_t launch_vanka_march2(const VankaParams& P, const double* x, const double* b, double* xo, bool x_zero,
                                NormSink S, cudaStream_t s, const ProlSrc* E) {
    const LevelParams& L = P.L;
    CUtensorMap mx, mb;
    cudaError_t e = encode_vec_map(&mx, x_zero ? b : x, L.n, L.pitch, L.plane, M2W, 1);
    if (e != cudaSuccess) return e;
    e = encode_vec_map(&mb, b, L.n, L.pitch, L.plane, M2W, 1);
    if (e != cudaSuccess) return e;
    // segments of ~max(32, n/64) rows: more, shorter marches keep CTAs of one SM out of lock step
    // (measured: 2048^2 sweep 0.45 -> 0.37 ms, 4096^2 1.24 -> 1.19 ms against ~128-row segments)
    static int prol_scale = -1;   // segment length factor of the fused-prolongation sweep (MG_PROL_SEG)
    if (prol_scale < 0) {
        const char* v = getenv("MG_PROL_SEG");
        prol_scale = v ? atoi(v) : 1;
    }
    const int MH = march_height(L.n, M2T, M2R, 3, relax_target(L.n) * (E ? prol_scale : 1));
    dim3 grid((L.n + M2T) / M2T, (L.n + MH) / MH);
    const ProlSrc none{nullptr, 0, 0, 0};
    if (E && x_zero) return cudaErrorInvalidValue;
    if (g_warp_min_n > 0 && L.n >= g_warp_min_n && (!E || g_warp_prol)) {
        const bool prol = E != nullptr;
        int wmh, nstrips, ntasks;
        warp_tasks(L.n, wmh, nstrips, ntasks, prol);
        CUtensorMap wx, wb, wc;
        e = encode_vec_map(&wx, x_zero ? b : x, L.n, L.pitch, L.plane, WXW, 1);
        if (e == cudaSuccess) e = encode_vec_map(&wb, b, L.n, L.pitch, L.plane, WBW, 1);
        if (e == cudaSuccess && prol) e = encode_vec_map(&wc, E->e, E->nc, E->pitchc, E->planec, WCC, 1);
        if (e != cudaSuccess) return e;
        const ProlSrc Ev = prol ? *E : none;
        const int nw = prol ? WGeom<true>::NW : WGeom<false>::NW;
        const dim3 wgrid((ntasks + nw - 1) / nw);
        const dim3 bgrid((bnd_count(L.n) + WB_NT - 1) / WB_NT);
        const dim3 bgrid2((L.n + WB2_T) / WB2_T, 4);
        if (g_warp_bk == 1) {
            if (x_zero) launch_k(vanka_bnd2_kernel<true, false>, bgrid2, WB2_NT, 0, s, P, x, b, Ev);
            else if (prol) launch_k(vanka_bnd2_kernel<false, true>, bgrid2, WB2_NT, 0, s, P, x, b, Ev);
            else launch_k(vanka_bnd2_kernel<false, false>, bgrid2, WB2_NT, 0, s, P, x, b, Ev);
        } else if (g_warp_bk == 2) {
            if (x_zero) launch_k(vanka_bnd_kernel<true, false>, bgrid, WB_NT, WB_SMEM, s, P, x, b, Ev);
            else if (prol) launch_k(vanka_bnd_kernel<false, true>, bgrid, WB_NT, WB_SMEM, s, P, x, b, Ev);
            else launch_k(vanka_bnd_kernel<false, false>, bgrid, WB_NT, WB_SMEM, s, P, x, b, Ev);
        }
#define WLAUNCH(Z_, P_, B_)                                                                                     \
    launch_k(vanka_warp_kernel<Z_, P_, B_>, wgrid, WGeom<P_>::NT, WGeom<P_>::SMEM, s, wx, wb, P_ ? wc : wx, P, xo, S, \
             wmh, nstrips, ntasks, Ev)
        if (g_warp_bk != 0) {
            if (x_zero) WLAUNCH(true, false, true);
            else if (prol) WLAUNCH(false, true, true);
            else WLAUNCH(false, false, true);
        } else {
            if (x_zero) WLAUNCH(true, false, false);
            else if (prol) WLAUNCH(false, true, false);
            else WLAUNCH(false, false, false);
        }
#undef WLAUNCH
        return cudaGetLastError();
    }
    if (x_zero) launch_k(vanka_march2_kernel<true, 0>, grid, M2NT, M2SMEM, s, mx, mb, P, xo, S, MH, none);
    else if (E && g_prol_ws == 1)
        launch_k(vanka_march2_kernel<false, 2>, grid, M2NT + 32 * m2np(2), M2SMEM, s, mx, mb, P, xo, S, MH, *E);
    else if (E && g_prol_ws == 3)
        launch_k(vanka_march2_kernel<false, 3>, grid, M2NT + 32 * m2np(3), M2SMEM, s, mx, mb, P, xo, S, MH, *E);
    else if (E) launch_k(vanka_march2_kernel<false, 1>, grid, M2NT + 32 * M2NP, M2SMEM, s, mx, mb, P, xo, S, MH, *E);
    else launch_k(vanka_march2_kernel<false, 0>, grid, M2NT, M2SMEM, s, mx, mb, P, xo, S, MH, none);
    return cudaGetLastError();
}
// heterogeneous-K warp-marching sweep (vanka_hwarp_kernel) + its boundary kernel
cudaError_t launch_vanka_hwarp(const VankaParams& P, const HvInterior& Ti, const double* x, const double* b, double* xo,
                               bool x_zero, NormSink S, cudaStream_t s) {
    const LevelParams& L = P.L;
    if (!P.hv.cls || !L.kinv_field) return cudaErrorInvalidValue;
    int wmh, nstrips, ntasks;
    warp_tasks_nw(L.n, 2 * HW_NW, wmh, nstrips, ntasks);
    CUtensorMap wx, wb, wk;
    cudaError_t e = encode_vec_map(&wx, x_zero ? b : x, L.n, L.pitch, L.plane, WXW, 1);
    if (e == cudaSuccess) e = encode_vec_map(&wb, b, L.n, L.pitch, L.plane, WBW, 1);
    if (e == cudaSuccess) e = encode_vec_map(&wk, L.kinv_field, L.n, L.pitch, L.plane, WXW, 1, 2);
    if (e != cudaSuccess) return e;
    const ProlSrc none{nullptr, 0, 0, 0};
    static int bk = -1, pf = -1;   // MG_HW_BK: boundary outputs by 1 the cooperative kernel, 2 one thread per vertex;
    if (bk < 0) {                  // MG_HW_PF: S~^{-1} rows prefetched 0 not, 1 into L2, 2 into L1
        const char* v = getenv("MG_HW_BK");
        bk = v ? atoi(v) : 1;
        v = getenv("MG_HW_PF");
        pf = v ? atoi(v) : 3;   // 3: into L2 below n = 2048 only (measured at 2048^2: level 0 0.42 -> 0.50 ms with the
    }                           // prefetches, levels 1-2 0.101 / 0.044 -> 0.095 / 0.039 ms)
    const int pfl = pf == 3 ? (L.n < 2048 ? 1 : 0) : pf;
    if (bk == 1) {
        const dim3 bgrid2((L.n + WB2_T) / WB2_T, 4);
        if (x_zero) launch_k(vanka_bnd2_kernel<true, false, true>, bgrid2, WB2_NT, 0, s, P, x, b, none);
        else launch_k(vanka_bnd2_kernel<false, false, true>, bgrid2, WB2_NT, 0, s, P, x, b, none);
    } else {
        const dim3 bgrid((bnd_count(L.n) + WB_NT - 1) / WB_NT);
        if (x_zero) launch_k(vanka_bnd_kernel<true, false, true>, bgrid, WB_NT, WB_SMEM, s, P, x, b, none);
        else launch_k(vanka_bnd_kernel<false, false, true>, bgrid, WB_NT, WB_SMEM, s, P, x, b, none);
    }
    const dim3 wgrid((ntasks + HW_NW - 1) / HW_NW);
    if (x_zero) launch_k(vanka_hwarp_kernel<true>, wgrid, HW_NT, HW_SMEM, s, wx, wb, wk, P, Ti, xo, S, wmh, nstrips, ntasks, pfl);
    else launch_k(vanka_hwarp_kernel<false>, wgrid, HW_NT, HW_SMEM, s, wx, wb, wk, P, Ti, xo, S, wmh, nstrips, ntasks, pfl);
    return cudaGetLastError();
}
int blocks_vanka_march2(int n) {
    const int MH = march_height(n, M2T, M2R, 3, relax_target(n));
    int wmh, nstrips, ntasks;
    warp_tasks(n, wmh, nstrips, ntasks);
    int wmhp, nstripsp, ntasksp;
    warp_tasks(n, wmhp, nstripsp, ntasksp, true);
    return std::max(std::max(((n + M2T) / M2T) * ((n + MH) / MH), (ntasks + WPC - 1) / WPC),
                    (ntasksp + WGeom<true>::NW - 1) / WGeom<true>::NW);
}



cudaError_t launch_bsr_a_march(const LevelParams& L, const DispParams& U, double omJ, const double* x, const double* b,
                               double* g, double* dp, NormSink S, bool x_zero, cudaStream_t s, const double* jtab,
                               double* rs) {
    CUtensorMap mx, mb, mk;
    cudaError_t e = encode_vec_map(&mx, x_zero ? b : x, L.n, L.pitch, L.plane, BQ_W, 1);
    if (e == cudaSuccess) e = encode_vec_map(&mb, b, L.n, L.pitch, L.plane, BQ_W, 1);
    const bool het = L.kinv_field != nullptr;
    if (e == cudaSuccess) e = encode_vec_map(&mk, het ? L.kinv_field : b, L.n, L.pitch, L.plane, BQ_W, 1, 2);
    if (e != cudaSuccess) return e;
    const int MH = march_height(L.n, BMA_T, BQ_R, 3, relax_target(L.n));
    dim3 grid((L.n + BMA_T) / BMA_T, (L.n + MH) / MH);
#define BA_LAUNCH(H_, Z_) launch_k(bsr_a_march_kernel<H_, Z_>, grid, BQ_NT, BMA_SMEM, s, mx, mb, mk, L, U, omJ, g, dp, S, MH, jtab, rs)
    if (het && x_zero) BA_LAUNCH(true, true);
    else if (het) BA_LAUNCH(true, false);
    else if (x_zero) BA_LAUNCH(false, true);
    else BA_LAUNCH(false, false);
#undef BA_LAUNCH
    return cudaGetLastError();
}

cudaError_t launch_bsr_b_march(const LevelParams& L, const DispParams& U, double omega, const double* x,
                               const double* b, const double* dp, double* xo, bool x_zero, cudaStream_t s,
                               const double* rs) {
    CUtensorMap mx, mb, md, mk;
    const bool rvec = rs != nullptr && !x_zero;   // r_u, r_w from stage A (8 planes) instead of a second residual
    cudaError_t e = encode_vec_map(&mx, x_zero ? b : x, L.n, L.pitch, L.plane, BQ_W, 1);
    if (e == cudaSuccess) e = rvec ? encode_vec_map(&mb, rs, L.n, L.pitch, L.plane, BQ_W, 1, 8)
                                   : encode_vec_map(&mb, b, L.n, L.pitch, L.plane, BQ_W, 1);
    if (e == cudaSuccess) e = encode_vec_map(&md, dp, L.n, L.pitch, L.plane, BQ_W, 1, 2);
    const bool het = L.kinv_field != nullptr;
    if (e == cudaSuccess) e = encode_vec_map(&mk, het ? L.kinv_field : dp, L.n, L.pitch, L.plane, BQ_W, 1, 2);
    if (e != cudaSuccess) return e;
    if (g_warp_min_n > 0 && L.n >= g_warp_min_n && g_warp_bsr && !rvec) {
        CUtensorMap wx, wb, wd, wk;
        e = encode_vec_map(&wx, x_zero ? b : x, L.n, L.pitch, L.plane, WXW, 1);
        if (e == cudaSuccess) e = encode_vec_map(&wb, b, L.n, L.pitch, L.plane, WBW, 1);
        if (e == cudaSuccess) e = encode_vec_map(&wd, dp, L.n, L.pitch, L.plane, WXW, 1, 2);
        if (e == cudaSuccess) e = encode_vec_map(&wk, het ? L.kinv_field : dp, L.n, L.pitch, L.plane, WXW, 1, 2);
        if (e != cudaSuccess) return e;
        int wmh, nstrips, ntasks;
        const int nw = het ? WQGeom<true>::NW : WQGeom<false>::NW;
        warp_tasks_nw(L.n, nw, wmh, nstrips, ntasks);
        const dim3 wgrid((ntasks + nw - 1) / nw);
#define WB_LAUNCH(H_, Z_) launch_k(bsr_b_warp_kernel<H_, Z_>, wgrid, WQGeom<H_>::NT, WQGeom<H_>::SMEM, s, wx, wb, wd, wk, L, U, \
                                   omega, xo, wmh, nstrips, ntasks)
        if (het && x_zero) WB_LAUNCH(true, true);
        else if (het) WB_LAUNCH(true, false);
        else if (x_zero) WB_LAUNCH(false, true);
        else WB_LAUNCH(false, false);
#undef WB_LAUNCH
        return cudaGetLastError();
    }
    // resident CTAs per SM: 3 with the x ring (68 KB), 5 without it (43 KB; MODE 1 and 2) -- MG_BSR_B_SLOTS overrides
    static int bslots = -1;
    if (bslots < 0) {
        const char* v = getenv("MG_BSR_B_SLOTS");
        bslots = v ? atoi(v) : 0;
    }
    const int MH = march_height(L.n, BB_T, BQ_R, bslots > 0 ? bslots : ((rvec || x_zero) ? 5 : 3), relax_target(L.n));
    dim3 grid((L.n + BB_T) / BB_T, (L.n + MH) / MH);
#define BB_LAUNCH(H_, M_) \
    launch_k(bsr_b_march_kernel<H_, M_>, grid, BQ_NT, M_ ? BB2_SMEM_NX : BB2_SMEM, s, mx, mb, md, mk, L, U, omega, xo, MH, x)
    if (het && x_zero) BB_LAUNCH(true, 1);
    else if (het && rvec) BB_LAUNCH(true, 2);
    else if (het) BB_LAUNCH(true, 0);
    else if (x_zero) BB_LAUNCH(false, 1);
    else if (rvec) BB_LAUNCH(false, 2);
    else BB_LAUNCH(false, 0);
#undef BB_LAUNCH
    return cudaGetLastError();
}

cudaError_t launch_restrict_march(const LevelParams& Lf, int nc, int pitchc, const double* x, const double* b,
                                  double* bc, cudaStream_t s) {
    CUtensorMap mx, mb, mk;
    cudaError_t e = encode_vec_map(&mx, x, Lf.n, Lf.pitch, Lf.plane, Q_XW, QF);
    if (e != cudaSuccess) return e;
    e = encode_vec_map(&mb, b, Lf.n, Lf.pitch, Lf.plane, Q_RW, QF);
    if (e != cudaSuccess) return e;
    e = encode_vec_map(&mk, Lf.kinv_field ? Lf.kinv_field : b, Lf.n, Lf.pitch, Lf.plane, Q_XW, QF, 2);
    if (e != cudaSuccess) return e;
    const int MH = march_height(nc, QT, QR, 3, 128);
    dim3 grid((nc + QT) / QT, (nc + MH) / MH);
    if (Lf.kinv_field) launch_k(restrict_march_kernel<true>, grid, QNT, Q_SMEM_K, s, mx, mb, mk, Lf, nc, pitchc, bc, MH);
    else launch_k(restrict_march_kernel<false>, grid, QNT, Q_SMEM, s, mx, mb, mk, Lf, nc, pitchc, bc, MH);
    return cudaGetLastError();
}

cudaError_t launch_restrict(const LevelParams& Lf, int nc, int pitchc, int mode, const double* x,
                            const double* br, double* bc, cudaStream_t s) {
    if (nc <= g_small_tile_n / 2) {
        using T = CTile<CSX, CSY>;
        dim3 grid((nc + CSX) / CSX, (nc + CSY) / CSY);
        if (mode == 1) {
            if (g_small_diet) {
                if (Lf.kinv_field) launch_k(restrict_small_kernel<true>, grid, T::NT, T::SMEM_FUSED, s, Lf, nc, pitchc, x, br, bc);
                else launch_k(restrict_small_kernel<false>, grid, T::NT, T::SMEM_FUSED, s, Lf, nc, pitchc, x, br, bc);
            } else if (Lf.kinv_field) {
                launch_k(restrict_kernel<1, true, CSX, CSY>, grid, T::NT, T::SMEM_FUSED, s, Lf, nc, pitchc, x, br, bc);
            } else {
                launch_k(restrict_kernel<1, false, CSX, CSY>, grid, T::NT, T::SMEM_FUSED, s, Lf, nc, pitchc, x, br, bc);
            }
        } else if (mode == 0) {
            launch_k(restrict_kernel<0, false, CSX, CSY>, grid, T::NT, T::SMEM_PLAIN, s, Lf, nc, pitchc, x, br, bc);
        } else {
            launch_k(restrict_kernel<2, false, CSX, CSY>, grid, T::NT, T::SMEM_PLAIN, s, Lf, nc, pitchc, x, br, bc);
        }
        return cudaGetLastError();
    }
    dim3 grid((nc + CX) / CX, (nc + CY) / CY);
    if (mode == 1) {
        if (Lf.kinv_field) launch_k(restrict_kernel<1, true>, grid, CNT, C_SMEM_FUSED, s, Lf, nc, pitchc, x, br, bc);
        else launch_k(restrict_kernel<1, false>, grid, CNT, C_SMEM_FUSED, s, Lf, nc, pitchc, x, br, bc);
    } else if (mode == 0) {
        launch_k(restrict_kernel<0, false>, grid, CNT, C_SMEM_PLAIN, s, Lf, nc, pitchc, x, br, bc);
    } else {
        launch_k(restrict_kernel<2, false>, grid, CNT, C_SMEM_PLAIN, s, Lf, nc, pitchc, x, br, bc);
    }
    return cudaGetLastError();
}

cudaError_t launch_bottom(const BottomArgs& A, cudaStream_t s) {
    // grid-wide: as many CTAs as can be co-resident (one per SM), launched cooperatively
    static int nblk = 0;
    if (!nblk) {
        int per = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, bottom_kernel, BOT_NT, BOT_SMEM);
        nblk = std::max(1, per) * sm_count();
        if (const char* v = getenv("MG_BOTTOM_CTAS")) nblk = std::max(1, std::min(nblk, atoi(v)));
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nblk);
    cfg.blockDim = dim3(BOT_NT);
    cfg.dynamicSmemBytes = BOT_SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, bottom_kernel, A);
}

cudaError_t launch_prolong(int nf, int pitchf, int nc, int pitchc, const double* e, double* x, const int* stop,
                           cudaStream_t s) {
    dim3 grid((nc + 31) / 32, (nc + 7) / 8);
    static int planes_n = -1;   // levels with nf >= this: the plane-split kernel (MG_PROL_PLANES_N; 0 = off)
    if (planes_n < 0) {
        const char* v = getenv("MG_PROL_PLANES_N");
        planes_n = v ? atoi(v) : 256;
    }
    if (planes_n > 0 && nf >= planes_n) {
        grid.z = 5;
        launch_k(prolong_planes_kernel, grid, 256, 0, s, nf, pitchf, nc, pitchc, e, x, stop);
    } else if (nf <= 256 && g_small_diet) launch_k(prolong_kernel<true>, grid, 256, 0, s, nf, pitchf, nc, pitchc, e, x, stop);
    else launch_k(prolong_kernel<false>, grid, 256, 0, s, nf, pitchf, nc, pitchc, e, x, stop);
    return cudaGetLastError();
}

cudaError_t launch_coarse(int N, const double* G, const int64_t* slots, const double* b, double* x,
                          const int* stop, cudaStream_t s) {
    if (N <= CS_MAXN && (reinterpret_cast<uintptr_t>(G) & 15) == 0) {
        launch_k(coarse_smem_kernel, 1, 256, (size_t)(((N * N + 1) & ~1) + N) * 8, s, N, G, slots, b, x, stop);
        return cudaGetLastError();
    }
    int blocks = N <= 1024 ? 1 : (N + 255) / 256;
    launch_k(coarse_kernel, blocks, 256, N * 8, s, N, G, slots, b, x, stop);
    return cudaGetLastError();
}

cudaError_t launch_bsr_a(const LevelParams& L, const DispParams& U, double omJ, const double* x, const double* b,
                         double* g, double* dp, NormSink S, bool x_zero, cudaStream_t s) {
    const bool het = L.kinv_field != nullptr;
    if (L.n <= g_small_tile_n) {
        using T = BATile<VSX, VSY>;
        dim3 grid((L.n + VSX) / VSX, (L.n + VSY) / VSY);
#define BAS(H_, Z_) launch_k(bsr_a_kernel<H_, Z_, VSX, VSY>, grid, T::NT, T::SMEM, s, L, U, omJ, x, b, g, dp, S)
        if (het && x_zero) BAS(true, true);
        else if (het) BAS(true, false);
        else if (x_zero) BAS(false, true);
        else BAS(false, false);
#undef BAS
        return cudaGetLastError();
    }
    dim3 grid((L.n + BTX) / BTX, (L.n + BTY) / BTY);
    if (het && x_zero) launch_k(bsr_a_kernel<true, true>, grid, BANT, BA_SMEM, s, L, U, omJ, x, b, g, dp, S);
    else if (het) launch_k(bsr_a_kernel<true, false>, grid, BANT, BA_SMEM, s, L, U, omJ, x, b, g, dp, S);
    else if (x_zero) launch_k(bsr_a_kernel<false, true>, grid, BANT, BA_SMEM, s, L, U, omJ, x, b, g, dp, S);
    else launch_k(bsr_a_kernel<false, false>, grid, BANT, BA_SMEM, s, L, U, omJ, x, b, g, dp, S);
    return cudaGetLastError();
}

cudaError_t launch_bsr_jacobi(const LevelParams& L, double omJ, const double* g, const double* dpi, double* dpo,
                              cudaStream_t s) {
    dim3 grid((L.n + 32) / 32, (L.n + 8) / 8);
    if (L.kinv_field) launch_k(bsr_jacobi_kernel<true>, grid, 256, 0, s, L, omJ, g, dpi, dpo);
    else launch_k(bsr_jacobi_kernel<false>, grid, 256, 0, s, L, omJ, g, dpi, dpo);
    return cudaGetLastError();
}

cudaError_t launch_jtable(const LevelParams& L, double* tab, cudaStream_t s) {
    dim3 grid((L.n + 32) / 32, (L.n + 8) / 8);
    if (L.kinv_field) launch_k(jtable_kernel<true>, grid, 256, 0, s, L, tab);
    else launch_k(jtable_kernel<false>, grid, 256, 0, s, L, tab);
    return cudaGetLastError();
}

cudaError_t launch_bsr_jacobi2_t(const LevelParams& L, double omJ, const double* g, const double* tab,
                                 const double* dpi, double* dpo, cudaStream_t s) {
    dim3 grid((L.n + 32) / 32, (L.n + 8) / 8);
    launch_k(bsr_jacobi2_t_kernel, grid, 256, 0, s, L, omJ, g, tab, dpi, dpo);
    return cudaGetLastError();
}

cudaError_t launch_bsr_jacobi_t(const LevelParams& L, double omJ, const double* g, const double* tab,
                                const double* dpi, double* dpo, cudaStream_t s) {
    dim3 grid((L.n + 32) / 32, (L.n + 8) / 8);
    launch_k(bsr_jacobi_t_kernel<0>, grid, 256, 0, s, L, omJ, g, tab, dpi, dpo);
    return cudaGetLastError();
}


cudaError_t launch_bsr_b(const LevelParams& L, const DispParams& U, double omega, const double* x, const double* b,
                         const double* dp, double* xo, bool x_zero, cudaStream_t s, const double* jg,
                         const double* jtab, double omJ) {
    const bool het = L.kinv_field != nullptr;
    if (L.n <= g_small_tile_n) {
        using T = BBTile<VSX, VSY>;
        dim3 grid((L.n + VSX) / VSX, (L.n + VSY) / VSY);
#define BBS(H_, Z_) launch_k(bsr_b_kernel<H_, Z_, VSX, VSY>, grid, T::NT, T::SMEM, s, L, U, omega, x, b, dp, xo, jg, jtab, omJ)
        if (het && x_zero) BBS(true, true);
        else if (het) BBS(true, false);
        else if (x_zero) BBS(false, true);
        else BBS(false, false);
#undef BBS
        return cudaGetLastError();
    }
    dim3 grid((L.n + BTX) / BTX, (L.n + BTY) / BTY);
    if (het && x_zero) launch_k(bsr_b_kernel<true, true>, grid, BBNT, BB_SMEM, s, L, U, omega, x, b, dp, xo, jg, jtab, omJ);
    else if (het) launch_k(bsr_b_kernel<true, false>, grid, BBNT, BB_SMEM, s, L, U, omega, x, b, dp, xo, jg, jtab, omJ);
    else if (x_zero) launch_k(bsr_b_kernel<false, true>, grid, BBNT, BB_SMEM, s, L, U, omega, x, b, dp, xo, jg, jtab, omJ);
    else launch_k(bsr_b_kernel<false, false>, grid, BBNT, BB_SMEM, s, L, U, omega, x, b, dp, xo, jg, jtab, omJ);
    return cudaGetLastError();
}

cudaError_t launch_kinv_from_K(int n, int pitch, const double* K, double* kinv, cudaStream_t s) {
    dim3 grid((n + 31) / 32, (n + 7) / 8);
    launch_k(kinv_from_K_kernel, grid, 256, 0, s, n, pitch, K, kinv);
    return cudaGetLastError();
}

cudaError_t launch_kinv_coarsen(int nf, int pitchf, const double* kf, int pitchc, double* kc, cudaStream_t s) {
    dim3 grid((nf / 2 + 31) / 32, (nf / 2 + 7) / 8);
    launch_k(kinv_coarsen_kernel, grid, 256, 0, s, nf, pitchf, kf, pitchc, kc);
    return cudaGetLastError();
}

// the kernels launched without a dynamic shared-memory attribute (set_smem carves the others)
static void carve_all() {
    carve(prolong_kernel<true>);
    carve(prolong_kernel<false>);
    carve(residual_kernel<false, false>);
    carve(residual_kernel<true, false>);
    carve(residual_kernel<false, true>);
    carve(residual_kernel<true, true>);
    carve(residual_march_kernel<0>);
    carve(residual_march_kernel<1>);
    carve(residual_march_kernel<2>);
    carve(residual_march_kernel<0, true>);
    carve(residual_march_kernel<1, true>);
    carve(residual_march_kernel<2, true>);
    carve(bsr_jacobi_kernel<false>);
    carve(bsr_jacobi_kernel<true>);
    carve(bsr_jacobi_t_kernel<0>);
    carve(vec_copy_kernel);
    carve(step_rhs_kernel);
}

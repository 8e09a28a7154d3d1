// C ABI of the B200 monolithic multigrid hot path (include/mg.h): context and hierarchy setup,
// the per-operation entry points and the V-cycle driver (captured once into a CUDA graph per
// (x, b, options) and replayed).  mg_solve keeps the iteration on the device: the level-0
// pre-smoothing kernel of each cycle fuses the residual norm of its input, the block that
// completes that norm appends it to the history and raises a stop flag that every later kernel
// polls at entry, so cycles can be launched ahead without host round trips.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mg.h"
#include "mg_internal.h"
#include "mg_kernels.cuh"

namespace {

thread_local std::string g_err;
mg_alloc_fn g_alloc = nullptr;
mg_free_fn g_free = nullptr;
void* g_user = nullptr;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(call)                                                                            \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess) return fail(MG_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

struct Level {
    int n = 0, pitch = 0;
    int64_t plane = 0, len = 0;
    double* x = nullptr;     // level >= 1 iterate
    double* b = nullptr;     // level >= 1 right-hand side
    double* t = nullptr;     // scratch for out-of-place sweeps
    double* g = nullptr;     // BSR: 2 planes
    double* dpa = nullptr;   // BSR: 2 planes
    double* dpb = nullptr;
    double* rs = nullptr;    // BSR marching levels: r_u, r_w of stage A for stage B (8 planes, allocated on first use)
    double* kinv = nullptr;  // 2 planes, heterogeneous K only
    double* jtab = nullptr;  // BSR Jacobi table: 5 planes (tau / D_w per RT0 edge, 1 / diag S per triangle)
    double* gbnd = nullptr;  // 9 x 400
    double* cgz = nullptr;      // exact BSR (Jacobi-PCG on S): z, p, q, 2 planes each (allocated on first use)
    double* cgp = nullptr;
    double* cgq = nullptr;
    double* hv_cls = nullptr;   // heterogeneous Vanka: 9 x MG_HV_CLS class tables
    double* hv_sinv = nullptr;  // heterogeneous Vanka: MG_HV_NSINV planes of per-vertex S_v^{-1}
    HvInterior hv_int{};        // heterogeneous Vanka: the interior class table (kernel parameter)
    double* ubnd = nullptr;  // 9 x 64
    VankaParams vp;
    DispParams up;
};

struct GraphEntry {
    const double* x;
    const double* b;
    mg_cycle_opts o;
    int solve;            // 0 plain, 1 solve state, 2 fused input norm into `nout`
    const double* nout;
    bool timed;
    cudaGraphExec_t exec;
};

}  // namespace

struct mg_ctx {
    int levels = 0;
    Material m{};
    bool het = false;
    bool exact = false;           // exact-integration operator (mg_grid.quadrature = MG_EXACT)
    double* cgst = nullptr;       // exact BSR: CG scalars (8 doubles) + partials + counter
    double* cgpart = nullptr;
    unsigned* cgcnt = nullptr;
    std::vector<Level> L;
    int Nc = 0;
    double* Ginv = nullptr;
    int64_t* slots = nullptr;
    // norms
    double* partials = nullptr;
    unsigned* counter = nullptr;
    double* norm = nullptr;
    int* stop = nullptr;
    SolveState* state = nullptr;  // device struct
    double* hist = nullptr;
    int hist_cap = 0;
    double* pinned = nullptr;     // host: 4 doubles + 256 of FGMRES scratch (device dots in, scales out)
    // e2e buffers
    double* hx = nullptr;
    double* hb = nullptr;
    // FGMRES work space (allocated on first use, grown with the restart length)
    std::vector<double*> kv, kz;
    double* kw = nullptr;
    double* kb = nullptr;         // mg_time_step: the step's right-hand side
    double* kdots = nullptr;      // device: 2 x 72 dot results + 8 coefficients
    double* kpart = nullptr;
    unsigned* kcnt = nullptr;
    int kcap = 0;
    std::vector<void*> allocs;
    mg_alloc_fn alloc = nullptr;  // allocator in force at mg_setup: every later allocation and free of
    mg_free_fn dfree = nullptr;   // this context uses it, whatever mg_set_allocator installs afterwards
    void* alloc_user = nullptr;
    std::vector<GraphEntry> graphs;
    cudaStream_t cap = nullptr;   // capture stream
    bool timing = false;
    bool timed_ran = false;
    std::vector<cudaEvent_t> lev;  // per-level phase events of the traced cycle (4 (L-1) + 2)
    int launches = 0;             // kernel launches enqueued by the last captured cycle
    int vanka_impl = 2;           // 2: row-granular marching TMA kernel (default), 0: 2-D tiles everywhere
    int restrict_impl = 1;        // 1: row-marching TMA fused residual + restriction, 0: 2-D tile kernel
    int jacobi_fuse_b = 1;        // 2-D tile levels: the last two table sweeps inside stage B (MG_JACOBI_FUSE_B)
    int jacobi_pair = 1;          // two table sweeps per launch where two remain (MG_JACOBI_PAIR)
    int bsr_rvec = 1;             // marching BSR: stage B reads stage A's residual instead of recomputing it (MG_BSR_RVEC)
    int het_warp_n = 256;         // K-field levels with n >= this: warp-marching het Vanka sweep (MG_HET_WARP_N; 0 = 2-D tiles)
    int march_min_n = 512;        // levels with fewer cells per side use the single-pass 2-D tile kernels
    int bottom_n = 0;             // > 0: Vanka levels with n <= bottom_n (down to the coarsest) in one kernel
                                  // (measured slower: one CTA 442 us, grid-wide cooperative 323 us vs 247 us
                                  //  per 256^2 cycle with the per-level kernels)
    int jacobi_table = 1;         // 1: Jacobi sweeps from the per-level table (bsr_jacobi_t_kernel)
    int bsr_impl = 1;             // 1: row-marching BSR stages on levels with n >= march_min_n, 0: 2-D tiles
    int fuse_prolong = 1;         // 1: prolongation fused into the first post-sweep of marching Vanka levels
    double dgks_eta2 = 0.01;      // selective reorthogonalisation (DGKS form): second Gram-Schmidt pass when the first
                                  // cancelled more than 10x, |U'|^2 < eta^2 |U|^2 (MG_DGKS_ETA2; 0.5 = the classical 1/sqrt2:
                                  // a pass in every iteration here; one pass leaves orthogonality ~ u / eta per vector)
    int cgs_passes = 0;           // FGMRES Gram-Schmidt: 0 adaptive (second pass when |U'| < |U|/sqrt2,
                                  // the DGKS criterion), 1 single, 2 always twice (MG_CGS_PASSES)
    cudaEvent_t ev[6] = {};
};

namespace {

void* dalloc(mg_ctx* c, size_t bytes) {
    void* p = nullptr;
    if (c->alloc) p = c->alloc(bytes, c->alloc_user);
    else if (cudaMalloc(&p, bytes) != cudaSuccess) p = nullptr;
    if (p) c->allocs.push_back(p);
    return p;
}

void dfree_all(mg_ctx* c) {
    for (void* p : c->allocs) {
        if (c->dfree) c->dfree(p, c->alloc_user);
        else cudaFree(p);
    }
    c->allocs.clear();
}

int pitch_of(int n) { return ((n + 1 + 31) / 32) * 32; }

// every vector pointer must be 16-byte aligned: the kernels move column pairs as double2 and TMA
// descriptors need 16-byte global addresses (include/mg.h OWNERSHIP)
bool aligned(const void* p) { return p && (reinterpret_cast<uintptr_t>(p) % 16 == 0); }

int check_level(const mg_ctx* c, int level, int maxl) {
    if (!c) return fail(MG_EINVAL, "null context");
    if (level < 0 || level > maxl) return fail(MG_EINVAL, "level %d out of range [0, %d]", level, maxl);
    return MG_OK;
}

NormSink no_norm() { return NormSink{nullptr, nullptr, nullptr, nullptr}; }

// iteration cap of the exact-BSR CG on a level of n cells: Jacobi-PCG on the P0 graph operator S
// needs O(n) iterations (cond ~ n^2); the device flag ends it earlier at the 1e-14 tolerance
int cg_iters(int n) { return 24 * n + 64; }

// does the first post-sweep on level l absorb the prolongation (relax_once with e_coarse)?
bool fused_prolong(const mg_ctx* c, int l, const mg_cycle_opts& o) {
    if (!c->fuse_prolong || o.relax != MG_VANKA || o.nu2 < 1 || c->het || c->exact) return false;
    if (c->vanka_impl == 2 && c->L[l].n >= c->march_min_n) return true;   // marching / warp sweeps
    return c->L[l].n <= small_tile_n() && small_diet();                   // small-tile sweep (vanka_small_kernel)
}

// one relaxation sweep on level l: xin -> xout (out of place).  e_coarse != nullptr (only where
// fused_prolong): the sweep relaxes xin + P e_coarse, e_coarse being level l + 1's iterate.
int relax_once(mg_ctx* c, int l, const double* xin, const double* b, double* xout, bool xzero,
               const mg_cycle_opts& o, NormSink S, cudaStream_t s, const double* e_coarse = nullptr) {
    Level& Lv = c->L[l];
    if (o.relax == MG_VANKA) {
        VankaParams P = Lv.vp;
        P.omega = o.omega;
        if (e_coarse) {
            const Level& Lc = c->L[l + 1];
            const ProlSrc E{e_coarse, Lc.n, Lc.pitch, (int64_t)(Lc.n + 1) * Lc.pitch};
            if (Lv.n <= small_tile_n()) CK(launch_vanka(P, xin, b, xout, false, S, s, nullptr, &E));
            else CK(launch_vanka_march2(P, xin, b, xout, false, S, s, &E));
            return MG_OK;
        }
        if (c->vanka_impl == 2 && Lv.n >= c->march_min_n && !c->het && !c->exact)
            CK(launch_vanka_march2(P, xin, b, xout, xzero, S, s));
        else if (c->het && !c->exact && c->het_warp_n > 0 && Lv.n >= c->het_warp_n)
            CK(launch_vanka_hwarp(P, Lv.hv_int, xin, b, xout, xzero, S, s));
        else CK(launch_vanka(P, xin, b, xout, xzero, S, s, c->het ? &Lv.hv_int : nullptr));
        return MG_OK;
    }
    const bool exact_s = o.relax == MG_BSR_EXACT;
    const double omJ = (!exact_s && o.jacobi_sweeps >= 1) ? o.omega_J : 0.0;
    const bool march = c->bsr_impl == 1 && Lv.n >= c->march_min_n && !c->exact;
    double* rs = (march && !xzero) ? Lv.rs : nullptr;   // allocated by ensure_rs when bsr_rvec
    if (march) CK(launch_bsr_a_march(Lv.vp.L, Lv.up, omJ, xin, b, Lv.g, Lv.dpa, S, xzero, s, Lv.jtab, rs));
    else CK(launch_bsr_a(Lv.vp.L, Lv.up, omJ, xin, b, Lv.g, Lv.dpa, S, xzero, s));
    double* cur = Lv.dpa;
    double* nxt = Lv.dpb;
    if (exact_s) {   // exact BSR: S dp = g by Jacobi-PCG to fp64 accuracy
        CK(launch_cg_exact(Lv.vp.L, Lv.jtab, Lv.g, Lv.dpa, Lv.cgz, Lv.cgp, Lv.cgq, c->cgpart, c->cgcnt, c->cgst,
                           cg_iters(Lv.n), s));
    }
    // 2-D tile levels: the last two table sweeps run inside stage B (one launch less per relaxation)
    const bool fuse_b = !march && !exact_s && c->jacobi_table && c->jacobi_fuse_b && o.jacobi_sweeps >= 3;
    const int jend = fuse_b ? o.jacobi_sweeps - 2 : o.jacobi_sweeps;
    for (int k = 1; !exact_s && k < jend;) {
        if (c->jacobi_table && c->jacobi_pair && k + 2 <= jend) {
            CK(launch_bsr_jacobi2_t(Lv.vp.L, o.omega_J, Lv.g, Lv.jtab, cur, nxt, s));
            k += 2;
        } else if (c->jacobi_table) {
            CK(launch_bsr_jacobi_t(Lv.vp.L, o.omega_J, Lv.g, Lv.jtab, cur, nxt, s));
            k += 1;
        } else {
            CK(launch_bsr_jacobi(Lv.vp.L, o.omega_J, Lv.g, cur, nxt, s));
            k += 1;
        }
        std::swap(cur, nxt);
    }
    if (march) CK(launch_bsr_b_march(Lv.vp.L, Lv.up, o.omega, xin, b, cur, xout, xzero, s, rs));
    else if (fuse_b) CK(launch_bsr_b(Lv.vp.L, Lv.up, o.omega, xin, b, cur, xout, xzero, s, Lv.g, Lv.jtab, o.omega_J));
    else CK(launch_bsr_b(Lv.vp.L, Lv.up, o.omega, xin, b, cur, xout, xzero, s));
    return MG_OK;
}

// marching BSR: the residual vector stage A hands to stage B (planes 0-7 = r_u, r_w) on the marching levels
int ensure_rs(mg_ctx* c) {
    if (!c->bsr_rvec || c->bsr_impl != 1 || c->exact) return MG_OK;
    for (auto& Lv : c->L) {
        if (Lv.rs || Lv.n < c->march_min_n) continue;
        const size_t pb = sizeof(double) * 8 * Lv.plane;
        Lv.rs = (double*)dalloc(c, pb);
        if (!Lv.rs) return fail(MG_ENOMEM, "BSR residual work space");
        CK(cudaMemset(Lv.rs, 0, pb));
    }
    return MG_OK;
}

// exact BSR work space: z, p, q (2 P0 planes each) per level and the CG scalars
int ensure_cg(mg_ctx* c) {
    if (c->cgst) return MG_OK;
    for (auto& Lv : c->L) {
        const size_t pb = sizeof(double) * 2 * Lv.plane;
        Lv.cgz = (double*)dalloc(c, pb);
        Lv.cgp = (double*)dalloc(c, pb);
        Lv.cgq = (double*)dalloc(c, pb);
        if (!Lv.cgz || !Lv.cgp || !Lv.cgq) return fail(MG_ENOMEM, "exact BSR work space");
        CK(cudaMemset(Lv.cgz, 0, pb));
        CK(cudaMemset(Lv.cgp, 0, pb));
        CK(cudaMemset(Lv.cgq, 0, pb));
    }
    c->cgpart = (double*)dalloc(c, sizeof(double) * cg_partials_needed(c->L[0].n));
    c->cgcnt = (unsigned*)dalloc(c, 64);
    double* st = (double*)dalloc(c, sizeof(double) * 8);
    if (!c->cgpart || !c->cgcnt || !st) return fail(MG_ENOMEM, "exact BSR work space");
    CK(cudaMemset(c->cgcnt, 0, 64));
    const double init[8] = {0, 0, 0, 0, 1e-28, 0, 0, 0};   // [4] = tol^2 (1e-14 in the D^{-1} norm)
    CK(cudaMemcpy(st, init, sizeof(init), cudaMemcpyHostToDevice));
    c->cgst = st;
    return MG_OK;
}

// first level handled by the single-CTA bottom kernel, or -1
int bottom_level(const mg_ctx* c, const mg_cycle_opts& o) {
    const int Lc = c->levels - 1;
    if (c->bottom_n <= 0 || o.relax != MG_VANKA || o.nu1 < 1 || o.nu2 < 1 || !c->Ginv || c->het) return -1;
    int lb = -1;
    for (int l = Lc - 1; l >= 1; --l)
        if (c->L[l].n <= c->bottom_n && Lc - l <= BOT_MAXL) lb = l;
    return lb;
}

// enqueue one V(nu1, nu2) cycle (PAPER.md:471-476 recursed).  solve != 0: the
// first level-0 operation appends ||b - A x||^2 to the solve state.
int enqueue_cycle(mg_ctx* c, double* x0, const double* b0, const mg_cycle_opts& o, int solve, double* nout,
                  bool timed, cudaStream_t s) {
    const int Lc = c->levels - 1;
    std::vector<double*> cur(c->levels, nullptr);
    NormSink S = no_norm();
    if (solve == 1) S = NormSink{nullptr, c->partials, c->counter, c->state};
    if (solve == 2) S = NormSink{nout, c->partials, c->counter, nullptr};
    auto mark = [&](int i) -> int {
        if (timed) CK(cudaEventRecordWithFlags(c->ev[i], s, cudaEventRecordExternal));
        return MG_OK;
    };
    int nlev = 0;   // per-level boundaries: pre(0) restrict(0) ... pre(L-2) restrict(L-2) coarse prolong(L-2) post(L-2) ...
    auto lmark = [&]() -> int {
        if (timed) CK(cudaEventRecordWithFlags(c->lev[nlev], s, cudaEventRecordExternal));
        ++nlev;
        return MG_OK;
    };
    if (int rc = lmark()) return rc;
    if (int rc = mark(0)) return rc;
    if ((solve == 1 || solve == 2) && o.nu1 == 0) {
        CK(launch_residual(c->L[0].vp.L, x0, b0, nullptr, S, s));
        S = no_norm();
    }
    const int lb = bottom_level(c, o);
    for (int l = 0; l < Lc; ++l) {
        if (l == lb) break;
        Level& Lv = c->L[l];
        double* xl = l == 0 ? x0 : Lv.x;
        const double* bl = l == 0 ? b0 : Lv.b;
        const bool zero = l > 0 || solve == 3;   // solve == 3: x0 is zero (FGMRES preconditioner)
        double* a = xl;
        double* t = Lv.t;
        for (int k = 0; k < o.nu1; ++k) {
            int rc = relax_once(c, l, a, bl, t, zero && k == 0, o, l == 0 && k == 0 ? S : no_norm(), s);
            if (rc) return rc;
            std::swap(a, t);
        }
        if (l == 0)
            if (int rc = mark(1)) return rc;
        if (int rc = lmark()) return rc;
        if (zero && o.nu1 == 0) CK(cudaMemsetAsync(xl, 0, sizeof(double) * Lv.len, s));
        const int mode = (zero && o.nu1 == 0) ? 2 : 1;
        if (mode == 1 && c->restrict_impl == 1 && Lv.n >= c->march_min_n && !c->exact)
            CK(launch_restrict_march(Lv.vp.L, c->L[l + 1].n, c->L[l + 1].pitch, a, bl, c->L[l + 1].b, s));
        else
            CK(launch_restrict(Lv.vp.L, c->L[l + 1].n, c->L[l + 1].pitch, mode, a, bl, c->L[l + 1].b, s));
        if (l == 0)
            if (int rc = mark(2)) return rc;
        if (int rc = lmark()) return rc;
        cur[l] = a;
    }
    if (lb >= 0) {
        // levels lb .. Lc in one CTA; the host replays its buffer swaps to know where level lb ends
        BottomArgs A{};
        A.nl = Lc - lb;
        A.nu1 = o.nu1;
        A.nu2 = o.nu2;
        for (int i = 0; i <= A.nl; ++i) {
            Level& Lv = c->L[lb + i];
            A.x[i] = Lv.x;
            A.b[i] = Lv.b;
            A.pitch[i] = Lv.pitch;
            if (i < A.nl) {
                A.vp[i] = Lv.vp;
                A.vp[i].omega = o.omega;
                A.t[i] = Lv.t;
            }
        }
        A.N = c->Nc;
        A.G = c->Ginv;
        A.slots = c->slots;
        A.stop = c->stop;
        CK(launch_bottom(A, s));
        for (int i = 0; i < A.nl; ++i) {
            double* a = A.x[i];
            double* t = A.t[i];
            for (int k = 0; k < o.nu1; ++k) std::swap(a, t);
            t = (a == A.x[i]) ? A.t[i] : A.x[i];
            for (int k = 0; k < o.nu2; ++k) std::swap(a, t);
            cur[lb + i] = a;
        }
        cur[Lc] = c->L[Lc].x;
        for (int k = 0; k < 4 * A.nl + 1; ++k)   // the per-level timing slots of levels lb .. Lc
            if (int rc = lmark()) return rc;
    } else {
        CK(launch_coarse(c->Nc, c->Ginv, c->slots, c->L[Lc].b, c->L[Lc].x, c->stop, s));
        if (int rc = lmark()) return rc;
        cur[Lc] = c->L[Lc].x;
    }
    for (int l = Lc - 1; l >= 0; --l) {
        if (lb >= 0 && l >= lb) continue;
        Level& Lv = c->L[l];
        if (l == 0)
            if (int rc = mark(3)) return rc;
        const bool fuse = fused_prolong(c, l, o);
        if (!fuse) CK(launch_prolong(Lv.n, Lv.pitch, c->L[l + 1].n, c->L[l + 1].pitch, cur[l + 1], cur[l], c->stop, s));
        if (l == 0)
            if (int rc = mark(4)) return rc;
        if (int rc = lmark()) return rc;
        const double* bl = l == 0 ? b0 : Lv.b;
        double* xl = l == 0 ? x0 : Lv.x;
        double* a = cur[l];
        double* t = (a == xl) ? Lv.t : xl;
        for (int k = 0; k < o.nu2; ++k) {
            int rc = relax_once(c, l, a, bl, t, false, o, no_norm(), s, fuse && k == 0 ? cur[l + 1] : nullptr);
            if (rc) return rc;
            std::swap(a, t);
        }
        // odd sweep count: copy back with a kernel that honours mg_solve's stop flag (a memcpy node
        // would also run in the stopping cycle and return the pre-sweep's output)
        if (l == 0 && a != x0) CK(launch_copy(x0, a, Lv.len, c->stop, s));
        if (int rc = lmark()) return rc;
        cur[l] = a;
    }
    return mark(5);
}

bool same_opts(const mg_cycle_opts& a, const mg_cycle_opts& b) {
    return a.nu1 == b.nu1 && a.nu2 == b.nu2 && a.relax == b.relax && a.omega == b.omega &&
           a.omega_J == b.omega_J && a.jacobi_sweeps == b.jacobi_sweeps;
}

int get_graph(mg_ctx* c, double* x, const double* b, const mg_cycle_opts& o, int solve, double* nout,
              cudaGraphExec_t* out) {
    for (auto& g : c->graphs)
        if (g.x == x && g.b == b && g.solve == solve && g.nout == nout && g.timed == c->timing && same_opts(g.o, o)) {
            *out = g.exec;
            return MG_OK;
        }
    if (c->graphs.size() >= 96) {
        cudaGraphExecDestroy(c->graphs.front().exec);
        c->graphs.erase(c->graphs.begin());
    }
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal));
    int rc = enqueue_cycle(c, x, b, o, solve, nout, c->timing, c->cap);
    cudaError_t e = cudaStreamEndCapture(c->cap, &graph);
    if (rc) return rc;
    if (e != cudaSuccess) return fail(MG_ECUDA, "graph capture: %s", cudaGetErrorString(e));
    {
        size_t nn = 0;
        cudaGraphGetNodes(graph, nullptr, &nn);
        std::vector<cudaGraphNode_t> nodes(nn);
        cudaGraphGetNodes(graph, nodes.data(), &nn);
        int k = 0;
        for (auto nd : nodes) {
            cudaGraphNodeType t;
            cudaGraphNodeGetType(nd, &t);
            if (t == cudaGraphNodeTypeKernel) ++k;
        }
        c->launches = k;
    }
    cudaGraphExec_t exec;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return fail(MG_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
    c->graphs.push_back(GraphEntry{x, b, o, solve, nout, c->timing, exec});
    *out = exec;
    return MG_OK;
}

int check_opts(mg_ctx* c, const mg_cycle_opts* o) {
    if (!o) return fail(MG_EINVAL, "null options");
    if (o->nu1 < 0 || o->nu2 < 0 || o->nu1 + o->nu2 < 0) return fail(MG_EINVAL, "nu1, nu2 must be >= 0");
    if (o->relax != MG_VANKA && o->relax != MG_BSR && o->relax != MG_BSR_EXACT)
        return fail(MG_EINVAL, "relax must be MG_VANKA, MG_BSR or MG_BSR_EXACT");
    if (!std::isfinite(o->omega) || !std::isfinite(o->omega_J)) return fail(MG_EINVAL, "omega not finite");
    if (o->relax == MG_BSR && o->jacobi_sweeps < 0) return fail(MG_EINVAL, "jacobi_sweeps < 0");
    if (o->relax == MG_BSR_EXACT && c->L[0].n > 1024)
        return fail(MG_EINVAL, "exact BSR (a full S solve per relaxation) is limited to n <= 1024");
    if (o->relax == MG_BSR_EXACT)
        if (int rc = ensure_cg(c)) return rc;
    if (o->relax == MG_BSR)
        if (int rc = ensure_rs(c)) return rc;
    return MG_OK;
}

}  // namespace

extern "C" {

void mg_set_allocator(mg_alloc_fn a, mg_free_fn f, void* user) {
    g_alloc = a;
    g_free = f;
    g_user = user;
}

const char* mg_last_error(void) { return g_err.c_str(); }

int32_t mg_levels(const mg_ctx* c) { return c ? c->levels : -1; }
int32_t mg_level_n(const mg_ctx* c, int32_t l) { return (c && l >= 0 && l < c->levels) ? c->L[l].n : -1; }
int32_t mg_pitch(const mg_ctx* c, int32_t l) { return (c && l >= 0 && l < c->levels) ? c->L[l].pitch : -1; }
int64_t mg_vec_len(const mg_ctx* c, int32_t l) { return (c && l >= 0 && l < c->levels) ? c->L[l].len : -1; }
int64_t mg_n_active(const mg_ctx* c, int32_t l) {
    return (c && l >= 0 && l < c->levels) ? n_active_of(c->L[l].n) : -1;
}

int mg_setup(const mg_grid* grid, double lambda, double mu, double K, double tau, double alpha, int32_t levels,
             mg_ctx** out) {
    if (!out) return fail(MG_EINVAL, "out is NULL");
    *out = nullptr;
    if (!grid) return fail(MG_EINVAL, "grid is NULL");
    const int n = grid->n;
    if (levels < 1) return fail(MG_EINVAL, "levels = %d < 1", levels);
    if (levels > 24 || n < 2 || n % (1 << (levels - 1)) != 0 || (n >> (levels - 1)) < 2)
        return fail(MG_EINVAL, "n = %d must be divisible by 2^(levels-1) with coarsest n >= 2 (levels = %d)", n, levels);
    if (!(mu > 0) || !(lambda >= 0) || !(tau > 0) || !std::isfinite(alpha) || !std::isfinite(lambda) ||
        !std::isfinite(mu) || !std::isfinite(tau))
        return fail(MG_EINVAL, "need lambda >= 0, mu > 0, tau > 0, finite alpha");
    if (!grid->K_field && !(K > 0 && std::isfinite(K))) return fail(MG_EINVAL, "K must be > 0 and finite");
    if (!(grid->inv_M > 0) || !std::isfinite(grid->inv_M))
        return fail(MG_EINVAL, "inv_M must be > 0 (the deflated solves need the -(1/M) M_p block)");
    if (!(grid->mu_f > 0)) return fail(MG_EINVAL, "mu_f must be > 0");
    if (grid->quadrature != MG_RQ && grid->quadrature != MG_EXACT) return fail(MG_EINVAL, "quadrature must be MG_RQ or MG_EXACT");
    if (grid->K_field && !aligned(grid->K_field)) return fail(MG_EINVAL, "K_field not 16-byte aligned");
    const int nc = n >> (levels - 1);
    // the dense coarsest solve needs n_c <= 20; a context with a larger coarsest level offers the
    // per-level operations only (mg_coarse_solve, mg_cycle and mg_solve return MG_EINVAL)
    const bool dense_ok = 10LL * nc * nc - 8LL * nc + 2 <= 4096;

    mg_ctx* c = new mg_ctx;
    c->alloc = g_alloc;
    c->dfree = g_free;
    c->alloc_user = g_user;
    c->levels = levels;
    c->het = grid->K_field != nullptr;
    c->m = Material{lambda, mu, grid->K_field ? 1.0 : K, tau, alpha, grid->inv_M, grid->mu_f};
    c->exact = grid->quadrature == MG_EXACT;
    c->m.exact = c->exact ? 1 : 0;
    c->L.resize(levels);
    set_carveout(getenv("MG_CARVEOUT") ? atoi(getenv("MG_CARVEOUT")) : 100);
    kernels_init();
    if (const char* v = getenv("MG_VANKA_IMPL")) c->vanka_impl = atoi(v);
    if (const char* v = getenv("MG_RESTRICT_IMPL")) c->restrict_impl = atoi(v);
    if (const char* v = getenv("MG_MARCH_MIN_N")) c->march_min_n = atoi(v);
    if (const char* v = getenv("MG_HET_WARP_N")) c->het_warp_n = atoi(v);
    if (const char* v = getenv("MG_BSR_RVEC")) c->bsr_rvec = atoi(v);
    if (const char* v = getenv("MG_JACOBI_PAIR")) c->jacobi_pair = atoi(v);
    if (const char* v = getenv("MG_JACOBI_FUSE_B")) c->jacobi_fuse_b = atoi(v);
    if (getenv("MG_WARP_BSR") && atoi(getenv("MG_WARP_BSR"))) c->bsr_rvec = 0;   // the warp stage B evaluates r itself
    if (const char* v = getenv("MG_FUSE_PROLONG")) c->fuse_prolong = atoi(v) != 0;
    if (const char* v = getenv("MG_BSR_IMPL")) c->bsr_impl = atoi(v);
    // process-wide kernel knobs: every setup re-reads them (unset -> default), so they never stick
    set_small_tile_n(getenv("MG_SMALL_TILE_N") ? atoi(getenv("MG_SMALL_TILE_N")) : 128);
    set_pdl(getenv("MG_PDL") ? atoi(getenv("MG_PDL")) != 0 : 0);
    set_prol_ws(getenv("MG_PROL_WS") ? atoi(getenv("MG_PROL_WS")) : 0);
    set_resid_march_n(getenv("MG_RESID_MARCH_N") ? atoi(getenv("MG_RESID_MARCH_N")) : 512);
    set_warp_min_n(getenv("MG_WARP_MIN_N") ? atoi(getenv("MG_WARP_MIN_N")) : 512);
    set_small_diet(getenv("MG_SMALL_DIET") ? atoi(getenv("MG_SMALL_DIET")) : 2);
    set_warp_prol(getenv("MG_WARP_PROL") ? atoi(getenv("MG_WARP_PROL")) : 1);
    set_warp_bk(getenv("MG_WARP_BK") ? atoi(getenv("MG_WARP_BK")) : 1);
    set_warp_bsr(getenv("MG_WARP_BSR") ? atoi(getenv("MG_WARP_BSR")) : 0);
    if (const char* v = getenv("MG_JACOBI_TABLE")) c->jacobi_table = atoi(v) != 0;
    if (const char* v = getenv("MG_BOTTOM_N")) c->bottom_n = atoi(v);
    if (const char* v = getenv("MG_CGS_PASSES")) c->cgs_passes = std::min(2, std::max(0, atoi(v)));
    if (const char* v = getenv("MG_DGKS_ETA2")) c->dgks_eta2 = atof(v);
    auto bail = [&](int rc) {
        mg_free(c);
        return rc;
    };
    char err[256];
    if (cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking) != cudaSuccess)
        return bail(fail(MG_ECUDA, "stream create failed"));
    int max_blocks = 1;
    for (int l = 0; l < levels; ++l) {
        Level& Lv = c->L[l];
        Lv.n = n >> l;
        Lv.pitch = pitch_of(Lv.n);
        Lv.plane = (int64_t)(Lv.n + 1) * Lv.pitch;
        Lv.len = 10 * Lv.plane;
        max_blocks = std::max(max_blocks, std::max(blocks_vanka(Lv.n), std::max(blocks_residual(Lv.n), blocks_bsr(Lv.n))));
        max_blocks = std::max(max_blocks, blocks_vanka_march2(Lv.n));
        max_blocks = std::max(max_blocks, blocks_residual_march(Lv.n));
        HostLevelTables* t = new HostLevelTables;
        if (host_level_tables(Lv.n, c->m, t, err, sizeof(err))) {
            delete t;
            return bail(fail(MG_EINVAL, "level %d: %s", l, err));
        }
        Lv.vp.L = t->L;
        Lv.vp.hv = HetVankaTabs{nullptr, nullptr};   // set below for a K field
        Lv.vp.L.pitch = Lv.pitch;
        Lv.vp.L.plane = Lv.plane;
        for (int a = 0; a < 9; ++a)
            for (int cc = 0; cc < 9; ++cc) Lv.vp.gpT[cc][a] = t->gp[a][cc];
        for (int a = 0; a < 11; ++a)
            for (int cc = 0; cc < 11; ++cc) Lv.vp.gmT[cc][a] = t->gm[a][cc];
        for (int a = 0; a < 3; ++a)
            for (int cc = 0; cc < 3; ++cc) Lv.up.upT[cc][a] = t->up[a][cc];
        for (int a = 0; a < 5; ++a)
            for (int cc = 0; cc < 5; ++cc) Lv.up.umT[cc][a] = t->um[a][cc];
        if (!c->het) {
            for (int s = 0; s < 2; ++s)
                for (int e = 0; e < 3; ++e)
                    for (int e2 = 0; e2 < 3; ++e2) Lv.vp.L.ww[s][e][e2] *= Lv.vp.L.kinv;
        }
        size_t vb = sizeof(double) * Lv.len, pb = sizeof(double) * 2 * Lv.plane;
        Lv.t = (double*)dalloc(c, vb);
        Lv.g = (double*)dalloc(c, pb);
        Lv.dpa = (double*)dalloc(c, pb);
        Lv.dpb = (double*)dalloc(c, pb);
        Lv.gbnd = (double*)dalloc(c, sizeof(t->vanka));
        Lv.ubnd = (double*)dalloc(c, sizeof(t->disp));
        if (l > 0) {
            Lv.x = (double*)dalloc(c, vb);
            Lv.b = (double*)dalloc(c, vb);
        }
        if (c->het) Lv.kinv = (double*)dalloc(c, pb);
        Lv.jtab = (double*)dalloc(c, sizeof(double) * 5 * Lv.plane);
        Lv.vp.bcorr = (double*)dalloc(c, sizeof(double) * 20 * 4 * std::max(Lv.n, 1));
        if (!Lv.vp.bcorr || !Lv.t || !Lv.g || !Lv.dpa || !Lv.dpb || !Lv.gbnd || !Lv.ubnd || !Lv.jtab || (l > 0 && (!Lv.x || !Lv.b)) ||
            (c->het && !Lv.kinv)) {
            delete t;
            return bail(fail(MG_ENOMEM, "device allocation failed at level %d", l));
        }
        if (cudaMemcpy(Lv.gbnd, t->vanka, sizeof(t->vanka), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(Lv.ubnd, t->disp, sizeof(t->disp), cudaMemcpyHostToDevice) != cudaSuccess) {
            delete t;
            return bail(fail(MG_ECUDA, "table upload failed"));
        }
        delete t;
        Lv.vp.gbnd = Lv.gbnd;
        Lv.up.ubnd = Lv.ubnd;
        Lv.vp.L.kinv_field = Lv.kinv;
        cudaMemset(Lv.t, 0, vb);
        cudaMemset(Lv.g, 0, pb);
        cudaMemset(Lv.dpa, 0, pb);
        cudaMemset(Lv.dpb, 0, pb);
        if (l > 0) {
            cudaMemset(Lv.x, 0, vb);
            cudaMemset(Lv.b, 0, vb);
        }
    }
    // K^{-1} pyramid (reading A11)
    if (c->het) {
        for (int l = 0; l < levels; ++l) cudaMemset(c->L[l].kinv, 0, sizeof(double) * 2 * c->L[l].plane);
        if (launch_kinv_from_K(n, c->L[0].pitch, grid->K_field, c->L[0].kinv, 0) != cudaSuccess)
            return bail(fail(MG_ECUDA, "kinv launch: %s", cudaGetErrorString(cudaGetLastError())));
        for (int l = 1; l < levels; ++l)
            if (launch_kinv_coarsen(c->L[l - 1].n, c->L[l - 1].pitch, c->L[l - 1].kinv, c->L[l].pitch, c->L[l].kinv, 0) !=
                cudaSuccess)
                return bail(fail(MG_ECUDA, "kinv coarsen launch failed"));
    }
    // BSR Jacobi tables (after the K^-1 pyramid they are formed from)
    for (int l = 0; l < levels; ++l) {
        cudaMemset(c->L[l].jtab, 0, sizeof(double) * 5 * c->L[l].plane);
        if (launch_jtable(c->L[l].vp.L, c->L[l].jtab, 0) != cudaSuccess)
            return bail(fail(MG_ECUDA, "jtable launch: %s", cudaGetErrorString(cudaGetLastError())));
    }
    // heterogeneous Vanka: condensed class tables + per-vertex S_v^{-1}
    if (c->het) {
        std::vector<double> hcls(MG_NCLASS * MG_HV_CLS), hw(MG_NCLASS * MG_HV_W), hc(MG_NCLASS * 36);
        for (int l = 0; l < levels; ++l) {
            Level& Lv = c->L[l];
            if (host_hv_tables(Lv.n, c->m, hcls.data(), hw.data(), hc.data(), &Lv.hv_int.pm, err, sizeof(err)))
                return bail(fail(MG_EINVAL, "level %d heterogeneous Vanka tables: %s", l, err));
            Lv.hv_cls = (double*)dalloc(c, sizeof(double) * hcls.size());
            Lv.hv_sinv = (double*)dalloc(c, sizeof(double) * MG_HV_NSINV * Lv.plane);
            double* dw = (double*)dalloc(c, sizeof(double) * (hw.size() + hc.size()));
            if (!Lv.hv_cls || !Lv.hv_sinv || !dw) return bail(fail(MG_ENOMEM, "heterogeneous Vanka tables (level %d)", l));
            if (cudaMemcpy(Lv.hv_cls, hcls.data(), sizeof(double) * hcls.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
                cudaMemcpy(dw, hw.data(), sizeof(double) * hw.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
                cudaMemcpy(dw + hw.size(), hc.data(), sizeof(double) * hc.size(), cudaMemcpyHostToDevice) != cudaSuccess)
                return bail(fail(MG_ECUDA, "heterogeneous Vanka table upload failed"));
            cudaMemset(Lv.hv_sinv, 0, sizeof(double) * MG_HV_NSINV * Lv.plane);
            if (launch_hv_sinv(Lv.vp.L, dw, dw + hw.size(), Lv.hv_sinv, 0) != cudaSuccess)
                return bail(fail(MG_ECUDA, "hv_sinv launch: %s", cudaGetErrorString(cudaGetLastError())));
            Lv.vp.hv = HetVankaTabs{Lv.hv_cls, Lv.hv_sinv};
        }
    }
    // norms and solve state
    c->partials = (double*)dalloc(c, sizeof(double) * max_blocks);
    c->counter = (unsigned*)dalloc(c, 64);
    c->norm = (double*)dalloc(c, 64);
    c->stop = (int*)dalloc(c, 64);
    c->state = (SolveState*)dalloc(c, sizeof(SolveState) + 64);
    if (!c->partials || !c->counter || !c->norm || !c->stop || !c->state)
        return bail(fail(MG_ENOMEM, "device allocation failed (norm buffers)"));
    cudaMemset(c->counter, 0, 64);
    cudaMemset(c->stop, 0, 64);
    for (int l = 0; l < levels; ++l) c->L[l].vp.L.stop = c->stop;
    if (cudaMallocHost(&c->pinned, (4 + 256) * sizeof(double)) != cudaSuccess) return bail(fail(MG_ENOMEM, "pinned alloc failed"));
    // coarsest dense deflated inverse (reading A9)
    if (dense_ok) {
        Level& Lc = c->L[levels - 1];
        int N = 0;
        host_coarse_inverse(Lc.n, Lc.pitch, c->m, nullptr, nullptr, nullptr, &N, err, sizeof(err));
        std::vector<double> G((size_t)N * N);
        std::vector<int64_t> sl(N);
        std::vector<double> kc;
        const double* kcp = nullptr;
        if (c->het) {
            std::vector<double> tmp(2 * Lc.plane);
            if (cudaDeviceSynchronize() != cudaSuccess ||
                cudaMemcpy(tmp.data(), Lc.kinv, sizeof(double) * 2 * Lc.plane, cudaMemcpyDeviceToHost) != cudaSuccess)
                return bail(fail(MG_ECUDA, "K^-1 download: %s", cudaGetErrorString(cudaGetLastError())));
            kc.resize(2 * (size_t)Lc.n * Lc.n);
            for (int sh = 0; sh < 2; ++sh)
                for (int j = 0; j < Lc.n; ++j)
                    for (int i = 0; i < Lc.n; ++i)
                        kc[((size_t)sh * Lc.n + j) * Lc.n + i] = tmp[sh * Lc.plane + (size_t)j * Lc.pitch + i];
            kcp = kc.data();
        }
        if (host_coarse_inverse(Lc.n, Lc.pitch, c->m, kcp, G.data(), sl.data(), &N, err, sizeof(err)))
            return bail(fail(MG_EINVAL, "coarsest level: %s", err));
        c->Nc = N;
        c->Ginv = (double*)dalloc(c, sizeof(double) * G.size());
        c->slots = (int64_t*)dalloc(c, sizeof(int64_t) * N);
        if (!c->Ginv || !c->slots) return bail(fail(MG_ENOMEM, "coarse allocation failed"));
        if (cudaMemcpy(c->Ginv, G.data(), sizeof(double) * G.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(c->slots, sl.data(), sizeof(int64_t) * N, cudaMemcpyHostToDevice) != cudaSuccess)
            return bail(fail(MG_ECUDA, "coarse upload failed"));
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return bail(fail(MG_ECUDA, "setup: %s", cudaGetErrorString(e)));
    *out = c;
    return MG_OK;
}

void mg_free(mg_ctx* c) {
    if (!c) return;
    cudaDeviceSynchronize();
    for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
    c->graphs.clear();
    for (int i = 0; i < 6; ++i)
        if (c->ev[i]) cudaEventDestroy(c->ev[i]);
    for (auto e : c->lev) cudaEventDestroy(e);
    dfree_all(c);
    if (c->pinned) cudaFreeHost(c->pinned);
    if (c->cap) cudaStreamDestroy(c->cap);
    delete c;
}

int mg_residual(mg_ctx* c, int32_t level, const double* x, const double* b, double* r, double* norm2_dev,
                cudaStream_t s) {
    if (int rc = check_level(c, level, c ? c->levels - 1 : 0)) return rc;
    if (!aligned(x) || !aligned(b) || (r && !aligned(r)) || (norm2_dev && !aligned(norm2_dev)))
        return fail(MG_EINVAL, "null or misaligned pointer");
    if (r && (r == x || r == b)) return fail(MG_EINVAL, "r must not alias x or b");
    NormSink S = norm2_dev ? NormSink{norm2_dev, c->partials, c->counter, nullptr} : no_norm();
    CK(launch_residual(c->L[level].vp.L, x, b, r, S, s));
    return MG_OK;
}

int mg_relax_vanka(mg_ctx* c, int32_t level, double* x, const double* b, double omega, int32_t sweeps,
                   cudaStream_t s) {
    if (int rc = check_level(c, level, c ? c->levels - 1 : 0)) return rc;
    if (!aligned(x) || !aligned(b)) return fail(MG_EINVAL, "null or misaligned pointer");
    if (sweeps < 0) return fail(MG_EINVAL, "sweeps < 0");
    mg_cycle_opts o{1, 1, MG_VANKA, omega, 0.0, 0};
    Level& Lv = c->L[level];
    double* a = x;
    double* t = Lv.t;
    for (int k = 0; k < sweeps; ++k) {
        if (int rc = relax_once(c, level, a, b, t, false, o, no_norm(), s)) return rc;
        std::swap(a, t);
    }
    if (a != x) CK(cudaMemcpyAsync(x, a, sizeof(double) * Lv.len, cudaMemcpyDeviceToDevice, s));
    return MG_OK;
}

int mg_relax_bsr(mg_ctx* c, int32_t level, double* x, const double* b, double omega, double omega_J,
                 int32_t jacobi_sweeps, int32_t sweeps, cudaStream_t s) {
    if (int rc = check_level(c, level, c ? c->levels - 1 : 0)) return rc;
    if (!aligned(x) || !aligned(b)) return fail(MG_EINVAL, "null or misaligned pointer");
    if (sweeps < 0 || jacobi_sweeps < 0) return fail(MG_EINVAL, "sweeps < 0");
    mg_cycle_opts o{1, 1, MG_BSR, omega, omega_J, jacobi_sweeps};
    if (int rc = ensure_rs(c)) return rc;
    Level& Lv = c->L[level];
    double* a = x;
    double* t = Lv.t;
    for (int k = 0; k < sweeps; ++k) {
        if (int rc = relax_once(c, level, a, b, t, false, o, no_norm(), s)) return rc;
        std::swap(a, t);
    }
    if (a != x) CK(cudaMemcpyAsync(x, a, sizeof(double) * Lv.len, cudaMemcpyDeviceToDevice, s));
    return MG_OK;
}

int mg_relax_bsr_exact(mg_ctx* c, int32_t level, double* x, const double* b, double omega, int32_t sweeps,
                       int32_t* cg_iters_out, cudaStream_t s) {
    if (int rc = check_level(c, level, c ? c->levels - 1 : 0)) return rc;
    if (!aligned(x) || !aligned(b)) return fail(MG_EINVAL, "null or misaligned pointer");
    if (sweeps < 0) return fail(MG_EINVAL, "sweeps < 0");
    mg_cycle_opts o{1, 1, MG_BSR_EXACT, omega, 0.0, 0};
    if (int rc = check_opts(c, &o)) return rc;
    Level& Lv = c->L[level];
    double* a = x;
    double* t = Lv.t;
    for (int k = 0; k < sweeps; ++k) {
        if (int rc = relax_once(c, level, a, b, t, false, o, no_norm(), s)) return rc;
        std::swap(a, t);
    }
    if (a != x) CK(cudaMemcpyAsync(x, a, sizeof(double) * Lv.len, cudaMemcpyDeviceToDevice, s));
    if (cg_iters_out && sweeps > 0) {   // iterations of the last S solve; MG_NOTCONV if it hit the cap
        double st[8];
        CK(cudaMemcpyAsync(st, c->cgst, sizeof(st), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        *cg_iters_out = (int32_t)st[6];
        if (st[5] == 0.0) return MG_NOTCONV;
    }
    return MG_OK;
}

int mg_restrict(mg_ctx* c, int32_t fl, const double* r, double* bc, cudaStream_t s) {
    if (int rc = check_level(c, fl, c ? c->levels - 2 : 0)) return rc;
    if (!aligned(r) || !aligned(bc)) return fail(MG_EINVAL, "null or misaligned pointer");
    CK(launch_restrict(c->L[fl].vp.L, c->L[fl + 1].n, c->L[fl + 1].pitch, 0, nullptr, r, bc, s));
    return MG_OK;
}

int mg_residual_restrict(mg_ctx* c, int32_t fl, const double* x, const double* b, double* bc, cudaStream_t s) {
    if (int rc = check_level(c, fl, c ? c->levels - 2 : 0)) return rc;
    if (!aligned(x) || !aligned(b) || !aligned(bc)) return fail(MG_EINVAL, "null or misaligned pointer");
    const Level& Lv = c->L[fl];
    // the cycle's own choice (enqueue_cycle): row-marching fused kernel on the big scalar-K RQ levels
    if (c->restrict_impl == 1 && Lv.n >= c->march_min_n && !c->exact)
        CK(launch_restrict_march(Lv.vp.L, c->L[fl + 1].n, c->L[fl + 1].pitch, x, b, bc, s));
    else
        CK(launch_restrict(Lv.vp.L, c->L[fl + 1].n, c->L[fl + 1].pitch, 1, x, b, bc, s));
    return MG_OK;
}

int mg_prolong_relax_vanka(mg_ctx* c, int32_t level, double* x, const double* e, const double* b, double omega,
                           cudaStream_t s) {
    if (int rc = check_level(c, level, c ? c->levels - 2 : 0)) return rc;
    if (!aligned(x) || !aligned(e) || !aligned(b)) return fail(MG_EINVAL, "null or misaligned pointer");
    mg_cycle_opts o{1, 1, MG_VANKA, omega, 0.0, 0};
    Level& Lv = c->L[level];
    if (fused_prolong(c, level, o)) {   // the cycle's fused kernel: x + P e relaxed in one pass
        if (int rc = relax_once(c, level, x, b, Lv.t, false, o, no_norm(), s, e)) return rc;
    } else {
        CK(launch_prolong(Lv.n, Lv.pitch, c->L[level + 1].n, c->L[level + 1].pitch, e, x, c->stop, s));
        if (int rc = relax_once(c, level, x, b, Lv.t, false, o, no_norm(), s)) return rc;
    }
    CK(cudaMemcpyAsync(x, Lv.t, sizeof(double) * Lv.len, cudaMemcpyDeviceToDevice, s));
    return MG_OK;
}

int mg_prolong(mg_ctx* c, int32_t fl, const double* e, double* xf, cudaStream_t s) {
    if (int rc = check_level(c, fl, c ? c->levels - 2 : 0)) return rc;
    if (!aligned(e) || !aligned(xf)) return fail(MG_EINVAL, "null or misaligned pointer");
    CK(launch_prolong(c->L[fl].n, c->L[fl].pitch, c->L[fl + 1].n, c->L[fl + 1].pitch, e, xf, c->stop, s));
    return MG_OK;
}

int mg_coarse_solve(mg_ctx* c, const double* b, double* x, cudaStream_t s) {
    if (!c) return fail(MG_EINVAL, "null context");
    if (!c->Ginv) return fail(MG_EINVAL, "no dense coarsest solve on this context (n_c > 20)");
    if (!aligned(b) || !aligned(x)) return fail(MG_EINVAL, "null or misaligned pointer");
    CK(cudaMemsetAsync(x, 0, sizeof(double) * c->L[c->levels - 1].len, s));
    CK(launch_coarse(c->Nc, c->Ginv, c->slots, b, x, c->stop, s));
    return MG_OK;
}

int mg_cycle(mg_ctx* c, double* x, const double* b, const mg_cycle_opts* o, double* res_norm_host, cudaStream_t s) {
    if (!c) return fail(MG_EINVAL, "null context");
    if (int rc = check_opts(c, o)) return rc;
    if (!aligned(x) || !aligned(b)) return fail(MG_EINVAL, "null or misaligned pointer");
    if (!c->Ginv) return fail(MG_EINVAL, "no dense coarsest solve on this context (n_c > 20)");
    if (c->levels == 1) {
        CK(launch_coarse(c->Nc, c->Ginv, c->slots, b, x, c->stop, s));
    } else {
        cudaGraphExec_t g;
        if (int rc = get_graph(c, x, b, *o, 0, nullptr, &g)) return rc;
        CK(cudaGraphLaunch(g, s));
        if (c->timing) c->timed_ran = true;
    }
    if (res_norm_host) {
        CK(launch_residual(c->L[0].vp.L, x, b, nullptr, NormSink{c->norm, c->partials, c->counter, nullptr}, s));
        CK(cudaMemcpyAsync(c->pinned, c->norm, sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        *res_norm_host = std::sqrt(c->pinned[0]);
    }
    return MG_OK;
}

int mg_cycle_async(mg_ctx* c, double* x, const double* b, const mg_cycle_opts* o, double* in_norm2_dev,
                   cudaStream_t s) {
    if (!c) return fail(MG_EINVAL, "null context");
    if (int rc = check_opts(c, o)) return rc;
    if (!aligned(x) || !aligned(b) || (in_norm2_dev && !aligned(in_norm2_dev)))
        return fail(MG_EINVAL, "null or misaligned pointer");
    if (!c->Ginv || c->levels < 2) return fail(MG_EINVAL, "mg_cycle_async needs levels >= 2 and a coarsest solve");
    cudaGraphExec_t g;
    if (int rc = get_graph(c, x, b, *o, in_norm2_dev ? 2 : 0, in_norm2_dev, &g)) return rc;
    CK(cudaGraphLaunch(g, s));
    if (c->timing) c->timed_ran = true;
    return MG_OK;
}

int32_t mg_cycle_kernels(const mg_ctx* c) { return c ? c->launches : -1; }

int mg_set_timing(mg_ctx* c, int32_t enable) {
    if (!c) return fail(MG_EINVAL, "null context");
    if (enable && !c->ev[0]) {
        for (int i = 0; i < 6; ++i) CK(cudaEventCreate(&c->ev[i]));
        c->lev.resize(4 * (c->levels - 1) + 2);
        for (auto& e : c->lev) CK(cudaEventCreate(&e));
    }
    c->timing = enable != 0;
    c->timed_ran = false;
    return MG_OK;
}

int mg_timing(mg_ctx* c, float* ms) {
    if (!c || !ms) return fail(MG_EINVAL, "null argument");
    if (!c->timed_ran || !c->ev[0]) return fail(MG_EINVAL, "no traced cycle ran");
    CK(cudaEventSynchronize(c->ev[5]));
    for (int i = 0; i < 5; ++i) CK(cudaEventElapsedTime(&ms[i], c->ev[i], c->ev[i + 1]));
    return MG_OK;
}

int mg_timing_levels(mg_ctx* c, float* ms, int32_t cap) {
    if (!c || !ms) return fail(MG_EINVAL, "null argument");
    if (!c->timed_ran || c->lev.empty()) return fail(MG_EINVAL, "no traced cycle ran");
    const int m = (int)c->lev.size() - 1;
    if (cap < m) return fail(MG_EINVAL, "cap %d < %d intervals", cap, m);
    CK(cudaEventSynchronize(c->lev.back()));
    for (int i = 0; i < m; ++i) CK(cudaEventElapsedTime(&ms[i], c->lev[i], c->lev[i + 1]));
    return m;
}

int mg_fgmres(mg_ctx* c, double* x, const double* b, const mg_cycle_opts* o, double rtol, int32_t max_iters,
              int32_t restart, double* history_host, int32_t* n_iters, cudaStream_t s) {
    if (!c) return fail(MG_EINVAL, "null context");
    if (int rc = check_opts(c, o)) return rc;
    if (!aligned(x) || !aligned(b)) return fail(MG_EINVAL, "null or misaligned pointer");
    if (max_iters < 0 || restart < 1 || restart > 31)
        return fail(MG_EINVAL, "need max_iters >= 0, 1 <= restart <= 31");
    if (!c->Ginv || c->levels < 2) return fail(MG_EINVAL, "mg_fgmres needs levels >= 2 and a coarsest solve");
    Level& L0 = c->L[0];
    const int64_t len = L0.len;
    const size_t vb = sizeof(double) * len;
    if (restart > c->kcap) {
        // zero-filled once: the kernels never write the padding / inactive slots, and the FGMRES dot
        // products run over whole padded vectors
        while ((int)c->kv.size() < restart + 1) {
            double* p = (double*)dalloc(c, vb);
            if (!p) return fail(MG_ENOMEM, "FGMRES basis allocation failed (restart %d)", restart);
            CK(cudaMemsetAsync(p, 0, vb, s));
            c->kv.push_back(p);
        }
        while ((int)c->kz.size() < restart) {
            double* p = (double*)dalloc(c, vb);
            if (!p) return fail(MG_ENOMEM, "FGMRES basis allocation failed (restart %d)", restart);
            CK(cudaMemsetAsync(p, 0, vb, s));
            c->kz.push_back(p);
        }
        c->kcap = restart;
    }
    if (!c->kw) {
        c->kw = (double*)dalloc(c, vb);
        c->kdots = (double*)dalloc(c, sizeof(double) * 256);
        c->kpart = (double*)dalloc(c, sizeof(double) * std::max(dot_partials_needed(), gs_partials_needed()));
        c->kcnt = (unsigned*)dalloc(c, 64);
        if (!c->kw || !c->kdots || !c->kpart || !c->kcnt) return fail(MG_ENOMEM, "FGMRES work allocation failed");
        CK(cudaMemsetAsync(c->kcnt, 0, 64, s));
        CK(cudaMemsetAsync(c->kw, 0, vb, s));
    }
    const LevelParams& LP = L0.vp.L;
    // Device scratch (doubles): [0, 33) pass-1 dots + |U|^2, [40, 73) pass-2 dots + |U'|^2, [80] |U''|^2,
    // [96, 128) s_i^2, [128, 160) solution-update coefficients, [160] |r|^2.
    double* hd = c->kdots;
    double* d1 = hd, * d2 = hd + 40, * d3 = hd + 80, * s2d = hd + 96, * yd = hd + 128, * rn = hd + 160;
    // Basis kept UNSCALED: W_i (kv[i]) with v_i = s_i W_i of unit norm; Z'_i = M^-1 W_i (kz[i]) so
    // z_i = s_i Z'_i; the scaling passes of textbook GMRES disappear into host-side bookkeeping.
    // Classical Gram-Schmidt twice, fused: pass 1 dots (mode 0); pass-1 update written to W_{j+1}
    // together with the pass-2 dots (mode 1); pass-2 update with the norm (mode 2).
    std::vector<double> hist, sv(restart + 2), hh(96);
    int iters = 0;
    double beta0 = -1.0, target = 0.0;
    bool done = false;
    std::vector<double> H, cs, sn, g;
    while (!done) {
        // r = b - A x -> W_0, |r|^2 fused into the residual kernel
        CK(launch_residual(LP, x, b, c->kv[0], NormSink{rn, c->partials, c->counter, nullptr}, s));
        CK(cudaMemcpyAsync(hh.data(), rn, sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const double beta = std::sqrt(hh[0]);
        if (beta0 < 0.0) {
            beta0 = beta;
            target = rtol * beta0;
            hist.push_back(beta);
        }
        if (!std::isfinite(beta)) return fail(MG_ECUDA, "non-finite residual in FGMRES");
        if (beta <= target || beta == 0.0 || iters >= max_iters) break;
        sv[0] = 1.0 / beta;
        hh[0] = sv[0] * sv[0];
        CK(cudaMemcpyAsync(s2d, hh.data(), sizeof(double), cudaMemcpyHostToDevice, s));
        const int m = std::min(restart, max_iters - iters);
        H.assign((m + 1) * m, 0.0);
        cs.assign(m, 0.0);
        sn.assign(m, 0.0);
        g.assign(m + 1, 0.0);
        g[0] = beta;
        int k = 0;
        for (int j = 0; j < m; ++j) {
            // Z'_j = one V-cycle from zero on W_j; U = A Z'_j
            cudaGraphExec_t ge;
            if (int rc = get_graph(c, c->kz[j], c->kv[j], *o, 3, nullptr, &ge)) return rc;
            CK(cudaGraphLaunch(ge, s));
            CK(launch_apply(LP, c->kz[j], c->kw, no_norm(), s));
            GsPtrs V{};
            for (int i = 0; i <= j; ++i) V.p[i] = c->kv[i];
            const int kk = j + 1;
            // coefficients of W_i: c_i = <U, W_i> s_i^2 (the kernels scale by s2d)
            CK(launch_gs(0, c->kw, nullptr, V, kk, nullptr, nullptr, len, c->kpart, c->kcnt, d1, s));
            CK(launch_gs(1, c->kw, c->kv[j + 1], V, kk, d1, s2d, len, c->kpart, c->kcnt, d2, s));
            bool two = c->cgs_passes == 2;
            bool have = false;   // hh already holds the dots of this iteration (no second pass followed)
            if (c->cgs_passes == 0) {
                // DGKS-type test: reorthogonalise only when the first pass cancelled U by more than 1 / eta
                // (|U'|^2 < eta^2 |U|^2); |U|^2 and |U'|^2 come with the two passes' dot products
                CK(cudaMemcpyAsync(hh.data(), hd, sizeof(double) * 81, cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                two = hh[40 + kk] < c->dgks_eta2 * hh[kk];
                have = !two;
            }
            if (two) CK(launch_gs(2, c->kv[j + 1], c->kv[j + 1], V, kk, d2, s2d, len, c->kpart, c->kcnt, d3, s));
            if (!have) {
                CK(cudaMemcpyAsync(hh.data(), hd, sizeof(double) * 81, cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
            }
            const double rho = std::sqrt(two ? hh[80] : hh[40 + kk]);
            // h_ij = (A z_j) . v_i = s_j s_i <U, W_i> = s_j (c1_i + c2_i) / s_i
            for (int i = 0; i <= j; ++i)
                H[i * m + j] = sv[j] * sv[i] * (hh[i] + (two ? hh[40 + i] : 0.0));
            H[(j + 1) * m + j] = sv[j] * rho;
            sv[j + 1] = rho > 0.0 ? 1.0 / rho : 0.0;
            // one pinned slot per basis index: no synchronisation needed before the next iteration reuses hh
            c->pinned[4 + 128 + j + 1] = sv[j + 1] * sv[j + 1];
            CK(cudaMemcpyAsync(s2d + j + 1, c->pinned + 4 + 128 + j + 1, sizeof(double), cudaMemcpyHostToDevice, s));
            for (int i = 0; i < j; ++i) {   // previous Givens rotations
                const double t = cs[i] * H[i * m + j] + sn[i] * H[(i + 1) * m + j];
                H[(i + 1) * m + j] = -sn[i] * H[i * m + j] + cs[i] * H[(i + 1) * m + j];
                H[i * m + j] = t;
            }
            const double d = std::hypot(H[j * m + j], H[(j + 1) * m + j]);
            cs[j] = H[j * m + j] / d;
            sn[j] = H[(j + 1) * m + j] / d;
            H[j * m + j] = d;
            H[(j + 1) * m + j] = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            k = j + 1;
            ++iters;
            hist.push_back(std::fabs(g[j + 1]));
            if (!std::isfinite(hist.back())) return fail(MG_ECUDA, "non-finite FGMRES residual estimate");
            if (hist.back() <= target) break;
        }
        // y = H^{-1} g (upper triangular), x += sum_i y_i z_i = sum_i (y_i s_i) Z'_i in one pass
        std::vector<double> y(k);
        for (int i = k - 1; i >= 0; --i) {
            double t = g[i];
            for (int l = i + 1; l < k; ++l) t -= H[i * m + l] * y[l];
            y[i] = t / H[i * m + i];
        }
        for (int i = 0; i < k; ++i) y[i] = -y[i] * sv[i];   // the update kernel subtracts
        CK(cudaMemcpyAsync(yd, y.data(), sizeof(double) * k, cudaMemcpyHostToDevice, s));
        GsPtrs Z{};
        for (int i = 0; i < k; ++i) Z.p[i] = c->kz[i];
        CK(launch_gs(3, x, x, Z, k, yd, nullptr, len, nullptr, nullptr, nullptr, s));
        CK(cudaStreamSynchronize(s));   // y is host memory read by the async copy
        if (hist.back() <= target || iters >= max_iters) done = true;
    }
    CK(cudaStreamSynchronize(s));
    const int nh = (int)hist.size();
    if (history_host)
        for (int i = 0; i < nh; ++i) history_host[i] = hist[i];
    if (n_iters) *n_iters = nh - 1;
    return hist.back() <= target ? MG_OK : MG_NOTCONV;
}

int mg_step_rhs(mg_ctx* c, const double* x_prev, const double* b_load, double* b_out, cudaStream_t s) {
    if (!c) return fail(MG_EINVAL, "null context");
    if (!aligned(x_prev) || !aligned(b_load) || !aligned(b_out)) return fail(MG_EINVAL, "null or misaligned pointer");
    if (b_out == x_prev) return fail(MG_EINVAL, "b_out must not alias x_prev");
    const Level& L0 = c->L[0];
    if (b_out != b_load) CK(cudaMemcpyAsync(b_out, b_load, sizeof(double) * L0.len, cudaMemcpyDeviceToDevice, s));
    CK(launch_step_rhs(L0.vp.L, c->m.inv_M, c->m.alpha, x_prev, b_out, s));
    return MG_OK;
}

int mg_time_step(mg_ctx* c, double* x, const double* b_load, const mg_cycle_opts* o, double rtol, int32_t max_iters,
                 int32_t restart, double* history_host, int32_t* n_iters, cudaStream_t s) {
    if (!c) return fail(MG_EINVAL, "null context");
    if (!aligned(x) || !aligned(b_load)) return fail(MG_EINVAL, "null or misaligned pointer");
    if (!c->kb) {
        c->kb = (double*)dalloc(c, sizeof(double) * c->L[0].len);
        if (!c->kb) return fail(MG_ENOMEM, "time-step right-hand side allocation failed");
    }
    if (int rc = mg_step_rhs(c, x, b_load, c->kb, s)) return rc;
    return mg_fgmres(c, x, c->kb, o, rtol, max_iters, restart, history_host, n_iters, s);
}

int mg_solve(mg_ctx* c, double* x, const double* b, const mg_cycle_opts* o, double rtol, int32_t max_cycles,
             double* history_host, int32_t* n_cycles, cudaStream_t s) {
    if (!c) return fail(MG_EINVAL, "null context");
    if (int rc = check_opts(c, o)) return rc;
    if (!aligned(x) || !aligned(b)) return fail(MG_EINVAL, "null or misaligned pointer");
    if (max_cycles < 0) return fail(MG_EINVAL, "max_cycles < 0");
    if (c->levels == 1) return fail(MG_EINVAL, "mg_solve needs levels >= 2");
    if (!c->Ginv) return fail(MG_EINVAL, "no dense coarsest solve on this context (n_c > 20)");
    if (max_cycles + 1 > c->hist_cap) {
        int cap = std::max(256, max_cycles + 1);
        double* h = (double*)dalloc(c, sizeof(double) * cap);
        if (!h) return fail(MG_ENOMEM, "history allocation failed");
        c->hist = h;
        c->hist_cap = cap;
    }
    SolveState st{0, max_cycles, rtol * rtol, c->hist, c->stop};
    // whatever path leaves this function, the stop flag is cleared: a flag left raised would make
    // every later kernel on the context return at entry
    struct StopGuard {
        mg_ctx* c;
        cudaStream_t s;
        ~StopGuard() {
            cudaMemsetAsync(c->stop, 0, sizeof(int), s);
            cudaStreamSynchronize(s);
        }
    } guard{c, s};
    CK(cudaMemcpyAsync(c->state, &st, sizeof(st), cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(c->stop, 0, sizeof(int), s));
    cudaGraphExec_t g;
    if (int rc = get_graph(c, x, b, *o, 1, nullptr, &g)) return rc;
    int launched = 0, stop = 0, k = 0;
    const int batch = 4;
    while (launched < max_cycles + 1) {
        int nb = std::min(batch, max_cycles + 1 - launched);
        for (int i = 0; i < nb; ++i) CK(cudaGraphLaunch(g, s));
        launched += nb;
        CK(cudaMemcpyAsync(c->pinned, c->stop, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(c->pinned + 1, c->state, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        memcpy(&stop, c->pinned, sizeof(int));
        memcpy(&k, c->pinned + 1, sizeof(int));
        if (stop) break;
    }
    if (!stop) return fail(MG_ECUDA, "solve state inconsistent (no stop after %d launches)", launched);
    std::vector<double> h(k);
    CK(cudaMemcpy(h.data(), c->hist, sizeof(double) * k, cudaMemcpyDeviceToHost));
    if (history_host)
        for (int i = 0; i < k; ++i) history_host[i] = std::sqrt(h[i]);
    if (n_cycles) *n_cycles = k - 1;
    if (stop == 1) return MG_OK;
    if (stop == 2) return MG_DIVERGED;
    return MG_NOTCONV;
}

int mg_solve_host(mg_ctx* c, double* x_host, const double* b_host, const mg_cycle_opts* o, double rtol,
                  int32_t max_cycles, double* history_host, int32_t* n_cycles, cudaStream_t s) {
    if (!c) return fail(MG_EINVAL, "null context");
    if (!x_host || !b_host) return fail(MG_EINVAL, "null host pointer");
    Level& L0 = c->L[0];
    if (!c->hx) {
        c->hx = (double*)dalloc(c, sizeof(double) * L0.len);
        c->hb = (double*)dalloc(c, sizeof(double) * L0.len);
        if (!c->hx || !c->hb) return fail(MG_ENOMEM, "device allocation failed (e2e buffers)");
        CK(cudaMemset(c->hx, 0, sizeof(double) * L0.len));
        CK(cudaMemset(c->hb, 0, sizeof(double) * L0.len));
    }
    const size_t w = sizeof(double) * (L0.n + 1), dp = sizeof(double) * L0.pitch;
    const size_t rows = 10 * (size_t)(L0.n + 1);
    CK(cudaMemcpy2DAsync(c->hb, dp, b_host, w, w, rows, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpy2DAsync(c->hx, dp, x_host, w, w, rows, cudaMemcpyHostToDevice, s));
    int rc = mg_solve(c, c->hx, c->hb, o, rtol, max_cycles, history_host, n_cycles, s);
    if (rc < 0) return rc;
    CK(cudaMemcpy2DAsync(x_host, w, c->hx, dp, w, rows, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return rc;
}

}  // extern "C"

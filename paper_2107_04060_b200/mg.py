"""Thin Python binding of libmg.so (include/mg.h): argument marshalling only.

Every step of the multigrid path runs in the CUDA kernels of libmg.so; this module converts
torch tensors to device pointers and stream handles and raises on error codes.  PyTorch is
used for device memory (the context's own buffers come from torch's caching allocator through
mg_set_allocator) and streams.  There is no CPU fallback: if libmg.so is missing or no CUDA
device is present, calls fail loudly.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmg.so")

MG_OK, MG_NOTCONV, MG_DIVERGED = 0, 1, 2
MG_VANKA, MG_BSR, MG_BSR_EXACT = 0, 1, 2
MG_RQ, MG_EXACT = 0, 1
_RELAX = {"vanka": MG_VANKA, "bsr": MG_BSR, "bsr_exact": MG_BSR_EXACT}

_lib = None
_alloc_cbs = None

_D = ctypes.POINTER(ctypes.c_double)
_VP = ctypes.c_void_p


class MGError(RuntimeError):
    pass


class Grid(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("K_field", _VP), ("inv_M", ctypes.c_double), ("mu_f", ctypes.c_double),
                ("quadrature", ctypes.c_int32)]


class CycleOpts(ctypes.Structure):
    _fields_ = [("nu1", ctypes.c_int32), ("nu2", ctypes.c_int32), ("relax", ctypes.c_int32),
                ("omega", ctypes.c_double), ("omega_J", ctypes.c_double), ("jacobi_sweeps", ctypes.c_int32)]


# every symbol include/mg.h declares, with its ctypes signature
SIGNATURES = {
    "mg_set_allocator": (None, [_VP, _VP, _VP]),
    "mg_setup": (ctypes.c_int, [ctypes.POINTER(Grid), ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                ctypes.c_double, ctypes.c_double, ctypes.c_int32, ctypes.POINTER(_VP)]),
    "mg_free": (None, [_VP]),
    "mg_levels": (ctypes.c_int32, [_VP]),
    "mg_level_n": (ctypes.c_int32, [_VP, ctypes.c_int32]),
    "mg_pitch": (ctypes.c_int32, [_VP, ctypes.c_int32]),
    "mg_vec_len": (ctypes.c_int64, [_VP, ctypes.c_int32]),
    "mg_n_active": (ctypes.c_int64, [_VP, ctypes.c_int32]),
    "mg_residual": (ctypes.c_int, [_VP, ctypes.c_int32, _VP, _VP, _VP, _VP, _VP]),
    "mg_relax_vanka": (ctypes.c_int, [_VP, ctypes.c_int32, _VP, _VP, ctypes.c_double, ctypes.c_int32, _VP]),
    "mg_relax_bsr": (ctypes.c_int, [_VP, ctypes.c_int32, _VP, _VP, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_int32, ctypes.c_int32, _VP]),
    "mg_relax_bsr_exact": (ctypes.c_int, [_VP, ctypes.c_int32, _VP, _VP, ctypes.c_double, ctypes.c_int32,
                                          ctypes.POINTER(ctypes.c_int32), _VP]),
    "mg_restrict": (ctypes.c_int, [_VP, ctypes.c_int32, _VP, _VP, _VP]),
    "mg_prolong": (ctypes.c_int, [_VP, ctypes.c_int32, _VP, _VP, _VP]),
    "mg_residual_restrict": (ctypes.c_int, [_VP, ctypes.c_int32, _VP, _VP, _VP, _VP]),
    "mg_prolong_relax_vanka": (ctypes.c_int, [_VP, ctypes.c_int32, _VP, _VP, _VP, ctypes.c_double, _VP]),
    "mg_coarse_solve": (ctypes.c_int, [_VP, _VP, _VP, _VP]),
    "mg_cycle": (ctypes.c_int, [_VP, _VP, _VP, ctypes.POINTER(CycleOpts), _D, _VP]),
    "mg_solve": (ctypes.c_int, [_VP, _VP, _VP, ctypes.POINTER(CycleOpts), ctypes.c_double, ctypes.c_int32,
                                _D, ctypes.POINTER(ctypes.c_int32), _VP]),
    "mg_fgmres": (ctypes.c_int, [_VP, _VP, _VP, ctypes.POINTER(CycleOpts), ctypes.c_double, ctypes.c_int32,
                                 ctypes.c_int32, _D, ctypes.POINTER(ctypes.c_int32), _VP]),
    "mg_step_rhs": (ctypes.c_int, [_VP, _VP, _VP, _VP, _VP]),
    "mg_time_step": (ctypes.c_int, [_VP, _VP, _VP, ctypes.POINTER(CycleOpts), ctypes.c_double, ctypes.c_int32,
                                    ctypes.c_int32, _D, ctypes.POINTER(ctypes.c_int32), _VP]),
    "mg_solve_host": (ctypes.c_int, [_VP, _VP, _VP, ctypes.POINTER(CycleOpts), ctypes.c_double, ctypes.c_int32,
                                     _D, ctypes.POINTER(ctypes.c_int32), _VP]),
    "mg_cycle_async": (ctypes.c_int, [_VP, _VP, _VP, ctypes.POINTER(CycleOpts), _VP, _VP]),
    "mg_set_timing": (ctypes.c_int, [_VP, ctypes.c_int32]),
    "mg_cycle_kernels": (ctypes.c_int32, [_VP]),
    "mg_timing": (ctypes.c_int, [_VP, ctypes.POINTER(ctypes.c_float)]),
    "mg_timing_levels": (ctypes.c_int, [_VP, ctypes.POINTER(ctypes.c_float), ctypes.c_int32]),
    "mg_last_error": (ctypes.c_char_p, []),
    "mg_host_level_tables": (ctypes.c_int, [ctypes.c_int32] + [ctypes.c_double] * 7 + [_D] * 4),
}


def load_library(path: str = LIB_PATH):
    """Load libmg.so and declare the C ABI.  Raises if the library is missing (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with paper_2107_04060_b200.build.build() "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(rc: int, what: str):
    if rc < 0:
        raise MGError(f"{what} failed ({rc}): {load_library().mg_last_error().decode()}")
    return rc


def _install_torch_allocator(lib):
    """Route the context's device buffers through torch's caching allocator."""
    global _alloc_cbs
    if _alloc_cbs is not None:
        return
    import torch

    ALLOC = ctypes.CFUNCTYPE(_VP, ctypes.c_size_t, _VP)
    FREE = ctypes.CFUNCTYPE(None, _VP, _VP)

    def _a(nbytes, _user):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), torch.cuda.current_device())
        except Exception:
            return None

    def _f(ptr, _user):
        try:
            if ptr:
                torch.cuda.caching_allocator_delete(ptr)
        except Exception:      # interpreter shutdown: torch already torn down, memory goes with the process
            pass

    _alloc_cbs = (ALLOC(_a), FREE(_f))
    lib.mg_set_allocator(ctypes.cast(_alloc_cbs[0], _VP), ctypes.cast(_alloc_cbs[1], _VP), None)


def _ptr(t, numel=None):
    """Device pointer of a CUDA float64 tensor; numel: the element count the C call will touch
    (mg_vec_len of the level), checked so that a short or strided tensor never reaches a kernel."""
    if t is None:
        return None
    import torch
    if not t.is_cuda or t.dtype != torch.float64:
        raise MGError("expected a CUDA float64 tensor")
    if not t.is_contiguous():
        raise MGError("expected a contiguous tensor (the C ABI takes plain pointers)")
    if numel is not None and t.numel() != numel:
        raise MGError(f"tensor has {t.numel()} elements, the level vector has {numel} (10 x (n_l+1) x pitch_l)")
    if t.data_ptr() % 16:
        raise MGError("tensor storage is not 16-byte aligned")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


@dataclass
class Opts:
    """V(nu1, nu2) cycle options (mg_cycle_opts)."""
    nu1: int = 1
    nu2: int = 1
    relax: str = "vanka"        # "vanka" | "bsr" | "bsr_exact"
    omega: float = 0.74
    omega_J: float = 1.0
    jacobi_sweeps: int = 3

    def c(self) -> CycleOpts:
        return CycleOpts(self.nu1, self.nu2, _RELAX[self.relax],
                         float(self.omega), float(self.omega_J), int(self.jacobi_sweeps))


class Hierarchy:
    """An mg_ctx: the level hierarchy of one problem (mg_setup / mg_free)."""

    def __init__(self, n: int, levels: int, lam: float, mu: float, K: float = 1.0, tau: float = 1.0,
                 alpha: float = 1.0, inv_M: float = 1.0, mu_f: float = 1.0, K_field=None, quadrature: str = "rq"):
        import torch
        if not torch.cuda.is_available():
            raise MGError("no CUDA device: the multigrid path runs only on the GPU")
        self.lib = load_library()
        _install_torch_allocator(self.lib)
        self._kf = None
        kf = None
        if K_field is not None:
            self._kf = torch.as_tensor(K_field, dtype=torch.float64, device="cuda").contiguous()
            assert self._kf.shape == (2, n, n)
            kf = self._kf.data_ptr()
        grid = Grid(int(n), kf, float(inv_M), float(mu_f), {"rq": MG_RQ, "exact": MG_EXACT}[quadrature])
        ctx = _VP()
        _check(self.lib.mg_setup(ctypes.byref(grid), float(lam), float(mu), float(K), float(tau), float(alpha),
                                 int(levels), ctypes.byref(ctx)), "mg_setup")
        self.ctx = ctx
        self.n, self.levels = n, levels

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.mg_free(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- layout helpers (marshalling only) -------------------------------------------------
    def vec_len(self, level: int) -> int:
        return self.lib.mg_vec_len(self.ctx, level)

    def _v(self, t, level: int = 0):
        return _ptr(t, self.vec_len(level))

    def level_n(self, level: int) -> int:
        return self.lib.mg_level_n(self.ctx, level)

    def pitch(self, level: int) -> int:
        return self.lib.mg_pitch(self.ctx, level)

    def n_active(self, level: int = 0) -> int:
        return self.lib.mg_n_active(self.ctx, level)

    def zeros(self, level: int = 0):
        import torch
        nl = self.level_n(level)
        return torch.zeros((10, nl + 1, self.pitch(level)), dtype=torch.float64, device="cuda")

    def to_device(self, arr, level: int = 0):
        """(10, n_l+1, n_l+1) array -> padded device vector."""
        import torch
        v = self.zeros(level)
        nl = self.level_n(level)
        v[:, :, : nl + 1] = torch.as_tensor(np.asarray(arr, dtype=np.float64).reshape(10, nl + 1, nl + 1))
        return v

    def to_host(self, v, level: int = 0) -> np.ndarray:
        nl = self.level_n(level)
        return v[:, :, : nl + 1].cpu().numpy().copy()

    # ---- the C ABI ----------------------------------------------------------------------------
    def residual(self, level, x, b, r=None, norm=False, stream=None):
        import torch
        nd = torch.zeros(1, dtype=torch.float64, device="cuda") if norm else None
        _check(self.lib.mg_residual(self.ctx, level, self._v(x, level), self._v(b, level), self._v(r, level), _ptr(nd, 1), _stream(stream)),
               "mg_residual")
        return float(nd.sqrt().item()) if norm else None

    def relax_vanka(self, level, x, b, omega, sweeps=1, stream=None):
        _check(self.lib.mg_relax_vanka(self.ctx, level, self._v(x, level), self._v(b, level), float(omega), int(sweeps),
                                       _stream(stream)), "mg_relax_vanka")

    def relax_bsr(self, level, x, b, omega, omega_J, jacobi_sweeps, sweeps=1, stream=None):
        _check(self.lib.mg_relax_bsr(self.ctx, level, self._v(x, level), self._v(b, level), float(omega), float(omega_J),
                                     int(jacobi_sweeps), int(sweeps), _stream(stream)), "mg_relax_bsr")

    def relax_bsr_exact(self, level, x, b, omega, sweeps=1, stream=None):
        """Exact BSR sweeps; returns (rc, CG iterations of the last S solve)."""
        its = ctypes.c_int32(0)
        rc = _check(self.lib.mg_relax_bsr_exact(self.ctx, level, self._v(x, level), self._v(b, level), float(omega),
                                                int(sweeps), ctypes.byref(its), _stream(stream)), "mg_relax_bsr_exact")
        return rc, its.value

    def restrict(self, fine_level, r, bc, stream=None):
        _check(self.lib.mg_restrict(self.ctx, fine_level, self._v(r, fine_level), self._v(bc, fine_level + 1), _stream(stream)), "mg_restrict")

    def prolong(self, fine_level, e, xf, stream=None):
        _check(self.lib.mg_prolong(self.ctx, fine_level, self._v(e, fine_level + 1), self._v(xf, fine_level), _stream(stream)), "mg_prolong")

    def residual_restrict(self, fine_level, x, b, bc, stream=None):
        """b_coarse = P^T (b - A x), the cycle's fused production kernel."""
        _check(self.lib.mg_residual_restrict(self.ctx, fine_level, self._v(x, fine_level), self._v(b, fine_level),
                                             self._v(bc, fine_level + 1), _stream(stream)), "mg_residual_restrict")

    def prolong_relax_vanka(self, level, x, e, b, omega, stream=None):
        """x <- one Vanka sweep of x + P e (the cycle's fused post-sweep), in place."""
        _check(self.lib.mg_prolong_relax_vanka(self.ctx, level, self._v(x, level), self._v(e, level + 1),
                                               self._v(b, level), float(omega), _stream(stream)),
               "mg_prolong_relax_vanka")

    def coarse_solve(self, b, x, stream=None):
        _check(self.lib.mg_coarse_solve(self.ctx, self._v(b, self.levels - 1), self._v(x, self.levels - 1), _stream(stream)), "mg_coarse_solve")

    def cycle(self, x, b, opts: Opts, norm=True, stream=None):
        out = ctypes.c_double(0.0)
        o = opts.c()
        _check(self.lib.mg_cycle(self.ctx, self._v(x), self._v(b), ctypes.byref(o), ctypes.byref(out) if norm else None,
                                 _stream(stream)), "mg_cycle")
        return out.value if norm else None

    def cycle_async(self, x, b, opts: Opts, norm2_out=None, stream=None):
        """One cycle, no host sync; norm2_out: optional 1-element CUDA tensor receiving ||b - A x_in||^2."""
        o = opts.c()
        _check(self.lib.mg_cycle_async(self.ctx, self._v(x), self._v(b), ctypes.byref(o), _ptr(norm2_out, None if norm2_out is None else norm2_out.numel()),
                                       _stream(stream)), "mg_cycle_async")

    def cycle_kernels(self) -> int:
        """Kernel launches per cycle of the last captured cycle graph."""
        return self.lib.mg_cycle_kernels(self.ctx)

    def set_timing(self, enable: bool):
        _check(self.lib.mg_set_timing(self.ctx, 1 if enable else 0), "mg_set_timing")

    def timing(self):
        """Elapsed ms of the latest traced cycle: (pre, restrict, coarse levels, prolong, post)."""
        out = (ctypes.c_float * 5)()
        _check(self.lib.mg_timing(self.ctx, out), "mg_timing")
        return list(out)

    def timing_levels(self):
        """Per-level ms of the latest traced cycle: dict(pre=[...], restrict=[...], coarse=..,
        prolong=[...], post=[...]) indexed by level."""
        cap = 4 * self.levels
        out = (ctypes.c_float * cap)()
        m = _check(self.lib.mg_timing_levels(self.ctx, out, cap), "mg_timing_levels")
        v = list(out)[:m]
        L1 = self.levels - 1
        pre = [v[2 * l] for l in range(L1)]
        res = [v[2 * l + 1] for l in range(L1)]
        coarse = v[2 * L1]
        tail = v[2 * L1 + 1:]
        pro = [0.0] * L1
        post = [0.0] * L1
        for k, l in enumerate(range(L1 - 1, -1, -1)):
            pro[l], post[l] = tail[2 * k], tail[2 * k + 1]
        return dict(pre=pre, restrict=res, coarse=coarse, prolong=pro, post=post)

    def solve(self, x, b, opts: Opts, rtol=1e-8, max_cycles=100, stream=None):
        hist = np.zeros(max_cycles + 1)
        nc = ctypes.c_int32(0)
        o = opts.c()
        rc = _check(self.lib.mg_solve(self.ctx, self._v(x), self._v(b), ctypes.byref(o), float(rtol), int(max_cycles),
                                      hist.ctypes.data_as(_D), ctypes.byref(nc), _stream(stream)), "mg_solve")
        return rc, hist[: nc.value + 1]

    def fgmres(self, x, b, opts: Opts, rtol=1e-6, max_iters=100, restart=20, stream=None):
        """FGMRES preconditioned by one V-cycle per iteration; returns (rc, history)."""
        hist = np.zeros(max_iters + 1)
        nc = ctypes.c_int32(0)
        o = opts.c()
        rc = _check(self.lib.mg_fgmres(self.ctx, self._v(x), self._v(b), ctypes.byref(o), float(rtol), int(max_iters),
                                       int(restart), hist.ctypes.data_as(_D), ctypes.byref(nc), _stream(stream)),
                    "mg_fgmres")
        return rc, hist[: nc.value + 1]

    def step_rhs(self, x_prev, b_load, b_out, stream=None):
        """b_out = b_load + backward-Euler history of x_prev (mg_step_rhs)."""
        _check(self.lib.mg_step_rhs(self.ctx, self._v(x_prev), self._v(b_load), self._v(b_out), _stream(stream)),
               "mg_step_rhs")

    def time_step(self, x, b_load, opts: Opts, rtol=1e-10, max_iters=100, restart=30, stream=None):
        """One backward-Euler step in place on x (x^{m-1} -> x^m): mg_time_step; returns (rc, history)."""
        hist = np.zeros(max_iters + 1)
        nc = ctypes.c_int32(0)
        o = opts.c()
        rc = _check(self.lib.mg_time_step(self.ctx, self._v(x), self._v(b_load), ctypes.byref(o), float(rtol),
                                          int(max_iters), int(restart), hist.ctypes.data_as(_D), ctypes.byref(nc),
                                          _stream(stream)), "mg_time_step")
        return rc, hist[: nc.value + 1]

    def solve_host(self, x_host: np.ndarray, b_host: np.ndarray, opts: Opts, rtol=1e-8, max_cycles=100,
                   stream=None):
        """End-to-end solve from host arrays (10, n+1, n+1); x_host is overwritten with the solution."""
        shape = (10, self.n + 1, self.n + 1)
        for a in (x_host, b_host):
            if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous and a.shape == shape):
                raise MGError(f"host vectors must be C-contiguous float64 arrays of shape {shape}")
        hist = np.zeros(max_cycles + 1)
        nc = ctypes.c_int32(0)
        o = opts.c()
        rc = _check(self.lib.mg_solve_host(self.ctx, x_host.ctypes.data_as(_VP), b_host.ctypes.data_as(_VP),
                                           ctypes.byref(o), float(rtol), int(max_cycles), hist.ctypes.data_as(_D),
                                           ctypes.byref(nc), _stream(stream)), "mg_solve_host")
        return rc, hist[: nc.value + 1]


def host_level_tables(n, lam, mu, K, tau, alpha, inv_M, mu_f=1.0):
    """mg_host_level_tables (no GPU needed): stencil coefficients, M_w entries, Vanka and
    displacement patch inverses of one level."""
    lib = load_library()
    coef = np.zeros(141)
    ww = np.zeros(18)
    van = np.zeros(9 * 400)
    disp = np.zeros(9 * 64)
    p = lambda a: a.ctypes.data_as(_D)
    _check(lib.mg_host_level_tables(int(n), lam, mu, K, tau, alpha, inv_M, mu_f, p(coef), p(ww), p(van), p(disp)),
           "mg_host_level_tables")
    return dict(coef=coef, ww=ww.reshape(2, 3, 3), vanka=van.reshape(9, 20, 20), disp=disp.reshape(9, 8, 8))

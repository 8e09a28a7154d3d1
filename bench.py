#!/usr/bin/env python
"""Benchmark of the B200 monolithic multigrid hot path (BASELINE.json metric).

A step is one V(1,1) cycle of the whole hot path (residual, additive Vanka or
inexact Braess-Sarazin relaxation, divergence-preserving restriction / prolongation, coarsest
solve, fused residual norm) on the BASELINE workload, default config 5: 4096^2 cells, 11 levels,
lambda = 100, mu = 1, K = 1e-2, tau = alpha = 1, 1/M = 1, b ~ U(-1,1) from seed 5, x0 = 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

* value: DoF-updates/s = active unknowns of level 0 x cycles (x ranks) / max-over-ranks device time
  of the K timed cycles (CUDA events on the launching stream, inputs resident in HBM).
* e2e: the same metric through the public C-ABI call with HOST buffers (mg_solve_host: pinned host
  b and x copied in, K cycles, x copied back) timed by wall clock.
* roofline: the dominant kernel (level-0 Vanka sweep: warp-marching kernel + its boundary-vertex
  kernel, 2 sweeps per cycle) -- algorithmic bytes
  (24 B per active DoF: read x, read b, write x) / its CUDA-event duration, against the measured
  HBM copy bandwidth of MEASURED_PEAKS.json.
* cpu_baseline / --impl reference: the CPU oracle (oracle/, test infrastructure) timed as it
  stands on a bounded sample of the same workload (same parameters and RHS recipe on a smaller
  grid, since the oracle cannot hold the 4096^2 operator).
Multi-GPU (torchrun): every rank solves its own copy of the problem (independent problems, no
data-path collective; weak scaling); barrier + max-over-ranks timing.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import mg_inputs  # noqa: E402

REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


def max_over_ranks(value: float, dist=None) -> float:
    """Max of a per-rank timing over all ranks (all_reduce MAX; CUDA tensor under NCCL, CPU under gloo)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_rate(units_per_rank: float, steps: int, world: int, ms_max: float) -> float:
    """Whole-job throughput: the units all ranks processed (independent replicas: weak scaling)
    divided by the slowest rank's time."""
    return units_per_rank * steps * world / (ms_max * 1e-3)


def workload(cfg_id: int):
    c = dict(mg_inputs.CONFIGS[cfg_id])
    relax = "bsr" if c["relax"] == "bsr" else "vanka"
    c["relax_used"] = relax
    return c


def opts_for(c):
    from paper_2107_04060_b200 import Opts
    if c["relax_used"] == "vanka":
        return Opts(1, 1, "vanka", c.get("omega", 0.74))
    if c["relax_used"] == "bsr_exact":
        return Opts(1, 1, "bsr_exact", c.get("bsr_omega", 0.75), 1.0, 0)
    return Opts(1, 1, "bsr", c["bsr_omega"], c["omega_J"], 3)


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    def __init__(self, dev: int):
        self.dev = dev
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        for ln in self.lines:
            try:
                a, b, r = [p.strip() for p in ln.split(",")]
                sm.append(float(a))
                mx = max(mx, float(b))
                bits = int(r, 16)
                for k, v in REASONS.items():
                    if bits & k and v != "gpu_idle":
                        reasons.add(v)
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def oracle_sample(c, cycles: int, warmup: int = 1, n_sample: int = 128):
    """Time the oracle V(1,1) cycle on an n_sample^2 grid (the workload itself when smaller) with the
    workload's parameters."""
    from oracle.cycle import Hierarchy as OH
    n_sample = min(n_sample, c["n"])
    levels = max(2, int(np.log2(n_sample // 4)) + 1)
    kinv = None if c["K_seed"] is None else 1.0 / mg_inputs.lognormal_K(n_sample, c["K_seed"])
    H = OH(n_sample, levels, c["lam"], c["mu"], c["tau"], c["alpha"], c["inv_M"], c["mu_f"],
           K=c["K"] if c["K"] is not None else 1.0, Kinv_field=kinv, relax=c["relax_used"])
    b = H.meshes[0].to_active(mg_inputs.uniform_rhs(n_sample, c["b_seed"]))
    o = opts_for(c)
    od = dict(nu1=1, nu2=1, omega=o.omega, omega_J=o.omega_J, jacobi_sweeps=o.jacobi_sweeps)
    x = np.zeros_like(b)
    for _ in range(warmup):
        x = H.cycle(x, b, od)
    times = []
    for _ in range(cycles):
        t = time.perf_counter()
        x = H.cycle(x, b, od)
        times.append(time.perf_counter() - t)
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        cores = 1
    nact = mg_inputs.n_active(n_sample)
    return dict(value=nact * len(times) / sum(times), ms=1e3 * sum(times) / len(times), cores=cores,
                n=n_sample, levels=levels,
                sample=f"oracle V(1,1) on {n_sample}^2 ({levels} levels, {nact} active DoFs), same parameters and "
                       f"RHS recipe, {len(times)} cycles after {warmup} warm-up; host has {os.cpu_count()} cores, "
                       f"numpy/scipy (sparse matvec single-threaded, BLAS threads {cores})")


METRIC = "DoF-updates/s per V(1,1) cycle (fp64) at 4096^2; ms per cycle; % of HBM roofline"


def workload_config(args, c):
    """The workload description shared by both arms (the reference arm times a bounded sample of it,
    stated in its cpu_baseline)."""
    relax = c["relax_used"]   # no import of the product package here: the reference arm uses this too
    omega = c["omega"] if relax == "vanka" else c["bsr_omega"]
    n, L = c["n"], c["levels"]
    pitch = ((n + 1 + 31) // 32) * 32
    return {"workload": f"BASELINE config {args.config}: {n}^2 cells, {L} levels, V(1,1) {relax}, "
                        f"lambda={c['lam']}, mu={c['mu']}, K={'exp(N(0,4)) field' if c['K_seed'] is not None else c['K']}, "
                        f"tau=alpha=1/M=1, b~U(-1,1) seed {c['b_seed']}, x0=0",
            "n": n, "levels": L, "relax": relax, "omega": omega,
            "omega_J": c["omega_J"] if relax == "bsr" else None,
            "active_dofs": mg_inputs.n_active(n),
            "l2": "inputs larger than L2 (one vector = %.2f GB)" % (10 * (n + 1) * pitch * 8 / 1e9)}


def run_reference(args, c, rank, world):
    if rank != 0:
        return
    s = oracle_sample(c, args.steps, args.warmup)
    # the config names what was actually timed: the oracle on an n_sample^2 sample with the
    # workload's parameters (the 4096^2 operator does not fit the oracle), not the workload itself
    cfg = workload_config(args, c)
    cfg.update({"workload": f"SAMPLE of BASELINE config {args.config}: the CPU oracle on {s['n']}^2 cells, "
                            f"{s['levels']} levels{'' if s['n'] == c['n'] else ' (not %d^2)' % c['n']}, same parameters, RHS recipe and V(1,1) cycle",
                "n": s["n"], "levels": s["levels"], "active_dofs": mg_inputs.n_active(s["n"]),
                "sample_of": cfg["workload"], "l2": "host CPU run (no L2 flush)"})
    line = {"impl": "reference", "metric": METRIC, "value": s["value"],
            "unit": "DoF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": s["ms"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": cfg,
            "cpu_baseline": {"value": s["value"], "unit": "DoF/s", "cores": s["cores"], "kind": "oracle",
                             "sample": s["sample"]},
            "e2e": {"value": s["value"], "unit": "DoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--trace-cycles", type=int, default=10)
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--n", type=int, default=0, help="experiment: override the grid size (levels keep n_c = 4)")
    ap.add_argument("--relax", default="", choices=["", "vanka", "bsr", "bsr_exact"],
                    help="override the relaxation (config 2 names both: Vanka by default, --relax bsr for BSR; "
                         "--relax vanka on config 4 runs the heterogeneous-K Vanka of SURVEY 8(f) rank 4; "
                         "bsr_exact: exact BSR, n <= 1024)")
    ap.add_argument("--quadrature", default="rq", choices=["rq", "exact"],
                    help="exact: the exact-integration operator of eq. block_form (SURVEY 8(f) rank 3)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    c = workload(args.config)
    if args.relax:
        c["relax_used"] = args.relax
        c.setdefault("bsr_omega", 0.75)
        c.setdefault("omega_J", 1.0)
        c.setdefault("omega", 0.74)
    if args.n:
        c["n"], c["levels"] = args.n, int(np.log2(args.n // 4)) + 1
    if args.impl == "reference":
        return run_reference(args, c, rank, world)

    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2107_04060_b200 import Hierarchy
    n, L = c["n"], c["levels"]
    kf = None if c["K_seed"] is None else mg_inputs.lognormal_K(n, c["K_seed"])
    H = Hierarchy(n, L, c["lam"], c["mu"], K=c["K"] if c["K"] is not None else 1.0, tau=c["tau"],
                  alpha=c["alpha"], inv_M=c["inv_M"], mu_f=c["mu_f"], K_field=kf, quadrature=args.quadrature)
    o = opts_for(c)
    b_host = mg_inputs.uniform_rhs(n, c["b_seed"])
    b = H.to_device(b_host)
    x = H.zeros()
    nrm = torch.zeros(1, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    nact = H.n_active(0)
    for _ in range(args.warmup):
        H.cycle_async(x, b, o, nrm)
    torch.cuda.synchronize()
    launches_per_cycle = H.cycle_kernels()

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            H.cycle_async(x, b, o, nrm)
        ev1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1), dist)
    res_norm = float(nrm.sqrt().item())

    # kernel-class timing of the same cycle (event-traced graph, separate pass)
    H.set_timing(True)
    phases = np.zeros(5)
    per_level = None
    for _ in range(args.trace_cycles):
        H.cycle_async(x, b, o, nrm)
        phases += np.array(H.timing())
        tl = H.timing_levels()
        if per_level is None:
            per_level = {k: np.array(v, dtype=float) for k, v in tl.items()}
        else:
            for k, v in tl.items():
                per_level[k] = per_level[k] + np.array(v, dtype=float)
    phases /= args.trace_cycles
    per_level = {k: (v / args.trace_cycles).round(4).tolist() for k, v in per_level.items()}
    H.set_timing(False)

    # full solve to 1e-8 with the paper's solver (FGMRES + one V-cycle per iteration)
    solve = None
    if not args.no_solve:
        xs = H.zeros()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        # restart length (tools/fgmres_sweep.py, repeated solves): 10 at 4096^2 (40 iterations, 0.40 s;
        # 20: 35 iterations, 0.50 s; 30: 35, 0.74 s -- the Gram-Schmidt passes grow with the basis),
        # 30 for the near-incompressible config 3 (20: 180 iterations; 15 and below stagnate)
        restart = 30 if args.config == 3 else 10
        rc, hist = H.fgmres(xs, b, o, rtol=1e-8, max_iters=300, restart=restart)
        e1.record(stream)
        torch.cuda.synchronize()
        first_ms = e0.elapsed_time(e1)
        true_rel = H.residual(0, xs, b, norm=True) / float(hist[0])
        # the same solve again: the per-iteration cycle graphs (one per basis slot) and the FGMRES
        # work space now exist, as in any later solve on this context
        xs.zero_()
        torch.cuda.synchronize()
        e0.record(stream)
        rc2, hist2 = H.fgmres(xs, b, o, rtol=1e-8, max_iters=300, restart=restart)
        e1.record(stream)
        torch.cuda.synchronize()
        solve = {"method": f"FGMRES({restart}) (classical Gram-Schmidt, second pass when the first cancelled more than 10x: DGKS test with eta = 0.1), "
                           "right-preconditioned by one V(1,1) cycle per iteration",
                 "rtol": 1e-8, "iterations": len(hist) - 1, "converged": rc == 0,
                 "final_rel_residual_estimate": float(hist[-1] / hist[0]),
                 "true_rel_residual": true_rel,
                 "ms": e0.elapsed_time(e1),
                 "ms_first": first_ms,
                 "note": "ms: a repeated solve on the same context; ms_first: the first one, which also allocates "
                         "the Krylov work space and instantiates the per-basis-slot cycle graphs"}
        del xs

    # e2e through the public C ABI with host buffers
    e2e = None
    if not args.no_e2e:
        bp = torch.from_numpy(b_host).pin_memory().numpy()
        xp = torch.zeros(b_host.shape, dtype=torch.float64).pin_memory().numpy()
        H.solve_host(xp, bp, o, rtol=0.0, max_cycles=2)              # warm the e2e buffers
        xp[:] = 0.0
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        rc, hist = H.solve_host(xp, bp, o, rtol=0.0, max_cycles=args.steps)
        el = max_over_ranks(time.perf_counter() - t0, dist)
        cyc = len(hist) - 1
        vbytes = 10 * (n + 1) * (n + 1) * 8
        e2e = {"value": aggregate_rate(nact, cyc, world, el * 1e3), "unit": "DoF/s", "h2d_bytes_per_step": 2 * vbytes / cyc,
               "d2h_bytes_per_step": (vbytes + 8 * (cyc + 1)) / cyc,
               "note": f"mg_solve_host of {cyc} cycles: pinned host b, x0 in; x, history out; bytes amortised per cycle"}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    peak, peak_src = peaks()
    relax_ms = (phases[0] + phases[4]) / 2.0
    # levels whose first post-sweep absorbs the prolongation (marching Vanka levels, mg_api.cu
    # fused_prolong): that sweep also reads the coarse iterate, 1/4 of a fine pass
    march_min = int(os.environ.get("MG_MARCH_MIN_N", "512"))
    het = c["K_seed"] is not None
    fused = o.relax == "vanka" and os.environ.get("MG_FUSE_PROLONG", "1") != "0" and \
        os.environ.get("MG_VANKA_IMPL", "2") == "2" and not het and args.quadrature == "rq"
    if o.relax == "vanka" and het:
        # heterogeneous Vanka: read x, b, write x + the per-vertex S~^{-1} table (21 doubles per vertex
        # = 16.8 B per active DoF at 10 DoFs per vertex) + K^{-1} (2 per cell)
        alg_bytes = (24.0 + 16.8 + 1.6) * nact
        hwarp = n >= int(os.environ.get("MG_HET_WARP_N", "256")) > 0
        dom = (("vanka_hwarp_kernel + vanka_bnd_kernel<HET>" if hwarp else "vanka_het_kernel") +
               " (level 0: residual with the K^{-1} field + condensed patch solves + update)")
    elif o.relax == "vanka":
        # read x, read b, write x over the active DoFs; averaged over the pre-sweep and the post-sweep
        # (which with the fused prolongation also reads e_H: + 8 B x N_1 ~ 2 B per fine DoF)
        alg_bytes = (24.0 * nact + (24.0 * nact + 8.0 * mg_inputs.n_active(n >> 1) if fused and n >= march_min
                                    else 24.0 * nact)) / 2.0
        warp = n >= int(os.environ.get("MG_WARP_MIN_N", "512")) > 0
        dom = (("vanka_warp_kernel + vanka_bnd2_kernel" if warp else "vanka_march2_kernel") +
               " (level 0: fused residual + 20-DoF patch solves + update; "
               "mean of the pre-sweep and the post-sweep" + (" with the prolongation fused in)" if fused else ")"))
    else:
        alg_bytes = 8.0 * nact * 4.8 + 8.0 * 0.2 * nact   # 3 + 1.8 passes (+0.2 K field)
        dom = "BSR relaxation (level 0: bsr_a + 2 jacobi + bsr_b)"
    achieved = alg_bytes / (relax_ms * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        if tj.get("config") == args.config:
            traffic = tj.get("dram_bytes_per_launch")
    except Exception:
        pass
    # algorithmic passes per level per V(1,1): Vanka 3 + 3 sweeps, 2.25 restriction,
    # 2.25 prolongation (fused into the post-sweep: 0.25, the read of e_H); BSR 14.1 (14.7 with K field)
    def level_passes(l):
        if o.relax != "vanka":
            return 14.7 if c["K_seed"] is not None else 14.1
        if l == L - 1:
            return 0.0 if L > 1 else 6.0
        if het:                       # + the S~^{-1} table and K^{-1} in both sweeps (2 x 2.3 passes)
            return 15.1
        return 8.5 if fused and (n >> l) >= march_min else 10.5
    # B_alg of SURVEY 8(d) (10.5 Vanka / 14.1 BSR / 14.7 BSR + K field passes on every level): the
    # roofline figure of the method; the fused schedule (prolongation inside the post-sweep) needs
    # fewer bytes, reported beside it
    sum_levels = sum(mg_inputs.n_active(n >> l) for l in range(L))
    b_alg = 8.0 * ((15.1 if het else 10.5) if o.relax == "vanka" else 14.7 if het else 14.1) * sum_levels
    cycle_bytes = 8.0 * sum(level_passes(l) * mg_inputs.n_active(n >> l) for l in range(L))
    ms_step = ms / args.steps
    line = {
        "metric": METRIC,
        "value": aggregate_rate(nact, args.steps, world, ms),
        "unit": "DoF/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": dict(workload_config(args, c), final_residual_norm=res_norm),
        "gpu_launches": launches_per_cycle * args.steps,
        "clocks": clk.summary(),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": dom, "kernel_ms": relax_ms,
                     "algorithmic_bytes_per_launch": alg_bytes, "peak_source": peak_src},
        "cycle_roofline": {"algorithmic_bytes": b_alg, "achieved_gbs": b_alg / (ms_step * 1e-3) / 1e9,
                           "frac": b_alg / (ms_step * 1e-3) / 1e9 / peak,
                           "frac_of_nominal_8tbs": b_alg / (ms_step * 1e-3) / 8.0e12,
                           "fused_schedule_bytes": cycle_bytes,
                           "fused_schedule_frac": cycle_bytes / (ms_step * 1e-3) / 1e9 / peak,
                           "phase_ms": {"pre": phases[0], "restrict": phases[1], "coarse_levels": phases[2],
                                        "prolong": phases[3], "post": phases[4]},
                           "per_level_ms": per_level},
        "e2e": e2e,
        "solve": solve,
    }
    if world == 1 and not args.no_cpu_baseline:
        s = oracle_sample(c, 20)
        line["cpu_baseline"] = {"value": s["value"], "unit": "DoF/s", "cores": s["cores"], "kind": "oracle",
                                "sample": s["sample"]}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Warm per-kernel times of every level of a hierarchy (CUDA events around R back-to-back
launches of one C-ABI call; diagnostic only, not a bench line).  The vanka column is half of an
mg_relax_vanka call with 2 sweeps (an even count ends in x: no copy back).

    python tools/level_times.py [--n 4096] [--levels 11] [--reps 50]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2107_04060_b200 import Hierarchy  # noqa: E402


def timed(fn, reps):
    """Device time per call: R calls captured in one CUDA graph (no host launch overhead)."""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3   # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--levels", type=int, default=11)
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    H = Hierarchy(a.n, a.levels, 100.0, 1.0, K=1e-2)
    print(f"{'level':>5} {'n':>5} {'vanka':>9} {'residual':>9} {'restrict':>9} {'prolong':>9}  (us per launch)")
    for l in range(a.levels):
        n = H.level_n(l)
        x, b, r = H.zeros(l), H.zeros(l), H.zeros(l)
        b.normal_()
        x.normal_()
        tv = timed(lambda: H.relax_vanka(l, x, b, 0.7, sweeps=2), a.reps) / 2
        tr = timed(lambda: H.residual(l, x, b, r), a.reps)
        if l + 1 < a.levels:
            bc = H.zeros(l + 1)
            tq = timed(lambda: H.restrict(l, r, bc), a.reps)
            tp = timed(lambda: H.prolong(l, bc, x), a.reps)
        else:
            tq = tp = float("nan")
        print(f"{l:5d} {n:5d} {tv:9.1f} {tr:9.1f} {tq:9.1f} {tp:9.1f}")
    H.close()


if __name__ == "__main__":
    main()

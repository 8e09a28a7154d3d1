"""Timing of backward-Euler steps on the GPU (context, not a bench line):
the smooth time-dependent problem of reading A28 at the paper's tab:easy_time setting (E = 3e4,
nu = 0.4 / 0.499, k = 1e-6, M = 1e6, FGMRES(30) to 1e-10 with one Vanka V(2,2) cycle per iteration,
tab:vanka22's omega) on N = n + 1 points, tau = 1/16 (tab:easy_time's first column), 8 steps.
Loads come from the oracle's manufactured assembly (oracle/timestep.py, test infrastructure: this
tool is diagnostics, not the product).  Prints per-step iterations and device ms.

    python tools/timestep_bench.py [--n 256] [--steps 8]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import timestep as T  # noqa: E402
from oracle.cycle import lame  # noqa: E402
from oracle.fem import Operator  # noqa: E402
from oracle.mesh import Mesh  # noqa: E402
from paper_2107_04060_b200 import Hierarchy, Opts  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--steps", type=int, default=8)
    a = ap.parse_args()
    n, tau, k = a.n, 1.0 / 16, 1e-6
    levels = int(np.log2(n // 8)) + 1                      # coarsest h = 1/8
    for nu in (0.4, 0.499):
        mu, lam = lame(3e4, nu)
        op = Operator(Mesh(n), lam, mu, tau, 1.0, 1e-6, 1.0, K=k)
        m = op.mesh
        loads = [m.from_active(T.load(op, s * tau, k)) for s in range(1, a.steps + 1)]
        x0 = m.from_active(T.initial(op))
        H = Hierarchy(n, levels, lam, mu, K=k, tau=tau, alpha=1.0, inv_M=1e-6)
        o = Opts(2, 2, "vanka", 0.80 if nu == 0.4 else 0.72)
        bl = [H.to_device(L) for L in loads]
        x = H.to_device(x0)
        H.time_step(x, bl[0], o, rtol=1e-10, max_iters=200, restart=30)   # graphs + work space
        x = H.to_device(x0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        its = []
        e0.record()
        for s in range(a.steps):
            rc, h = H.time_step(x, bl[s], o, rtol=1e-10, max_iters=200, restart=30)
            its.append(len(h) - 1)
        e1.record()
        torch.cuda.synchronize()
        eu, ep = T.errors(op, m.to_active(H.to_host(x)), a.steps * tau)
        print(json.dumps(dict(nu=nu, N=n + 1, levels=levels, tau=tau, steps=a.steps, iterations=its,
                              ms_per_step=e0.elapsed_time(e1) / a.steps, err_u_H1=eu, err_p_L2=ep)), flush=True)
        H.close()


if __name__ == "__main__":
    main()

"""Context for the paper's own timings (tab:mgtime; 8-core Sandy Bridge, HAZmath):
FGMRES preconditioned by one V-cycle on the GPU at the paper's parameters (E = 3e4, M = 1e6, K = 1e-6 I,
tau = alpha = mu_f = 1), N = 17 .. 257 (n = 16 .. 256 cells, coarsest h = 1/8), rtol 1e-6, x0 = 0.

Differences from the paper's runs: the right-hand side is b = A x* for the smooth field x* of the
paper's manufactured solution sampled at the DoFs (u = curl phi, phi = [xy(1-x)(1-y)]^2 at the
vertices, p = 1, bubbles and w = 0; A applied by mg_residual), not the paper's FE load vector of
PAPER.md:936-945 (assembled only by the oracle); and the Vanka cycle is V(2,2)
with omega = tab:vanka22's (reading A25); BSR is V(1,1) with one Jacobi sweep at tab:bsr_vanka11's
(omega_J, omega).  Times are device times of a repeated solve (the first solve on a context also
instantiates its graphs).  Context only, not a bench line.

    python tools/paper_context.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import mg_inputs  # noqa: E402
from paper_2107_04060_b200 import Hierarchy, Opts  # noqa: E402

PAPER = {  # tab:mgtime: seconds (iterations) for N = 17, 33, 65, 129, 257
    (0.4, "vanka"): [(0.034, 8), (0.194, 9), (0.976, 9), (4.053, 9), (16.462, 9)],
    (0.4, "bsr"): [(0.025, 11), (0.128, 12), (0.663, 13), (3.035, 14), (12.726, 14)],
    (0.499, "vanka"): [(0.055, 13), (0.279, 13), (1.340, 13), (5.501, 13), (24.439, 13)],
    (0.499, "bsr"): [(0.049, 20), (0.258, 23), (1.417, 26), (6.888, 29), (30.820, 33)],
}
OPTS = {  # tab:vanka22 / tab:bsr_vanka11 at k = 1e-6
    (0.4, "vanka"): Opts(2, 2, "vanka", 0.80),
    (0.4, "bsr"): Opts(1, 1, "bsr", 0.74, 0.94, 1),
    (0.499, "vanka"): Opts(2, 2, "vanka", 0.72),
    (0.499, "bsr"): Opts(1, 1, "bsr", 0.68, 0.86, 1),
}


def lame(E, nu):
    return E / (2.0 + 2.0 * nu), E * nu / ((1.0 - 2.0 * nu) * (1.0 + nu))


def smooth_rhs(H, n):
    """b = A x* (mg_residual with b = 0 gives -A x*)."""
    import numpy as np
    t = np.arange(n + 1) / n
    y, x = np.meshgrid(t, t, indexing="ij")                  # [j, i]
    g = lambda s: s * (1 - s)                                # noqa: E731
    dg = lambda s: 1 - 2 * s                                 # noqa: E731
    # phi = g(x)^2 g(y)^2: u_x = d phi / dy, u_y = -d phi / dx
    xs = np.zeros((10, n + 1, n + 1))
    xs[0] = g(x) ** 2 * 2 * g(y) * dg(y)
    xs[1] = -(2 * g(x) * dg(x)) * g(y) ** 2
    xs[8] = xs[9] = 1.0
    xs[~mg_inputs.active_mask(n)] = 0.0
    xd, z, r = H.to_device(xs), H.zeros(), H.zeros()
    H.residual(0, xd, z, r)
    return -r


def main():
    for (nu, relax), paper in PAPER.items():
        mu, lam = lame(3e4, nu)
        for k, n in enumerate((16, 32, 64, 128, 256)):
            H = Hierarchy(n, k + 2, lam, mu, K=1e-6, tau=1.0, alpha=1.0, inv_M=1e-6)
            b = smooth_rhs(H, n)
            o = OPTS[(nu, relax)]
            x = H.zeros()
            H.fgmres(x, b, o, rtol=1e-6, max_iters=200, restart=30)    # graphs, work space
            x.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rc, h = H.fgmres(x, b, o, rtol=1e-6, max_iters=200, restart=30)
            e1.record()
            torch.cuda.synchronize()
            print(json.dumps(dict(nu=nu, relax=relax, N=n + 1, levels=k + 2, rc=rc, iters=len(h) - 1,
                                  gpu_ms=round(e0.elapsed_time(e1), 3), paper_s=paper[k][0],
                                  paper_iters=paper[k][1])), flush=True)
            H.close()


if __name__ == "__main__":
    main()

"""Write the oracle's residual histories at every BASELINE config, at that config's own size
(VERDICT r01 "Next round" 2).  Imports only ``oracle/`` and ``mg_inputs`` (no CUDA path).

    python tests/scripts/golden_histories.py CONFIG RELAX [--alt] [--cycles K]

One job per call (the 1024^2 and 2048^2 oracles need tens of GB and tens of minutes, so the main
and the reversed-summation-order runs are separate processes).  Writes
``tests/golden/hist_cfg{CONFIG}_{RELAX}{_alt}.json`` with

* ``hist``    ||b - A x_k||_2, k = 0..K (x_0 = 0; V(1,1) cycles);
* ``floor8``  8 u || |b| + |A| |x_k| ||_2 per k, the a-priori rounding scale of one residual
  evaluation (first term of F_k, SURVEY 8c-11 / reading A22);
* ``final``   the last iterate: per-block 2-norms (u: planes 0-4, w: 5-7, p: 8-9, and p minus its
  mean), the mean of p, and its values at 4096 seeded sample slots plus the 4 corner-adjacent
  cells (unpadded plane-major slot indices of the mg_inputs layout).

``--alt`` runs the same method with every summation order reversed (Hierarchy(alt_order=True));
the spread between the two files calibrates the parity floor (4 x spread).  The GPU tests
(tests/test_gpu_golden.py) replay the configs on the production contexts and compare.

Config parameters come from ``mg_inputs.CONFIGS`` (readings A5, A7, A24 of DESIGN.md); BSR uses
n_J = 3 Jacobi sweeps (BASELINE configs 2 and 4).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import resource
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import mg_inputs  # noqa: E402
from oracle.cycle import Hierarchy  # noqa: E402

U = 2.0 ** -53
DEFAULT_CYCLES = {1: 10, 2: 20, 3: 5, 4: 4, 5: 3}   # config 4 with Vanka: also 4 (the oracle needs ~110 GB)


def opts_for(c, relax):
    if relax == "vanka":   # config 4 with Vanka: the heterogeneous-K Vanka of reading A20 at omega = 0.74
        return dict(nu1=1, nu2=1, omega=c.get("omega", 0.74))
    return dict(nu1=1, nu2=1, omega=c["bsr_omega"], omega_J=c["omega_J"], jacobi_sweeps=3)


def sample_slots(n, count=4096, seed=12345):
    """Seeded active slots (unpadded plane-major indices) + the P0 / RT0 slots of the corner cells."""
    act = np.nonzero(mg_inputs.active_mask(n).reshape(-1))[0]
    rng = np.random.Generator(np.random.PCG64(seed))
    pick = np.sort(rng.choice(act, size=min(count, act.size), replace=False))
    N1 = n + 1
    extra = [(k * N1 + j) * N1 + i for k in (7, 8, 9) for (i, j) in ((0, 0), (n - 1, 0), (0, n - 1), (n - 1, n - 1))]
    return np.unique(np.concatenate([pick, np.array(extra)]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int)
    ap.add_argument("relax", choices=["vanka", "bsr"])
    ap.add_argument("--alt", action="store_true")
    ap.add_argument("--cycles", type=int, default=None)
    a = ap.parse_args()
    c = mg_inputs.CONFIGS[a.config]
    K = a.cycles or DEFAULT_CYCLES[a.config]
    n, L = c["n"], c["levels"]
    kinv = None if c["K_seed"] is None else 1.0 / mg_inputs.lognormal_K(n, c["K_seed"])
    t0 = time.time()
    H = Hierarchy(n, L, c["lam"], c["mu"], c["tau"], c["alpha"], c["inv_M"], c["mu_f"],
                  K=1.0 if c["K"] is None else c["K"], Kinv_field=kinv, relax=a.relax, alt_order=a.alt)
    t_setup = time.time() - t0
    m = H.meshes[0]
    op = H.ops[0]
    absA = op.A.copy()
    absA.data = np.abs(absA.data)
    b = m.to_active(mg_inputs.uniform_rhs(n, c["b_seed"]))
    x = np.zeros_like(b)
    od = opts_for(c, a.relax)
    hist, floor = [], []

    def record(x):
        hist.append(float(np.linalg.norm(b - op.A @ x)))
        floor.append(float(8 * U * np.linalg.norm(np.abs(b) + absA @ np.abs(x))))
    record(x)
    t1 = time.time()
    for k in range(K):
        x = H.cycle(x, b, od)
        record(x)
        print(f"cycle {k + 1}: {hist[-1]:.6e} ({time.time() - t1:.0f} s)", flush=True)
    t_cycles = time.time() - t1
    X = m.from_active(x)
    p = X[8:10][mg_inputs.active_mask(n)[8:10]]
    sl = sample_slots(n)
    out = dict(
        config=a.config, n=n, levels=L, relax=a.relax, alt_order=a.alt, opts=od, cycles=K,
        b_seed=c["b_seed"], K_seed=c["K_seed"],
        material=dict(lam=c["lam"], mu=c["mu"], K=c["K"], tau=c["tau"], alpha=c["alpha"], inv_M=c["inv_M"],
                      mu_f=c["mu_f"]),
        hist=hist, floor8=floor,
        final=dict(norm_u=float(np.linalg.norm(X[0:5])), norm_w=float(np.linalg.norm(X[5:8])),
                   norm_p=float(np.linalg.norm(p)), norm_p0=float(np.linalg.norm(p - p.mean())),
                   mean_p=float(p.mean()), slots=sl.tolist(), values=X.reshape(-1)[sl].tolist()),
        provenance=dict(script="tests/scripts/golden_histories.py", host=platform.node(), cpus=os.cpu_count(),
                        setup_s=round(t_setup, 1), cycles_s=round(t_cycles, 1),
                        maxrss_gb=round(resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6, 2)),
    )
    name = f"hist_cfg{a.config}_{a.relax}{'_alt' if a.alt else ''}.json"
    # GOLDEN_OUT: another directory (the 2048^2 oracle needs ~65 GB and runs on a larger host)
    with open(os.path.join(os.environ.get("GOLDEN_OUT", os.path.join(ROOT, "tests", "golden")), name), "w") as f:
        json.dump(out, f)
    print("wrote", name, out["provenance"])


if __name__ == "__main__":
    main()

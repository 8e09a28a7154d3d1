"""Config 4 (reading A24): where does the BSR V(1,1) cycle start to diverge as the lognormal
permeability field gets rougher?  Oracle only: K = exp(sigma Z), Z = PCG64(3).normal(0, 1) (the
config-4 draw rescaled: mg_inputs.lognormal_K(n, 3, sigma)), lambda = mu = tau = alpha = 1/M = 1,
64^2, 5 levels, n_J = 3, measured factor rho_N (b = 0, random x_0, 30 cycles, mean of the last 4;
PAPER.md:809-811) for sigma in {0, 0.5, 1, 1.5, 2} and the two (omega_J, omega) pairs the build
uses: (1.0, 0.75) (E0 optimum for config 2, K = 1) and (0.7, 0.3) (config 4).  Also the smoother
alone (60 sweeps).  Writes tests/golden/sigma_sweep_bsr.json."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import mg_inputs  # noqa: E402
from oracle.cycle import Hierarchy  # noqa: E402

n, L = int(os.environ.get("SIGMA_N", 64)), int(os.environ.get("SIGMA_L", 5))
RELAX = os.environ.get("SIGMA_RELAX", "bsr")     # "vanka": heterogeneous additive Vanka


def rho_smoother(H, opts, sweeps=60):
    rng = np.random.Generator(np.random.PCG64(0))
    N = H.ops[0].A.shape[0]
    x = rng.uniform(-1, 1, N)
    b = np.zeros(N)
    prev = np.linalg.norm(H.ops[0].A @ x)
    rs = []
    for _ in range(sweeps):
        x = H.smooth(0, x, b, opts)
        r = np.linalg.norm(H.ops[0].A @ x)
        rs.append(r / prev)
        prev = r
    return float(np.mean(rs[-5:]))


out = dict(what=f"{RELAX} V(1,1) rho_N vs sigma of the lognormal K, {n}^2, {L} levels", rows=[])
PAIRS = ((1.0, 0.75), (0.7, 0.3)) if RELAX == "bsr" else ((0.0, 0.74), (0.0, 0.6))
for sigma in (0.0, 0.5, 1.0, 1.5, 2.0):
    kinv = 1.0 / mg_inputs.lognormal_K(n, 3, sigma=sigma)
    H = Hierarchy(n, L, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, Kinv_field=kinv, relax=RELAX)
    for omJ, om in PAIRS:
        o = dict(nu1=1, nu2=1, omega=om, omega_J=omJ, jacobi_sweeps=3)
        _, rs = H.measure_rho(o, seed=0, min_cycles=30, max_cycles=30)
        row = dict(sigma=sigma, omega_J=omJ, omega=om, rho_cycle=float(np.mean(rs[-4:])),
                   rho_smoother=rho_smoother(H, o), K_min=float(1 / kinv.max()), K_max=float(1 / kinv.min()))
        out["rows"].append(row)
        print(row, flush=True)
with open(os.path.join(ROOT, "tests", "golden", f"sigma_sweep_{RELAX}.json"), "w") as f:
    json.dump(out, f, indent=1)

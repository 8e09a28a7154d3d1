"""Evidence for reading A5: the BASELINE configs run 1/M = 1, not SURVEY 8(b)'s
proposed 1e-6.  Oracle only: config-5 materials (lambda = 100, mu = 1, K = 1e-2, tau = alpha = 1),
32^2, V(1,1) additive Vanka, omega = 0.70 (E0), measured factor rho_N (PAPER.md:809-811 protocol:
b = 0, random x_0, 40 cycles, mean of the last 4) for 2 and 4 levels and
1/M in {1e-6, 1e-3, 1e-2, 1}.  Writes tests/golden/a5_invM_scan.json.

Why 1/M matters here (A5): the dimensionless group is mu/M.  The paper's
runs have E = 3e4 (mu ~ 1e4) with M = 1e6, i.e. mu/M ~ 1e-2; BASELINE's
mu = 1 with M = 1e6 would be mu/M = 1e-6, four decades outside anything the paper ran, and there the
constant-pressure eigenvalue gamma = h^2/(2M) of every patch is tiny compared with the patch's
displacement scale."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.cycle import Hierarchy  # noqa: E402

out = dict(what="rho_N of V(1,1) additive Vanka, omega=0.70, config-5 materials, 32^2", rows=[])
for invM in (1e-6, 1e-3, 1e-2, 1.0):
    for L in (2, 4):
        H = Hierarchy(32, L, 100.0, 1.0, 1.0, 1.0, invM, 1.0, K=1e-2, relax="vanka")
        _, rs = H.measure_rho(dict(nu1=1, nu2=1, omega=0.70), seed=0, min_cycles=40, max_cycles=40)
        rho = float(np.mean(rs[-4:]))
        out["rows"].append(dict(inv_M=invM, levels=L, rho=rho, mu_over_M=1.0 * invM))
        print(invM, L, rho, flush=True)
with open(os.path.join(ROOT, "tests", "golden", "a5_invM_scan.json"), "w") as f:
    json.dump(out, f, indent=1)

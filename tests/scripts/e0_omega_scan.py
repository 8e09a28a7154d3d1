"""Experiment E0: oracle V(1,1) convergence factors at the
BASELINE parameters on a 64x64 grid (5 levels, coarsest 4x4) versus the damping
parameters, following the brute-force protocol of PAPER.md:822 (step 0.02 near
the optimum).  1/M = 1 (reading A5).  Uses only oracle/; writes
tests/golden/e0_omega_scan.json (a derived record, not a paper value)."""
import json, sys
import numpy as np
sys.path.insert(0, '.')
from oracle.cycle import Hierarchy
import mg_inputs

def rho(H, opts):
    r, rs = H.measure_rho(opts, seed=0, min_cycles=40, max_cycles=40)
    return float(np.mean(rs[-4:]))

out = {}
n, L = 64, 5
cases = {'cfg1_2_vanka': (1.0, 1.0, 1.0), 'cfg3_vanka': (1e6, 1.0, 1e-6), 'cfg5_vanka': (100.0, 1.0, 1e-2)}
for name, (lam, mu, K) in cases.items():
    H = Hierarchy(n, L, lam, mu, 1.0, 1.0, 1.0, 1.0, K=K, relax='vanka')
    res = {}
    for om in np.arange(0.62, 0.79, 0.02):
        res[f'{om:.2f}'] = rho(H, dict(nu1=1, nu2=1, omega=float(om)))
        print(name, f'{om:.2f}', res[f'{om:.2f}'], flush=True)
    out[name] = res
grids = {'cfg2_bsr': ([0.8, 0.9, 1.0, 1.1], [0.7, 0.75, 0.8, 0.85]),
         'cfg4_bsr': ([0.3, 0.5, 0.7, 1.0], [0.2, 0.3, 0.4, 0.5])}
for name, kw in {'cfg2_bsr': dict(K=1.0), 'cfg4_bsr': dict(Kinv_field=1.0 / mg_inputs.lognormal_K(n, 3))}.items():
    H = Hierarchy(n, L, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, relax='bsr', **kw)
    res = {}
    for omJ in grids[name][0]:
        for om in grids[name][1]:
            key = f'{omJ:.2f},{om:.2f}'
            res[key] = rho(H, dict(nu1=1, nu2=1, omega=om, omega_J=omJ, jacobi_sweeps=3))
            print(name, key, res[key], flush=True)
    out[name] = res
json.dump(out, open('tests/golden/e0_omega_scan.json', 'w'), indent=1)

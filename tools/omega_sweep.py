"""Experiment: outer relaxation weight omega vs FGMRES iterations / time and the stationary
V-cycle's asymptotic factor on the GPU (config CFG, default 5).  Compares the two-grid LFA choice
(reading A27: omega_opt = 0.68 for configs 3 and 5) with E0's (0.70)."""
import os, sys, json
sys.path.insert(0, '.')
import torch
import mg_inputs
from paper_2107_04060_b200 import Hierarchy, Opts
cfg = int(os.environ.get("CFG", "5"))
c = mg_inputs.CONFIGS[cfg]
restart = 30 if cfg == 3 else 10
H = Hierarchy(c["n"], c["levels"], c["lam"], c["mu"], K=c["K"], tau=c["tau"], alpha=c["alpha"], inv_M=c["inv_M"])
b = H.to_device(mg_inputs.uniform_rhs(c["n"], c["b_seed"]))
for om in [float(w) for w in os.environ.get("OMEGAS", "0.64,0.66,0.67,0.68,0.69,0.70,0.71,0.72").split(",")]:
    o = Opts(1, 1, "vanka", om)
    x = H.zeros()
    H.fgmres(x, b, o, rtol=1e-8, max_iters=2 * restart, restart=restart)   # graphs
    x.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rc, h = H.fgmres(x, b, o, rtol=1e-8, max_iters=300, restart=restart)
    e1.record(); torch.cuda.synchronize()
    # stationary V(1,1) from a random start with zero RHS: factor of the last of 30 cycles
    z = H.zeros()
    xr = H.to_device(mg_inputs.uniform_vector(c["n"], 7))
    hs = [H.residual(0, xr, z, norm=True)]
    for _ in range(30):
        hs.append(H.cycle(xr, z, o))
    print(json.dumps(dict(cfg=cfg, omega=om, restart=restart, iters=len(h) - 1, rc=rc, ms=round(e0.elapsed_time(e1), 1),
                          rho_stationary=round(hs[-1] / hs[-2], 4), rho_mean10=round((hs[-1] / hs[-11]) ** 0.1, 4))), flush=True)
H.close()

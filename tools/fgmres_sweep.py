"""Experiment: FGMRES restart length and Gram-Schmidt passes vs iterations and time (config 5)."""
import os, sys, json
import numpy as np
sys.path.insert(0, '.')
import torch
import mg_inputs
from paper_2107_04060_b200 import Hierarchy, Opts
c = mg_inputs.CONFIGS[int(os.environ.get("CFG", "5"))]
H = Hierarchy(c["n"], c["levels"], c["lam"], c["mu"], K=c["K"], tau=c["tau"], alpha=c["alpha"], inv_M=c["inv_M"])
b = H.to_device(mg_inputs.uniform_rhs(c["n"], c["b_seed"]))
for restart in (8, 10, 15, 20, 30):
    x = H.zeros()
    H.fgmres(x, b, Opts(1, 1, "vanka", c["omega"]), rtol=1e-8, max_iters=2 * restart, restart=restart)  # graphs
    x.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rc, h = H.fgmres(x, b, Opts(1, 1, "vanka", c["omega"]), rtol=1e-8, max_iters=300, restart=restart)
    e1.record(); torch.cuda.synchronize()
    print(json.dumps(dict(cgs=os.environ.get("MG_CGS_PASSES", "0"), restart=restart, iters=len(h) - 1, rc=rc,
                          ms=round(e0.elapsed_time(e1), 1), true=H.residual(0, x, b, norm=True) / h[0])))

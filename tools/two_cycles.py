"""Two V(1,1) cycles of a BASELINE config (default 5): a small driver for ncu captures of the cycle
kernels.  CFG=<1..5> picks the config; RELAX=vanka|bsr overrides the relaxation; KFIELD=0 drops
config 4's K field (scalar K = 1) to separate the heterogeneous-coefficient cost."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import mg_inputs  # noqa: E402
from paper_2107_04060_b200 import Hierarchy, Opts  # noqa: E402

c = mg_inputs.CONFIGS[int(os.environ.get("CFG", "5"))]
relax = os.environ.get("RELAX", "bsr" if c["relax"] == "bsr" else "vanka")
kf = None
if c["K_seed"] is not None and os.environ.get("KFIELD", "1") != "0":
    kf = mg_inputs.lognormal_K(c["n"], c["K_seed"])
H = Hierarchy(c["n"], c["levels"], c["lam"], c["mu"], K=c["K"] or 1.0, tau=c["tau"], alpha=c["alpha"],
              inv_M=c["inv_M"], K_field=kf)
b = H.to_device(mg_inputs.uniform_rhs(c["n"], c["b_seed"]))
x = H.zeros()
if relax == "bsr":
    o = Opts(1, 1, "bsr", c.get("bsr_omega", 0.75), c.get("omega_J", 1.0), 3)
else:
    o = Opts(1, 1, "vanka", c.get("omega", 0.74))
for _ in range(2):
    H.cycle(x, b, o)
torch.cuda.synchronize()
print("ok")

"""Two V(1,1) cycles at config 5 (4096^2): a small driver for ncu captures of the cycle kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import mg_inputs  # noqa: E402
from paper_2107_04060_b200 import Hierarchy, Opts  # noqa: E402

c = mg_inputs.CONFIGS[int(os.environ.get("CFG", "5"))]
H = Hierarchy(c["n"], c["levels"], c["lam"], c["mu"], K=c["K"], tau=c["tau"], alpha=c["alpha"], inv_M=c["inv_M"])
b = H.to_device(mg_inputs.uniform_rhs(c["n"], c["b_seed"]))
x = H.zeros()
o = Opts(1, 1, "vanka", c["omega"])
for _ in range(2):
    H.cycle(x, b, o)
torch.cuda.synchronize()
print("ok")

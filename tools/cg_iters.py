"""CG iterations of the exact-BSR Schur solve (mg_relax_bsr_exact) across sizes and materials
(diagnostic for the iteration cap of the graph-captured CG)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import mg_inputs  # noqa: E402
from paper_2107_04060_b200 import Hierarchy  # noqa: E402

MATS = {"unit": (1.0, 1.0, 1.0, 1.0), "cfg5": (100.0, 1.0, 1e-2, 1.0), "stiff": (1e6, 1.0, 1e-6, 1.0),
        "paper0.4": (42857.14, 10714.29, 1e-6, 1e-6), "paper0.499": (4.99e6, 10008.0, 1e-6, 1e-6)}
for name, (lam, mu, K, invM) in MATS.items():
    row = []
    for n in (16, 32, 64, 128, 256, 512):
        for quad in ("rq", "exact"):
            H = Hierarchy(n, 3 if n == 32 else 2, lam, mu, K=K, inv_M=invM, quadrature=quad)
            x, b = H.to_device(mg_inputs.uniform_vector(n, 1)), H.to_device(mg_inputs.uniform_rhs(n, 2))
            rc, its = H.relax_bsr_exact(0, x, b, 0.8)
            torch.cuda.synchronize()
            row.append(f"n={n} {quad}: {its}{'' if rc == 0 else ' (cap)'}")
            H.close()
    print(name, "; ".join(row), flush=True)

"""at nu = 0.4 the FGMRES iterations of the BSR-preconditioned solve grow
with N faster than the paper's tab:mgtime (11, 12, 13, 14, 14 for N = 17 .. 257).
Oracle only, the tab:mgtime setting (E = 3e4, k = 1e-6, M = 1e6, FE load vector of the steady
manufactured problem, coarsest h = 1/8, FGMRES(30) to 1e-6): iterations for N = 17, 33, 65 with
variants of the cycle -- BSR V(1,1) at tab:bsr_vanka11's k = 1e-6 weights (0.94, 0.74) with one
Jacobi sweep (the GPU's paper_context setting), V(2,2), two and three Jacobi sweeps, and exact BSR
(S solved exactly).  Writes tests/golden/bsr_growth.json."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.cycle import Hierarchy, lame  # noqa: E402
from oracle.krylov import fgmres_mg  # noqa: E402
from oracle.manufactured import rhs  # noqa: E402

VARIANTS = {
    "V(1,1) nJ=1 (0.94,0.74)": ("bsr", dict(nu1=1, nu2=1, omega=0.74, omega_J=0.94, jacobi_sweeps=1)),
    "V(2,2) nJ=1 (0.94,0.74)": ("bsr", dict(nu1=2, nu2=2, omega=0.74, omega_J=0.94, jacobi_sweeps=1)),
    "V(1,1) nJ=2 (0.94,0.74)": ("bsr", dict(nu1=1, nu2=1, omega=0.74, omega_J=0.94, jacobi_sweeps=2)),
    "V(1,1) nJ=3 (0.94,0.74)": ("bsr", dict(nu1=1, nu2=1, omega=0.74, omega_J=0.94, jacobi_sweeps=3)),
    "V(1,1) exact S (0.74)": ("bsr_exact", dict(nu1=1, nu2=1, omega=0.74)),
}
out = dict(setting="tab:mgtime: nu = 0.4, E = 3e4, k = 1e-6, M = 1e6, coarsest h = 1/8, FGMRES(30) rtol 1e-6",
           printed={"17": 11, "33": 12, "65": 13, "129": 14, "257": 14}, rows={})
mu, lam = lame(3e4, 0.4)
for name, (relax, o) in VARIANTS.items():
    its = {}
    for n in (16, 32, 64):
        H = Hierarchy(n, n.bit_length() - 3, lam, mu, 1.0, 1.0, 1e-6, 1.0, K=1e-6, relax=relax)
        b = rhs(H.ops[0], mu, 1e-6)
        _, h = fgmres_mg(H, b, o, rtol=1e-6, max_iters=200, restart=30)
        its[str(n + 1)] = len(h) - 1
    out["rows"][name] = its
    print(name, its, flush=True)
with open(os.path.join(ROOT, "tests", "golden", "bsr_growth.json"), "w") as f:
    json.dump(out, f, indent=1)

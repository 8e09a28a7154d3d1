import sys, numpy as np
sys.path.insert(0, '.')
import mg_inputs
from tests import _cases as C
from paper_2107_04060_b200 import Opts
from oracle.krylov import fgmres_mg
for (n, L, pname) in ((16, 3, "unit"), (32, 4, "cfg5")):
    H = C.gpu_hierarchy(n, L, pname)
    Oh = C.hierarchy(n, L, pname, "vanka")
    m = Oh.meshes[0]
    b = mg_inputs.uniform_rhs(n, 3)
    ba = m.to_active(b)
    od, go = dict(nu1=1, nu2=1, omega=0.72), Opts(1, 1, "vanka", 0.72)
    for its in (1, 2, 3):
        xO, hO = fgmres_mg(Oh, ba, od, rtol=1e-12, max_iters=its, restart=30)
        xd, bd = H.to_device(np.zeros_like(b)), H.to_device(b)
        rc, hG = H.fgmres(xd, bd, go, rtol=1e-12, max_iters=its, restart=30)
        xG = m.to_active(H.to_host(xd))
        print(pname, its, 'hist G', hG, 'O', hO, 'x rel diff', np.linalg.norm(xG - xO) / np.linalg.norm(xO))
    # the preconditioner alone: mg_cycle from zero on b (mode 0) vs oracle cycle
    xd.zero_()
    H.cycle(xd, bd, go, norm=False)
    zG = m.to_active(H.to_host(xd)); zO = Oh.cycle(np.zeros_like(ba), ba, od)
    print(pname, 'cycle from zero rel diff', np.linalg.norm(zG - zO) / np.linalg.norm(zO))

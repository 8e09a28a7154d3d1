import sys, numpy as np
sys.path.insert(0, '.')
import mg_inputs
from tests import _cases as C
for n, pname in ((40, "stiff"), (66, "cfg5"), (16, "mixed")):
    H = C.gpu_hierarchy(n, 2, pname)
    r = mg_inputs.uniform_vector(n, 31); e = mg_inputs.uniform_vector(n // 2, 32); x = mg_inputs.uniform_vector(n, 33)
    rd, bc = H.to_device(r), H.zeros(1)
    H.restrict(0, rd, bc)
    ed, xd = H.to_device(e, 1), H.to_device(x)
    H.prolong(0, ed, xd)
    np.savez(f"gpurun_out/rp_{n}.npz", bG=H.to_host(bc, 1), xG=H.to_host(xd))
print("ok")

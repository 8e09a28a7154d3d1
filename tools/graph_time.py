import sys, time; sys.path.insert(0,'.')
import torch, mg_inputs
from paper_2107_04060_b200 import Hierarchy, Opts
c = mg_inputs.CONFIGS[5]
H = Hierarchy(c['n'], c['levels'], c['lam'], c['mu'], K=c['K'])
b = H.to_device(mg_inputs.uniform_rhs(c['n'], 5))
o = Opts(1,1,'vanka',0.7)
for k in range(3):
    x = H.zeros(); torch.cuda.synchronize()
    t0 = time.perf_counter(); H.cycle(x, b, o); torch.cuda.synchronize(); t1 = time.perf_counter()
    H.cycle(x, b, o); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"new x buffer: first cycle {1e3*(t1-t0):.1f} ms (capture+instantiate+run), second {1e3*(t2-t1):.1f} ms")
t0 = time.perf_counter(); H.fgmres(H.zeros(), b, o, rtol=1e-8, max_iters=1, restart=10); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"fgmres 1 iteration first call {1e3*(t1-t0):.1f} ms")

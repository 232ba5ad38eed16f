"""Dev helper: step-by-step smoke of each entry point with flushed progress."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
def p(*a): print(*a, flush=True)
t0 = time.time()
import torch
p("torch", torch.__version__, torch.cuda.is_available(), f"{time.time()-t0:.1f}s")
from paper_1512_08017_b200 import _capi, device as D
ctx = _capi.context(0)
p("ctx grid", ctx.grid_size())
for n in [1, 1000, 3584, 3585, 100000, 10**7]:
    xy = D.synth(n, 0, 1, 3, 0.1); torch.cuda.synchronize(); p("synth", n)
    for m in [0, 1, 3, 8]:
        r = D.read_result(D.fit(xy, m)); torch.cuda.synchronize()
        p("fit", n, m, r.status, r.n, list(r.s[:3]), list(r.coeffs[:2]))

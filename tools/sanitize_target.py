"""Small, fast exercise of every kernel for compute-sanitizer (one tool per run)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1512_08017_b200 import device as D, lsqfit as L, _capi
for n in (1, 3585, 100_003):
    xy = D.synth(n, 0, 1, 3, 0.1)
    for m in (0, 3, 8, 12):
        D.read_result(D.fit(xy, m))
parts = D.empty_result("cuda", 2)
xy = D.synth(50_001, 0, 1, 3, 0.1)
D.fit(xy[:20000], 3, flags=0, out=parts[:_capi.RESULT_BYTES]); D.fit(xy[20000:], 3, flags=0, out=parts[_capi.RESULT_BYTES:])
D.read_result(D.combine(parts, 2, 3))
D.read_diag(D.diagnostics(xy, 3, D.fit(xy, 3), residuals=torch.empty(50_001, dtype=torch.float64, device="cuda")))
for ppc in (1000, 1024, 7):
    xb = D.synth_batched(33, ppc, 5, 2, 0.1)
    D.fit_batched(xb, 33, ppc, 2)
L.solve_gaussian(L.NormalSystem(a=np.random.default_rng(1).standard_normal((40, 40)), b=np.ones(40), degree=39))
torch.cuda.synchronize()
print("sanitize target ok")

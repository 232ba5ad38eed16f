"""ncu target: one launch each of the secondary kernels at representative sizes —
diagnostics (n = 1e9, m = 3, with residuals), batched short curves (2^30 points,
ppc = 16, m = 2), reference-order warp kernel (n = 1e8, m = 3, 4096 chunks)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1512_08017_b200 import device as D  # noqa: E402

n = 10**9
xy = D.synth(n, 0, 4, 3, 0.1)
fr = D.fit(xy, 3)
res = torch.empty(n, dtype=torch.float64, device="cuda")
d = D.read_diag(D.diagnostics(xy, 3, fr, residuals=res))
print("diag", d.status, d.sse, d.r)
del res
xy8 = xy[:10**8]
r = D.read_result(D.fit_ordered(xy8, 3, 4096))
print("ordered", r.status, list(r.coeffs[:4]))
del xy, xy8
torch.cuda.empty_cache()
curves, ppc = (1 << 30) // 16, 16
xb = D.synth_batched(curves, ppc, 5, 2, 0.1)
c, s = D.fit_batched(xb, curves, ppc, 2)
torch.cuda.synchronize()
print("batched", int((s != 0).sum().item()))

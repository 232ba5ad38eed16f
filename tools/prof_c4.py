"""ncu target: one launch of the batched warp-per-curve kernel at BASELINE C4
(1e6 curves x 1024 points, m = 2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1512_08017_b200 import device as D  # noqa: E402

curves, ppc = 1_000_000, 1024
xb = D.synth_batched(curves, ppc, 5, 2, 0.1)
c, s = D.fit_batched(xb, curves, ppc, 2)
torch.cuda.synchronize()
print("C4 batched nonzero statuses:", int((s != 0).sum().item()))

"""Dev probe: per-launch latency of the fit / combine / solve kernels (CUDA events, back-to-back)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1512_08017_b200 import device as D

def t(fn, reps=200):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1000

xy = D.synth(1000, 0, 1, 3, 0.1)
for m in (0, 1, 3, 8, 12):
    out = D.empty_result("cuda"); part = D.empty_result("cuda")
    D.fit(xy, m, flags=0, out=part)
    print(m, "fit SOLVE %.1f us" % t(lambda: D.fit(xy, m, out=out)),
          "fit SUMS %.1f us" % t(lambda: D.fit(xy, m, flags=0, out=out)),
          "combine SOLVE %.1f us" % t(lambda: D.combine(part, 1, m, out=out)),
          "combine SUMS %.1f us" % t(lambda: D.combine(part, 1, m, flags=0, out=out)), flush=True)
x = torch.empty(1, device="cuda")
print("empty torch kernel %.1f us" % t(lambda: x.add_(1)))

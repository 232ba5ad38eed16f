import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1512_08017_b200 import device as D
def t(fn, reps=50):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1000
big = D.synth(1_000_000_000, 0, 1, 3, 0.1)
for m in (1, 3):
    out = D.empty_result("cuda")
    for n in (1000, 100_000, 1_000_000, 10_000_000, 30_000_000, 100_000_000, 300_000_000, 1_000_000_000):
        xy = big[:n]
        us = t(lambda: D.fit(xy, m, out=out))
        print(m, n, "%.1f us" % us, "%.0f GB/s" % (n*16/us/1e3), flush=True)

"""Batched-fit throughput vs points per curve (fixed 2^30 points total).
usage: python tools/batched_sweep.py [m] [ppc,ppc,...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1512_08017_b200 import device as D  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ppcs = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [3, 4, 8, 16, 32, 64, 128, 256, 1024, 4096]
total = 1 << 30
for ppc in ppcs:
    curves = total // ppc
    xy = D.synth_batched(curves, ppc, 5, min(m, 2), 0.1)
    c = torch.empty((curves, m + 1), dtype=torch.float64, device="cuda")
    s = torch.empty(curves, dtype=torch.int32, device="cuda")
    for _ in range(2):
        D.fit_batched(xy, curves, ppc, m, c, s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        D.fit_batched(xy, curves, ppc, m, c, s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    bytes_ = 16 * curves * ppc + curves * (8 * (m + 1) + 4)
    print(json.dumps({"m": m, "ppc": ppc, "curves": curves, "ms": round(ms, 3),
                      "curves_per_s": curves / ms * 1e3, "GBps": round(bytes_ / ms / 1e6),
                      "bad": int((s != 0).sum().item())}), flush=True)
    del xy, c, s
    torch.cuda.empty_cache()

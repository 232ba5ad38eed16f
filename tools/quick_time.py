"""Dev helper: CUDA-event timing of the fused fit kernel over degrees/sizes."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1512_08017_b200 import device as D

def t_fit(xy, m, reps=10):
    out = D.empty_result(xy.device)
    for _ in range(3): D.fit(xy, m, out=out)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record()
    for i in range(reps):
        D.fit(xy, m, out=out); ev[i + 1].record()
    torch.cuda.synchronize()
    ts = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(reps))
    r = D.read_result(out)
    return ts[len(ts) // 2], r.status

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**8
degs = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 3, 4, 6, 8, 12]
xy = D.synth(n, 0, 3, 3, 0.1)
for m in degs:
    ms, st = t_fit(xy, m)
    print(json.dumps({"n": n, "m": m, "ms": round(ms, 4), "pts_per_s": n / (ms * 1e-3), "GB_per_s": 16 * n / (ms * 1e-3) / 1e9, "status": st}))

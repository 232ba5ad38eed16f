"""Dev probe: host-path throughput (lsqfit_cuda_fit_host) for pinned vs pageable
inputs, and the small-n latency floor of the device path."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1512_08017_b200 import _capi, device as D

ctx = _capi.context(0)
res = {}
n = 200_000_000
xy_dev = D.synth(n, 0, 4, 3, 0.1)
pinned = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
pinned.copy_(xy_dev)
pageable = pinned.numpy().copy()
for name, ptr in (("pinned", pinned.data_ptr()), ("pageable", pageable.ctypes.data)):
    ctx.fit_host(ptr, n, 3, 1)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); st, r = ctx.fit_host(ptr, n, 3, 1); ts.append(time.perf_counter() - t0)
    res[name] = {"s": min(ts), "GB_per_s": 16 * n / min(ts) / 1e9, "status": st}
lat = {}
for k in (1, 1000, 100_000, 1_000_000, 10_000_000):
    out = D.empty_result("cuda")
    xs = xy_dev[:k]
    for _ in range(5): D.fit(xs, 1, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): D.fit(xs, 1, out=out)
    e1.record(); torch.cuda.synchronize()
    lat[k] = e0.elapsed_time(e1) / 50 * 1000
res["latency_us_m1"] = lat
print(json.dumps(res, indent=1))

"""Any-degree power sums (m > 12): device-resident generic kernel vs the
compiled reference's accumulate_parallel(d, m, 8*nproc) on this host.
usage: python tools/any_degree_perf.py [n] [m,m,...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1512_08017_b200 import _capi, device as D  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
degs = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [13, 16, 20, 32]
oracle.build()
xy = D.synth(n, 0, 4, 3, 0.1)
host = xy.cpu().numpy()
ctx = _capi.context(0)
stream = torch.cuda.current_stream().cuda_stream
nproc = os.cpu_count() or 1
for m in degs:
    st_buf = torch.empty(3 * m + 2, dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.power_sums_device(xy.data_ptr(), n, m, st_buf.data_ptr(), status.data_ptr(), stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        ctx.power_sums_device(xy.data_ptr(), n, m, st_buf.data_ptr(), status.data_ptr(), stream)
    e1.record()
    torch.cuda.synchronize()
    gpu_ms = e0.elapsed_time(e1) / 3
    t0 = time.perf_counter()
    st, s, t = oracle.ref_accumulate_parallel(host, m, 8 * nproc)
    cpu_s = time.perf_counter() - t0
    got = st_buf.cpu().numpy()
    rel = float(np.max(np.abs(got[: 2 * m + 1] - s) / np.maximum(np.abs(s), 1e-300)))
    print(json.dumps({"n": n, "m": m, "gpu_ms": round(gpu_ms, 3), "gpu_pts_per_s": n / gpu_ms * 1e3,
                      "reference_s": round(cpu_s, 3), "reference_pts_per_s": n / cpu_s, "cores": nproc,
                      "speedup": cpu_s * 1e3 / gpu_ms, "status": int(status.item()), "ref_status": st,
                      "max_rel_dev_s_vs_reference": rel}), flush=True)

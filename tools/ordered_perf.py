"""Dev probe: reference-order (bit-exact) mode throughput vs chunk count.
usage: python tools/ordered_perf.py [n] [chunks,chunks,...] [m,m,...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1512_08017_b200 import device as D  # noqa: E402


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**8
chunk_list = [int(float(v)) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2**12, 2**14, 2**16, 2**18, 2**20]
degs = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 3, 8]
xy = D.synth(n, 0, 4, 3, 0.1)
out = D.empty_result("cuda")
for m in degs:
    base = t(lambda: D.fit(xy, m, out=out))
    for c in chunk_list:
        ms = t(lambda: D.fit_ordered(xy, m, c, out=out), reps=1 if n // c > 10**6 else 3)
        print(json.dumps({"n": n, "m": m, "chunks": c, "ms": round(ms, 3), "GB_per_s": round(16 * n / ms / 1e6),
                          "fused_ms": round(base, 3)}), flush=True)

"""Per-launch device time of back-to-back fits replayed from a CUDA graph (no
host launch overhead in the measurement: small-n configs such as C1 are
otherwise bound by the Python/ctypes launch path, not by the GPU).
usage: python tools/graph_time.py n[,n..] m[,m..] [launches_per_graph]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1512_08017_b200 import device as D  # noqa: E402


def graph_us(xy, m, K=50, replays=20):
    s = torch.cuda.Stream()
    out = D.empty_result(xy.device)
    with torch.cuda.stream(s):
        for _ in range(3):
            D.fit(xy, m, out=out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(K):
            D.fit(xy, m, out=out)
    torch.cuda.synchronize()
    ts = []
    for r in range(replays + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1) * 1e3 / K)
    r = D.read_result(out)
    return statistics.median(ts), r


def main():
    ns = [int(float(v)) for v in sys.argv[1].split(",")]
    ms = [int(v) for v in sys.argv[2].split(",")]
    K = int(sys.argv[3]) if len(sys.argv) > 3 else 50
    big = D.synth(max(ns), 0, 1, 3, 0.1)
    rows = []
    for m in ms:
        for n in ns:
            us, r = graph_us(big[:n], m, K)
            rows.append({"n": n, "m": m, "us_per_fit": us, "pts_per_s": n / (us * 1e-6),
                         "GB_per_s": 16 * n / (us * 1e3), "status": int(r.status)})
            print(json.dumps(rows[-1]), flush=True)


if __name__ == "__main__":
    main()

"""C5 (n = 1e9, m = 1..12) measured robustly on one box: R rounds, each
round visits every degree once (so clock / power drift spreads over all
degrees), a sample = the median of K back-to-back launches (CUDA events).
Prints one JSON document: per degree the median / min / max over the rounds
in ms and as a fraction of the measured read ceiling.

    python tools/c5_repeat.py [rounds] [launches_per_sample]
"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import load_ceilings  # noqa: E402
from paper_1512_08017_b200 import device as D  # noqa: E402

N = 1_000_000_000
R = int(sys.argv[1]) if len(sys.argv) > 1 else 5
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
DEGREES = list(range(1, 13))


def sample(xy, m, out):
    for _ in range(2):
        D.fit(xy, m, out=out)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    ev[0].record()
    for i in range(K):
        D.fit(xy, m, out=out)
        ev[i + 1].record()
    torch.cuda.synchronize()
    return statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(K))


def main():
    ceil = load_ceilings()["read_stream_gbs"]
    xy = D.synth(N, 0, 6, 3, 0.1)
    out = D.empty_result(xy.device)
    ts = {m: [] for m in DEGREES}
    for r in range(R):
        order = DEGREES if r % 2 == 0 else DEGREES[::-1]
        for m in order:
            ts[m].append(sample(xy, m, out))
    res = {}
    for m in DEGREES:
        med = statistics.median(ts[m])
        res[str(m)] = {"ms_median": med, "ms_min": min(ts[m]), "ms_max": max(ts[m]),
                       "frac_read_ceiling_median": 16 * N / (med * 1e-3) / 1e9 / ceil,
                       "samples_ms": ts[m]}
    print(json.dumps({"device": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
                      "n": N, "rounds": R, "launches_per_sample": K, "read_ceiling_gbs": ceil, "C5": res}, indent=1))


if __name__ == "__main__":
    main()

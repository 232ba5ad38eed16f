"""A/B of dynamic-tail plans of power_sums_kernel in ONE process: settings
(den, chunk, min_tiles_per_cta) are switched between interleaved launches
through the dev hook lsqfit_debug_set_ps_tuning (0 = compiled default).
A fourth field toggles programmatic dependent launch (lsqfit_debug_set_ps_pdl,
default 1). usage: python tools/ab_dyn.py n[,n..] m[,m..] "den:chunk:min[:pdl] ..." [reps]"""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1512_08017_b200 import device as D, _capi  # noqa: E402

ns = [int(float(v)) for v in sys.argv[1].split(",")]
ms = [int(v) for v in sys.argv[2].split(",")]
settings = [tuple(int(x) for x in s.split(":")) for s in sys.argv[3].split()]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 40
lib = _capi.lib()
tune = lib.lsqfit_debug_set_ps_tuning
tune.argtypes = [C.c_int, C.c_int, C.c_int]
pdl = lib.lsqfit_debug_set_ps_pdl
pdl.argtypes = [C.c_int]


def apply(s):
    tune(*s[:3])
    pdl(s[3] if len(s) > 3 else 1)


big = D.synth(max(ns), 0, 4, 3, 0.1)
out = D.empty_result(big.device)
for n in ns:
    xy = big[:n]
    for m in ms:
        ts = {s: [] for s in settings}
        for r in range(reps + 2):
            order = settings if r % 2 == 0 else settings[::-1]
            for s in order:
                apply(s)
                # 5 back-to-back launches per sample (the bench's regime)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(5):
                    D.fit(xy, m, out=out)
                e1.record()
                torch.cuda.synchronize()
                if r >= 2:
                    ts[s].append(e0.elapsed_time(e1) / 5)
        apply((0, 0, 0, 1))
        base = statistics.median(ts[settings[0]])
        row = "  ".join(f"{':'.join(map(str, s))} {statistics.median(ts[s])*1e3:8.1f}us ({statistics.median(ts[s])/base:5.3f})"
                        for s in settings)
        print(f"n={n:.0e} m={m}  {row}", flush=True)
_ = _capi

"""Dev probe: per-CTA timeline of one power_sums launch (globaltimer stamps
from a -DLSQ_PS_TRACE build: entry, main loop end, ticket, last-CTA end).
  tools/build_variant.sh build/lib_trace.so -DLSQ_PS_TRACE
  LSQFIT_CUDA_LIB=build/lib_trace.so python tools/ps_trace.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1512_08017_b200 import _capi, device as D

lib = _capi.lib()
fn = lib.lsqfit_debug_ps_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
big = D.synth(1_000_000_000, 0, 1, 3, 0.1)
MS = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1,3,5,8").split(",")]
NS = [int(float(v)) for v in (sys.argv[2] if len(sys.argv) > 2 else "1e7,1e8,1e9").split(",")]
for m in MS:
    for n in NS:
        out = D.empty_result("cuda")
        xy = big[:n]
        for _ in range(3): D.fit(xy, m, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); D.fit(xy, m, out=out); e1.record(); torch.cuda.synchronize()
        tr = np.zeros((1024, 8), dtype=np.uint64)
        assert fn(tr.ctypes.data, 1024) == 0
        tile = 3584 if m <= 5 else 4096
        g = min(148, -(-n // tile))
        tr = tr[:g].astype(np.int64)
        t0 = tr[:, 0].min()
        rel = lambda c: (tr[:, c] - t0) / 1e3  # noqa: E731
        ent, le, tk, red, first = rel(0), rel(1), rel(2), rel(4), rel(6)
        last = tr[:, 3] > tr[:, 0]
        end = rel(3)[last]
        fin_red = rel(5)[last]
        print(f"m={m} n={n:.0e} event {e0.elapsed_time(e1)*1e3:.1f} us | grid {g} entry spread {ent.max():.1f} | "
              f"first tile med/max {np.median(first):.1f}/{first.max():.1f} | "
              f"loop end min/med/max {le.min():.1f}/{np.median(le):.1f}/{le.max():.1f} | "
              f"cta reduced med/max {np.median(red):.1f}/{red.max():.1f} | ticket med/max {np.median(tk):.1f}/{tk.max():.1f} | "
              f"last: slots reduced {fin_red.max() if fin_red.size else -1:.1f} end {end.max() if end.size else -1:.1f} us",
              flush=True)

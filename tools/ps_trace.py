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
for m in (1, 3, 5, 8):
    for n in (10_000_000, 100_000_000, 1_000_000_000):
        out = D.empty_result("cuda")
        xy = big[:n]
        for _ in range(3): D.fit(xy, m, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); D.fit(xy, m, out=out); e1.record(); torch.cuda.synchronize()
        tr = np.zeros((1024, 4), dtype=np.uint64)
        assert fn(tr.ctypes.data, 1024) == 0
        g = int((tr[:, 0] > 0).sum())
        tr = tr[:g].astype(np.int64)
        t0 = tr[:, 0].min()
        ent = (tr[:, 0] - t0) / 1e3; le = (tr[:, 1] - t0) / 1e3; tk = (tr[:, 2] - t0) / 1e3
        end = (tr[:, 3][tr[:, 3] > tr[:, 0]] - t0) / 1e3
        print(f"m={m} n={n:.0e} event {e0.elapsed_time(e1)*1e3:.1f} us | grid {g} entry spread {ent.max():.1f} | "
              f"loop end min/med/max {le.min():.1f}/{np.median(le):.1f}/{le.max():.1f} | ticket max {tk.max():.1f} | "
              f"last end {end.max() if end.size else -1:.1f} us", flush=True)

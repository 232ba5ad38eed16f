"""Dev probe: diagnostics pass (residuals/SSE/R) throughput vs the fit kernel."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1512_08017_b200 import device as D

def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**9
xy = D.synth(n, 0, 4, 3, 0.1)
res = torch.empty(n, dtype=torch.float64, device="cuda")
for m in (1, 3, 8):
    fr = D.fit(xy, m)
    fit_ms = t(lambda: D.fit(xy, m, out=fr))
    diag_ms = t(lambda: D.diagnostics(xy, m, fr))
    diag_res_ms = t(lambda: D.diagnostics(xy, m, fr, residuals=res))
    print(json.dumps({"n": n, "m": m, "fit_ms": round(fit_ms, 3), "diag_ms": round(diag_ms, 3),
                      "diag_with_residuals_ms": round(diag_res_ms, 3),
                      "diag_GBps": round(16 * n / diag_ms / 1e6), "diag_res_GBps": round(24 * n / diag_res_ms / 1e6)}), flush=True)

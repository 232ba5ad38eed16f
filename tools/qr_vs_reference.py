"""fit_qr (the reference's Householder-QR cross-check backend, qr_backend.cpp:126-133)
end to end from host memory: B200 TSQR drop-in vs the compiled reference.
usage: python tools/qr_vs_reference.py [n]   -> JSON (profiles/r01_qr_vs_reference.json)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1512_08017_b200 import lsqfit  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
oracle.build()
xy = oracle.synth(n, 0, 3, 3, 0.1)
d = lsqfit.Dataset._trusted(xy)
out = {"n": n, "input": "pageable host memory; residual vector returned by both"}
for m in (1, 3, 6, 8):
    lsqfit.fit_qr(d, m)
    t0 = time.perf_counter()
    rep = lsqfit.fit_qr(d, m)
    g = time.perf_counter() - t0
    t0 = time.perf_counter()
    st, c, sse, r = oracle.ref_fit_qr(xy, m)
    cpu = time.perf_counter() - t0
    gc = np.array(rep.polynomial.coefficients())
    out[f"m={m}"] = {"b200_s": g, "reference_s": cpu, "speedup": cpu / g, "ref_status": st,
                     "coeff_max_rel_diff": float(np.max(np.abs(gc - c) / np.maximum(np.abs(c), 1e-300))),
                     "sse_rel_diff": abs(rep.sse - sse) / sse}
print(json.dumps(out, indent=1))

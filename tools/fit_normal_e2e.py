"""fit_normal end to end — the reference's primary API (normal_backend.cpp:76-85:
sums + solve + make_fit_report with its residual vector) — on host (pageable)
data, B200 drop-in vs the compiled reference on this host's cores.

usage: python tools/fit_normal_e2e.py [n] [m]   (default BASELINE C2: n = 1e8, m = 3)
Prints one JSON document (profiles/r01_fit_normal_e2e.json)."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1512_08017_b200 import lsqfit  # noqa: E402


def timed(fn, reps):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts), out


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    oracle.build()
    xy = oracle.synth(n, 0, 3, 3, 0.1)  # BASELINE C2 seed for m = 3
    nproc = os.cpu_count() or 1
    d = lsqfit.Dataset._trusted(xy)
    gpu_s, rep = timed(lambda: lsqfit.fit_normal(d, m), 5)
    out = {"n": n, "m": m, "input": "pageable host memory (std::vector-like), residual vector returned",
           "b200_drop_in": {"median_s": gpu_s, "pts_per_s": n / gpu_s, "sse": rep.sse, "r": rep.r,
                            "coeffs": list(rep.polynomial.coefficients())}}
    if oracle.have_ref():
        rd = oracle.RefDataset(xy)
        for chunks in (1, nproc, 8 * nproc):
            reps = 1 if chunks == 1 else 3
            s, (st, c, sse, r) = timed(lambda: rd.fit_normal(m, chunks), reps)
            out[f"reference_chunks={chunks}"] = {
                "median_s": s, "pts_per_s": n / s, "status": st, "sse": sse, "r": r,
                "coeff_max_rel_vs_b200": float(np.max(np.abs(c - np.array(rep.polynomial.coefficients()))
                                                      / np.abs(c))),
                "speedup_of_b200": s / gpu_s}
        out["cores"] = nproc
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

"""Secondary measurements (BASELINE.json configs other than the bench line):

  C1  linear fit, n = 1e6                      (oracle config; launch-bound)
  C2  quadratic and cubic fit, n = 1e8
  C4  batched: 1e6 curves x 1024 points, m = 2
  C5  degree sweep m = 1..12 at n = 1e9         (HBM -> FP64 crossover)

Device time with CUDA events (median of reps, after warm-up), plus accuracy
against the exact-sum oracle on a 1e8 prefix and the reference CPU path timed
on this host. Prints one JSON document (write it to profiles/).
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (checker only)
from paper_1512_08017_b200 import device as D  # noqa: E402

from bench import load_ceilings  # noqa: E402  (profiles/measured_ceilings.json)

U = 2.0 ** -53
_CEIL = load_ceilings()
FP64_PEAK = _CEIL["dadd_ops_per_s"]
READ_CEIL = _CEIL["read_stream_gbs"]


def time_it(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record()
    for i in range(reps):
        fn()
        ev[i + 1].record()
    torch.cuda.synchronize()
    ts = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(reps))
    return ts[len(ts) // 2]


def fp64_ops(m):
    return 5 * m


def single(n, m, seed, reps=20, acc_prefix=None):
    xy = D.synth(n, 0, seed, min(m, 3), 0.1)
    out = D.empty_result(xy.device)
    ms = time_it(lambda: D.fit(xy, m, out=out), reps=reps)
    r = D.read_result(out)
    rec = {"n": n, "m": m, "seed": seed, "ms": ms, "pts_per_s": n / (ms * 1e-3),
           "GB_per_s": 16 * n / (ms * 1e-3) / 1e9, "frac_read_ceiling": 16 * n / (ms * 1e-3) / 1e9 / READ_CEIL,
           "fp64_frac": fp64_ops(m) * n / (ms * 1e-3) / FP64_PEAK, "status": int(r.status),
           "coeffs": [float(c) for c in r.coeffs[: m + 1]]}
    if acc_prefix:
        k = min(n, acc_prefix)
        host = xy[:k].cpu().numpy()
        rr = D.read_result(D.fit(xy[:k], m))
        from paper_1512_08017_b200 import _capi
        s_hi, s_lo, s_abs, t_hi, t_lo, t_abs = oracle.kernel_exact_sums(
            host, m, _capi.sum_terms(m) == _capi.TERMS_PRODUCTS)
        got = np.concatenate([np.array(rr.s[1: 2 * m + 1]), np.array(rr.t[: m + 1])])
        hi = np.concatenate([s_hi[1:], t_hi])
        lo = np.concatenate([s_lo[1:], t_lo])
        ab = np.concatenate([s_abs[1:], t_abs])
        err = np.abs((got - hi) - lo)
        st, ex = oracle.solve_from_sums(s_hi + s_lo, t_hi + t_lo, m)
        c = np.array(rr.coeffs[: m + 1])
        ref_acc = oracle.ref_accumulate_parallel if oracle.have_ref() else oracle.accumulate_parallel
        ref_st, ref_s, ref_t = ref_acc(host, m, 8 * (os.cpu_count() or 1))
        ref_err = np.abs((np.concatenate([ref_s[1:], ref_t]) - hi) - lo)
        rec["accuracy"] = {
            "prefix_points": k,
            "max_sum_err_in_u_sum_abs": float(np.max(err / (U * ab))),
            "ref_cpu_max_sum_err_in_u_sum_abs": float(np.max(ref_err / (U * ab))),
            "coeff_max_rel_vs_exact_sum_solve": float(np.max(np.abs(c - ex) / np.maximum(np.abs(ex), 1e-300))),
            "kappa_A": float(np.linalg.cond(oracle.build_normal_system(s_hi + s_lo, m))),
        }
    del xy
    torch.cuda.empty_cache()
    return rec


def batched(n_curves, ppc, m, seed=5, reps=10):
    xy = D.synth_batched(n_curves, ppc, seed, m, 0.1)
    coeffs = torch.empty((n_curves, m + 1), dtype=torch.float64, device="cuda")
    status = torch.empty(n_curves, dtype=torch.int32, device="cuda")
    ms = time_it(lambda: D.fit_batched(xy, n_curves, ppc, m, coeffs, status), reps=reps)
    n = n_curves * ppc
    # accuracy + the reference's own per-curve loop (oracle/_ref: Dataset ->
    # accumulate -> build_normal_system -> solve_gaussian, OpenMP over curves)
    # timed on this host over ALL curves
    k = n_curves
    host = xy[: k * ppc].cpu().numpy()
    kind = "reference" if oracle.have_ref() else "port"
    loop = oracle.ref_fit_batched if kind == "reference" else oracle.fit_batched
    t0 = time.perf_counter()
    rc, rst = loop(host, k, ppc, m)
    cpu_s = time.perf_counter() - t0
    c = coeffs[:k].cpu().numpy()
    st = status[:k].cpu().numpy()
    ok = rst == 0
    err = np.max(np.max(np.abs(c[ok] - rc[ok]), axis=1) / np.max(np.abs(rc[ok]), axis=1))
    rec = {"n_curves": n_curves, "ppc": ppc, "m": m, "ms": ms, "curves_per_s": n_curves / (ms * 1e-3),
           "pts_per_s": n / (ms * 1e-3), "GB_per_s": 16 * n / (ms * 1e-3) / 1e9,
           "frac_read_ceiling": 16 * n / (ms * 1e-3) / 1e9 / READ_CEIL,
           "status_all_ok": bool((status == 0).all().item()), "status_match_prefix": bool((st == rst).all()),
           "coeff_max_normwise_rel_vs_cpu_loop": float(err),
           "cpu_reference_loop": {"kind": kind, "cores": oracle.max_threads(), "curves": k,
                                  "curves_per_s": k / cpu_s, "pts_per_s": k * ppc / cpu_s}}
    del xy
    torch.cuda.empty_cache()
    return rec


def tsqr(n, m, seed=6, reps=10):
    """TSQR cross-check backend throughput (flops: ~2(m+2)^2 per row of Givens work)."""
    xy = D.synth(n, 0, seed, min(m, 3), 0.1)
    out = D.empty_qr_result(xy.device)
    ms = time_it(lambda: D.qr_fit(xy, m, out=out), reps=reps)
    q = D.read_qr_result(out)
    ne = D.read_result(D.fit(xy, m))
    c, cn = np.array(q.coeffs[: m + 1]), np.array(ne.coeffs[: m + 1])
    rec = {"n": n, "m": m, "ms": ms, "rows_per_s": n / (ms * 1e-3), "GB_per_s": 16 * n / (ms * 1e-3) / 1e9,
           "status": int(q.status), "coeff_max_rel_vs_normal_eq": float(np.max(np.abs(c - cn)) / np.max(np.abs(cn)))}
    del xy
    torch.cuda.empty_cache()
    return rec


def graph_c1(n=1_000_000, m=1):
    """Small launches are bound by the host launch path from Python; the
    device time per fit comes from K launches replayed in a CUDA graph
    (tools/graph_bench.cpp, C ABI from C++)."""
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.abspath(__file__)), "graph_bench")
    p = subprocess.run([exe, str(n), str(m), "50"], capture_output=True, text=True, timeout=300, check=True)
    return json.loads(p.stdout.strip().splitlines()[-1])


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "tsqr":
        print(json.dumps({"TSQR": [tsqr(1_000_000_000, m) for m in (1, 2, 3, 4, 6, 8, 9, 10, 12)]}, indent=1))
        return
    out = {"device": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    out["C1"] = single(1_000_000, 1, 1, reps=50, acc_prefix=1_000_000)
    out["C1"]["graph_replay"] = graph_c1()
    out["C2_graph_replay"] = [graph_c1(100_000_000, m) for m in (2, 3)]
    out["C2"] = [single(100_000_000, 2, 2, acc_prefix=100_000_000), single(100_000_000, 3, 3, acc_prefix=100_000_000)]
    out["C4"] = batched(1_000_000, 1024, 2)
    out["C5"] = [single(1_000_000_000, m, 6, reps=10, acc_prefix=20_000_000) for m in range(1, 13)]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

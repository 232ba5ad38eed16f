"""TEST INFRASTRUCTURE ONLY — regenerate tests/golden/*.json from the compiled reference.

Run in the dev container (where /root/reference exists):

    make -C oracle && python oracle/make_golden.py

Every number in the fixtures is produced by the reference's own code
(oracle/_ref/libref_lsqfit.so, built from /root/reference/proj/src by
oracle/Makefile) and stored as exact IEEE-754 hex strings, so the GPU box —
which has no /root/reference — can check bit-exact parity against them.
"""
from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")

# tests/support/table1.hpp:13-19
TABLE1 = [(39.206, 751.912), (29.74, 567.121), (21.31, 403.746),
          (12.087, 221.738), (1.812, 18.8418), (0.001, 1.88672)]


def hx(v) -> list[str] | str:
    if np.ndim(v) == 0:
        return float(v).hex()
    return [float(x).hex() for x in np.asarray(v).ravel()]


def digest(xy: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(xy, dtype=np.float64).tobytes()).hexdigest()


def main() -> None:
    if not O.have_ref():
        raise SystemExit("oracle/_ref not built: run `make -C oracle` with /root/reference present")
    os.makedirs(GOLDEN, exist_ok=True)

    # ---------------- Table I (paper Tables I-IV) -----------------------------
    t1 = {"points": hx(np.array(TABLE1)), "by_degree": {}}
    for m in range(0, 4):
        st, s, t = O.ref_accumulate(TABLE1, m)
        assert st == 0
        entry = {"s": hx(s), "t": hx(t)}
        for chunks in (1, 2, 3, 16):
            st, sp, tp = O.ref_accumulate_parallel(TABLE1, m, chunks)
            entry[f"par{chunks}"] = {"s": hx(sp), "t": hx(tp)}
        ks, kt = O.ref_accumulate_oracle(TABLE1, m)
        entry["kahan_pow"] = {"s": hx(ks), "t": hx(kt)}
        if m >= 1:
            st, c, sse, r = O.ref_fit_normal(TABLE1, m)
            assert st == 0
            entry["fit"] = {"coeffs": hx(c), "sse": hx(sse), "r": hx(r)}
        t1["by_degree"][str(m)] = entry
    with open(os.path.join(GOLDEN, "table1.json"), "w") as f:
        json.dump(t1, f, indent=1)

    # ------------- reference generate_synthetic datasets + their sums ---------
    # Seeds/sizes are the ones the reference's hot-path tests use
    # (test_accumulator.cpp:70,90,109-110,126; test_normal_backend.cpp:48,99,151,175,187,229).
    synth_cases = [
        (10001, 4, 0.3, 11), (1000000, 4, 0.1, 2024), (501, 3, 0.2, 5), (499, 3, 0.2, 6),
        (20000, 5, 0.4, 8), (64, 5, 0.2, 3), (200, 4, 0.1, 1), (200, 4, 0.1, 2),
        (5000, 3, 0.2, 77), (300, 5, 0.1, 10), (150, 4, 0.3, 66), (100, 1, 0.0, 1),
    ]
    out = []
    for n, m, sigma, seed in synth_cases:
        xy = O.ref_generate_synthetic(n, m, sigma, seed)
        port = O.generate_synthetic(n, m, sigma, seed)
        assert np.array_equal(xy.view(np.uint64), port.view(np.uint64)), "mt19937_64 port diverged"
        st, s, t = O.ref_accumulate(xy, m)
        rec = {"n": n, "degree": m, "sigma": sigma, "seed": seed, "sha256": digest(xy),
               "head": hx(xy[:4]), "s": hx(s), "t": hx(t), "par": {}}
        for chunks in (1, 2, 4, 8):
            st, sp, tp = O.ref_accumulate_parallel(xy, m, chunks)
            rec["par"][str(chunks)] = {"s": hx(sp), "t": hx(tp)}
        st, c, sse, r = O.ref_fit_normal(xy, m)
        rec["fit"] = {"status": st, "coeffs": hx(c), "sse": hx(sse), "r": hx(r)}
        out.append(rec)
    with open(os.path.join(GOLDEN, "synthetic_ref.json"), "w") as f:
        json.dump(out, f, indent=1)

    # ---------------- solve_gaussian hand cases (test_normal_backend.cpp:57-126) --
    solve_cases = [
        ("identity", [[1, 0], [0, 1]], [3, 7]),
        ("2x2", [[2, 1], [1, 3]], [5, 10]),
        ("zero_leading_pivot", [[0, 1], [1, 0]], [2, 5]),
        ("all_equal_x_singular", [[3, 6], [6, 12]], [15, 30]),
        ("zero_matrix", [[0.0]], [0.0]),
        ("pivot_tie", [[1, 2, 3], [-1, 5, 1], [1, 0, 7]], [1, 2, 3]),
        ("needs_swap", [[1e-3, 1, 2], [4, 1, 0], [2, 8, 1]], [1, 0, -1]),
    ]
    rng = np.random.default_rng(7)
    for d in (3, 5, 8, 13, 20):
        a = rng.standard_normal((d, d))
        solve_cases.append((f"random{d}", a.tolist(), rng.standard_normal(d).tolist()))
    solve = []
    for name, a, b in solve_cases:
        a = np.array(a, dtype=np.float64)
        b = np.array(b, dtype=np.float64)
        st, x = O.ref_solve_gaussian(a, b)
        pst, px = O.solve_gaussian(a, b)
        assert st == pst and (st != 0 or np.array_equal(x.view(np.uint64), px.view(np.uint64)))
        solve.append({"name": name, "a": hx(a), "b": hx(b), "dim": int(b.shape[0]), "status": st,
                      "x": hx(x) if st == 0 else None})
    with open(os.path.join(GOLDEN, "solve.json"), "w") as f:
        json.dump(solve, f, indent=1)

    # --------- counter-based generator: digests of the host twin -----------------
    # (Not a reference artefact — the reference generator is mt19937_64 — but the
    # device generator must reproduce these bits, and the reference's own sums on
    # these inputs are recorded so the GPU parity tests can use them.)
    gen = []
    for n, off, seed, deg, sigma in [(1000, 0, 1, 1, 0.1), (4096 * 3 + 17, 12345, 3, 3, 0.1),
                                     (100000, 0, 6, 8, 0.1), (77, 1 << 33, 4, 3, 0.1)]:
        xy = O.synth(n, off, seed, deg, sigma)
        st, s, t = O.ref_accumulate(xy, deg)
        gen.append({"n": n, "offset": off, "seed": seed, "truth_degree": deg, "sigma": sigma,
                    "sha256": digest(xy), "head": hx(xy[:2]), "ref_s": hx(s), "ref_t": hx(t)})
    bt = O.synth_batched(64, 1024, 5, 2, 0.1)
    coeffs, status = O.fit_batched(bt, 64, 1024, 2)
    gen.append({"batched": True, "n_curves": 64, "ppc": 1024, "seed": 5, "truth_degree": 2,
                "sigma": 0.1, "sha256": digest(bt), "coeffs": hx(coeffs), "status": status.tolist()})
    with open(os.path.join(GOLDEN, "counter_synth.json"), "w") as f:
        json.dump(gen, f, indent=1)

    # ----------------- QR cross-check backend (fit_qr, qr_backend.cpp:126-133) ---
    qr = []
    qr_cases = [("table1", np.array(TABLE1), m) for m in (1, 2, 3)]
    for n, m, sigma, seed in [(300, 5, 0.1, 10), (5000, 3, 0.2, 77), (2000, 8, 0.05, 9), (150, 4, 0.3, 66)]:
        qr_cases.append((f"synthetic_{n}_{m}_{seed}", O.ref_generate_synthetic(n, m, sigma, seed), m))
    qr_cases.append(("counter_20000_m8", O.synth(20000, 0, 31, 8, 0.1), 8))
    qr_cases.append(("one_distinct_x", np.array([(2.0, 1.0), (2.0, 3.0), (2.0, 5.0)]), 1))
    qr_cases.append(("too_few_points", np.array([(0.0, 1.0), (1.0, 2.0)]), 2))
    for name, xy, m in qr_cases:
        st, c, sse, r = O.ref_fit_qr(xy, m)
        qr.append({"name": name, "degree": m, "points": hx(xy), "status": st,
                   "coeffs": hx(c) if st == 0 else None, "sse": hx(sse) if st == 0 else None,
                   "r": hx(r) if st == 0 else None})
    with open(os.path.join(GOLDEN, "qr_fits.json"), "w") as f:
        json.dump(qr, f, indent=1)

    # ----------------------- misc known answers ---------------------------------
    misc = {}
    st, s, t = O.ref_accumulate([(0.0, 0.0), (1.0, 1.0)], 1)
    misc["two_point"] = {"s": hx(s), "t": hx(t)}
    st, s, t = O.ref_accumulate([(1.0, 1.0)] * 37, 5)
    misc["ones37_m5"] = {"s": hx(s), "t": hx(t)}
    st, s, t = O.ref_accumulate([(2.0, 3.0), (4.0, 5.0)], 0)
    misc["degree0"] = {"s": hx(s), "t": hx(t)}
    st, s, t = O.ref_accumulate([(1e200, 1.0), (1e200, 2.0), (1.0, 3.0)], 2)
    misc["overflow_status"] = st
    st, c, sse, r = O.ref_fit_normal([(0.0, 1.0), (2.0, 5.0)], 1)
    misc["interp2"] = {"coeffs": hx(c), "sse": hx(sse)}
    cheb = [(math.cos(i * 3.14159265358979323846 / 99.0), math.sin(3.0 * math.cos(i * 3.14159265358979323846 / 99.0)))
            for i in range(100)]
    st, c, sse, r = O.ref_fit_normal(cheb, 12)
    misc["cheb12"] = {"status": st, "points": hx(np.array(cheb)), "coeffs": hx(c)}
    with open(os.path.join(GOLDEN, "misc.json"), "w") as f:
        json.dump(misc, f, indent=1)
    print("golden fixtures written to", GOLDEN)


if __name__ == "__main__":
    main()

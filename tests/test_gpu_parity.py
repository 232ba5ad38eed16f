"""GPU parity: the sm_100a path (through the C ABI) against the oracle, the
golden reference fixtures and the reference's own test contracts
(test_accumulator.cpp, test_normal_backend.cpp)."""
import hashlib

import numpy as np
import pytest

from paper_1512_08017_b200 import _capi

from conftest import TABLE1, bitwise_equal, load_golden, max_rel_dev, unhex, kernel_sums

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


@pytest.fixture(scope="module")
def L():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1512_08017_b200 import lsqfit
    return lsqfit


@pytest.fixture(scope="module")
def D():
    from paper_1512_08017_b200 import device
    return device


def sums(L, pts, m):
    r = L.accumulate(L.Dataset(pts), m)
    return np.array(r.s), np.array(r.t), r


def check_bound(O, xy, m, s, t, p_levels):
    """|S_gpu - S_exact| <= gamma_{levels} * sum|T| + 1 ulp(S_exact) (+ O(u^2) slack)."""
    s_hi, s_lo, s_abs, t_hi, t_lo, t_abs = kernel_sums(O, xy, m)
    ex_s = s_hi + s_lo
    ex_t = t_hi + t_lo
    g = p_levels * U / (1 - p_levels * U)
    worst = 0.0
    for got, ex, hi, lo, ab in ((s[1:], ex_s[1:], s_hi[1:], s_lo[1:], s_abs[1:]), (t, ex_t, t_hi, t_lo, t_abs)):
        if len(got) == 0:  # degree 0 has no s[k >= 1]
            continue
        err = np.abs((got - hi) - lo)
        bound = g * ab + np.spacing(np.abs(ex)) + 1e-30 * ab + 1e-300
        assert (err <= bound).all(), (err, bound)
        worst = max(worst, float(np.max(err / np.maximum(ab * U, 1e-300))))
    return worst


# ------------------------------------------------------- generator parity ----

def test_device_generator_bit_identical_to_host(D, oracle_mod):
    for rec in load_golden("counter_synth.json"):
        if rec.get("batched"):
            xy = D.synth_batched(rec["n_curves"], rec["ppc"], rec["seed"], rec["truth_degree"], rec["sigma"])
        else:
            xy = D.synth(rec["n"], rec["offset"], rec["seed"], rec["truth_degree"], rec["sigma"])
        got = hashlib.sha256(xy.cpu().numpy().tobytes()).hexdigest()
        assert got == rec["sha256"]


# ------------------------------------- test_accumulator.cpp contracts ------

def test_two_point_hand_case(L):
    s, t, r = sums(L, [(0.0, 0.0), (1.0, 1.0)], 1)
    assert list(s) == [2.0, 1.0, 1.0] and list(t) == [1.0, 1.0] and r.n == 2


def test_table1_degree1_sums(L, oracle_mod):
    s, t, _ = sums(L, TABLE1, 1)
    assert s[0] == 6.0
    assert abs(s[1] - 104.156) <= 1e-9
    assert abs(t[0] - 1965.24552) <= 1e-6
    ks, kt = oracle_mod.kahan_pow_sums(TABLE1, 1)
    assert (np.abs(s - ks) <= 1e-12 * np.abs(ks)).all()
    assert (np.abs(t - kt) <= 1e-12 * np.abs(kt)).all()


def test_table1_sums_vs_golden_reference(L):
    g = load_golden("table1.json")
    for m, e in g["by_degree"].items():
        s, t, _ = sums(L, TABLE1, int(m))
        assert max_rel_dev(s, unhex(e["s"])) <= 1e-14 and max_rel_dev(t, unhex(e["t"])) <= 1e-14


def test_flat_sums_for_ones(L):
    s, t, _ = sums(L, [(1.0, 1.0)] * 37, 5)
    assert (s == 37).all() and (t == 37).all()


def test_accumulate_parallel_one_chunk_bitwise(L, oracle_mod):
    d = L.Dataset(oracle_mod.generate_synthetic(10001, 4, 0.3, 11))
    a = L.accumulate(d, 4)
    b = L.accumulate_parallel(d, 4, 1)
    assert bitwise_equal(a.s, b.s) and bitwise_equal(a.t, b.t)


def test_million_points_across_chunks(L, oracle_mod):
    rec = [r for r in load_golden("synthetic_ref.json") if r["n"] == 1000000][0]
    xy = oracle_mod.generate_synthetic(1000000, 4, 0.1, 2024)
    assert hashlib.sha256(xy.tobytes()).hexdigest() == rec["sha256"]
    d = L.Dataset(xy)
    seq = L.accumulate(d, 4)
    # vs the reference's own sequential and chunked sums (golden): <= 1e-9 (test_accumulator.cpp:89-98)
    assert max_rel_dev(seq.s, unhex(rec["s"])) <= 1e-9 and max_rel_dev(seq.t, unhex(rec["t"])) <= 1e-9
    for chunks in (2, 4, 8):
        par = L.accumulate_parallel(d, 4, chunks)
        assert max_rel_dev(seq.s, par.s) <= 1e-9 and max_rel_dev(seq.t, par.t) <= 1e-9
        assert par.s[0] == 1000000.0
        e = rec["par"][str(chunks)]
        assert max_rel_dev(par.s, unhex(e["s"])) <= 1e-9 and max_rel_dev(par.t, unhex(e["t"])) <= 1e-9
    check_bound(oracle_mod, xy, 4, np.array(seq.s), np.array(seq.t), _capi.sum_error_levels(4))


def test_more_chunks_than_points(L):
    d = L.Dataset([(1.0, 2.0), (3.0, 4.0), (5.0, 6.0)])
    seq = L.accumulate(d, 2)
    par = L.accumulate_parallel(d, 2, 16)
    assert max_rel_dev(seq.s, par.s) <= 1e-12 and par.s[0] == 3.0
    assert list(seq.s) == [3.0, 9.0, 35.0, 153.0, 707.0]


def test_concatenation_adds(L, oracle_mod):
    d1 = oracle_mod.generate_synthetic(501, 3, 0.2, 5)
    d2 = oracle_mod.generate_synthetic(499, 3, 0.2, 6)
    a, b = L.accumulate(L.Dataset(d1), 3), L.accumulate(L.Dataset(d2), 3)
    w = L.accumulate(L.Dataset(np.concatenate([d1, d2])), 3)
    for k in range(7):
        assert abs(w.s[k] - (a.s[k] + b.s[k])) <= 1e-12 * abs(w.s[k])
    for j in range(4):
        assert abs(w.t[j] - (a.t[j] + b.t[j])) <= 1e-12 * max(abs(w.t[j]), 1.0)


def test_permutation_roundoff_only(L, oracle_mod):
    pts = oracle_mod.generate_synthetic(20000, 5, 0.4, 8)
    base = L.accumulate(L.Dataset(pts), 5)
    rng = np.random.default_rng(31)
    for _ in range(5):
        sh = pts[rng.permutation(len(pts))]
        r = L.accumulate(L.Dataset(sh), 5)
        assert max_rel_dev(base.s, r.s) <= 1e-9 and max_rel_dev(base.t, r.t) <= 1e-9


def test_degree_zero(L):
    s, t, _ = sums(L, [(2.0, 3.0), (4.0, 5.0)], 0)
    assert list(s) == [2.0] and list(t) == [8.0]


def test_overflow_is_an_error(L):
    d = L.Dataset([(1e200, 1.0), (1e200, 2.0), (1.0, 3.0)])
    with pytest.raises(L.OverflowError):
        L.accumulate(d, 2)
    with pytest.raises(L.OverflowError):
        L.accumulate_parallel(d, 2, 2)


def test_argument_validation(L):
    d = L.Dataset([(0.0, 0.0), (1.0, 1.0)])
    with pytest.raises(ValueError):
        L.accumulate(d, -1)
    with pytest.raises(ValueError):
        L.accumulate_parallel(d, 1, 0)
    with pytest.raises(ValueError):
        L.Dataset([])
    with pytest.raises(ValueError):
        L.Dataset([(0.0, float("nan"))])


# ---------------------------------------------- accuracy vs exact oracle ----

@pytest.mark.parametrize("n,m,seed", [(1, 3, 1), (2, 2, 2), (3583, 3, 3), (3584, 3, 4), (3585, 3, 5),
                                      (1000000, 1, 1), (1234567, 2, 2), (2000003, 3, 3), (777777, 6, 6),
                                      (777777, 7, 7), (500001, 8, 6), (300007, 12, 8),
                                      # long carried partials (many tiles per CTA per fold)
                                      (20000003, 8, 9), (8000001, 12, 10), (30000001, 5, 11)])
def test_sums_within_stated_ulp_bound(L, oracle_mod, n, m, seed):
    xy = oracle_mod.synth(n, 0, seed, min(m, 3), 0.1)
    r = L.accumulate(L.Dataset(xy), m)
    assert r.s[0] == float(n)
    levels = _capi.sum_error_levels(m)  # the library's stated bound
    assert levels == (5 if m <= 2 else 10 if m <= 4 else 16 if m == 5 else 17)
    check_bound(oracle_mod, xy, m, np.array(r.s), np.array(r.t), levels)


def _tile_points(m):
    """Points per ring tile of power_sums_kernel<m> (csrc/power_sums.cuh PsCfg):
    7 consumer warps + a producer for m <= 5, 8 self-feeding warps with
    column-split lane pairs from m = 6; P = 16 points per thread."""
    return (8 if m >= 6 else 7) * 32 * 16


@pytest.mark.parametrize("m", [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12])
def test_tile_and_grid_boundaries_every_feed_mode(L, oracle_mod, m):
    """Ragged last tile, fewer tiles than CTAs, fewer tiles than ring stages,
    and carried partials left over at the end of a CTA's range, for each
    (feed, P, tiles-per-fold) shape."""
    T, G = _tile_points(m), 148
    levels = _capi.sum_error_levels(m)
    for n in (1, T - 1, T, T + 1, 3 * T + 5, G * T - 1, G * T + 1, G * T * 11 + 17):
        xy = oracle_mod.synth(n, 0, 100 + m, min(m, 3), 0.1)
        r = L.accumulate(L.Dataset(xy), m)
        assert r.s[0] == float(n)
        check_bound(oracle_mod, xy, m, np.array(r.s), np.array(r.t), levels)


@pytest.mark.parametrize("m", [0, 1, 2, 3, 4, 5])
def test_dynamic_tail_schedule(D, oracle_mod, m):
    """Producer-fed degrees m <= 5 deal the tail of the tiles in dynamically
    claimed chunks (csrc/power_sums.cuh, PsCfg::DYN; device-resident data —
    the host path streams smaller launches): from 32 tiles per CTA the
    mid-size plan (last 1/8 in 16-tile chunks), from 1024 tiles per CTA the
    long plan (last 1/2, halving chunks down to 8 tiles; k_power_sums.cu).
    Just below and above each threshold, with the ragged last tile inside a
    chunk, the sums stay within the stated bound and bit-identical launch to
    launch (each chunk has its own record, whichever CTA claimed it)."""
    import torch
    T, G = _tile_points(m), 148
    levels = _capi.sum_error_levels(m)
    mid, long_ = 32 * G * T, 1024 * G * T
    for n in ((mid - 1, mid + 1, long_ - 1, long_ + 1) if m in (1, 3) else (mid + 1, long_ + 1)):
        xy = D.synth(n, 0, 300 + m, min(m, 3), 0.1)
        out = D.empty_result(xy.device)
        D.fit(xy, m, flags=0, out=out)
        r = D.read_result(out)
        assert r.status == 0 and r.n == n and r.s[0] == float(n)
        s_, t_ = np.array(r.s[: 2 * m + 1]), np.array(r.t[: m + 1])
        check_bound(oracle_mod, xy.cpu().numpy(), m, s_, t_, levels)
        for _ in range(3):
            D.fit(xy, m, flags=0, out=out)
            b = D.read_result(out)
            assert bitwise_equal(list(r.s[: 2 * m + 1]), list(b.s[: 2 * m + 1])), n
            assert bitwise_equal(list(r.t[: m + 1]), list(b.t[: m + 1])), n
        del xy
        torch.cuda.empty_cache()


def test_deterministic_run_to_run(L, oracle_mod):
    d = L.Dataset(oracle_mod.synth(3000001, 0, 77, 3, 0.1))
    a = L.accumulate(d, 3)
    for _ in range(3):
        b = L.accumulate(d, 3)
        assert bitwise_equal(a.s, b.s) and bitwise_equal(a.t, b.t)


@pytest.mark.parametrize("m,n", [(1, 1000000), (2, 2000000), (3, 4000000)])
def test_coefficients_within_1e10_of_exact_sum_oracle(L, oracle_mod, m, n):
    """North star: coefficients <= 1e-10 relative for m <= 3, x in [-1, 1]."""
    xy = oracle_mod.synth(n, 0, 40 + m, m, 0.1)
    rep = L.fit_normal(L.Dataset(xy), m)
    s_hi, s_lo, _, t_hi, t_lo, _ = kernel_sums(oracle_mod, xy, m)
    st, ex = oracle_mod.solve_from_sums(s_hi + s_lo, t_hi + t_lo, m)
    assert st == 0
    c = np.array(rep.polynomial.coefficients())
    assert np.max(np.abs(c - ex) / np.maximum(np.abs(ex), 1e-300)) <= 1e-10
    # and against the reference CPU path's own coefficients on the same data
    st, refc = oracle_mod.fit_normal(xy, m, 64)
    assert st == 0 and np.max(np.abs(c - refc) / np.abs(refc)) <= 1e-9


# ------------------------------------------ test_normal_backend.cpp ---------

def test_solve_bitwise_equals_reference_golden(L):
    for case in load_golden("solve.json"):
        dim = case["dim"]
        sys_ = L.NormalSystem(a=unhex(case["a"]).reshape(dim, dim), b=unhex(case["b"]), degree=dim - 1)
        if case["status"] == 0:
            p = L.solve_gaussian(sys_)
            assert bitwise_equal(p.coefficients(), unhex(case["x"])), case["name"]
        else:
            with pytest.raises(L.SingularSystemError):
                L.solve_gaussian(sys_)


def test_fused_solve_bitwise_equals_reference_solve_on_same_sums(L, oracle_mod):
    """The in-kernel solve mirrors solve_gaussian op for op (no contraction)."""
    for m in range(0, 13):
        xy = oracle_mod.synth(100003, 0, 300 + m, min(m, 4), 0.1)
        rep_sums = L.accumulate(L.Dataset(xy), m)
        rep = L.fit_normal(L.Dataset(xy), m)
        st, x = oracle_mod.solve_from_sums(np.array(rep_sums.s), np.array(rep_sums.t), m)
        if st == 0:
            assert bitwise_equal(rep.polynomial.coefficients(), x), m
        if oracle_mod.have_ref():
            rst, rx = oracle_mod.ref_solve_from_sums(np.array(rep_sums.s), np.array(rep_sums.t), m)
            assert rst == st and (st != 0 or bitwise_equal(rx, x))


def test_identity_pivot_and_singular(L):
    p = L.solve_gaussian(L.NormalSystem(a=np.eye(2), b=np.array([3.0, 7.0]), degree=1))
    assert p.coefficients() == [3.0, 7.0]
    p = L.solve_gaussian(L.NormalSystem(a=np.array([[0.0, 1.0], [1.0, 0.0]]), b=np.array([2.0, 5.0]), degree=1))
    assert p.coefficients() == [5.0, 2.0]
    p = L.solve_gaussian(L.NormalSystem(a=np.array([[2.0, 1.0], [1.0, 3.0]]), b=np.array([5.0, 10.0]), degree=1))
    assert abs(p.coefficients()[0] - 1.0) <= 1e-14 and abs(p.coefficients()[1] - 3.0) <= 1e-14
    d = L.Dataset([(2.0, 5.0)] * 3)
    with pytest.raises(L.SingularSystemError):
        L.solve_gaussian(L.build_normal_system(L.accumulate(d, 1)))
    with pytest.raises(L.SingularSystemError):
        L.solve_gaussian(L.NormalSystem(a=np.zeros((1, 1)), b=np.zeros(1), degree=0))
    with pytest.raises(L.SingularSystemError):
        L.fit_normal(d, 1)


def test_solve_random_systems_bitwise(L, oracle_mod):
    rng = np.random.default_rng(11)
    # up to 160x160 the system sits in shared memory, beyond it in global memory
    for dim in (1, 3, 13, 31, 32, 33, 64, 100, 128, 129, 161, 200, 333):
        a = rng.standard_normal((dim, dim))
        b = rng.standard_normal(dim)
        st, x = oracle_mod.solve_gaussian(a, b)
        if st == 0:
            p = L.solve_gaussian(L.NormalSystem(a=a, b=b, degree=dim - 1))
            assert bitwise_equal(p.coefficients(), x), dim
    with pytest.raises(ValueError):
        L.solve_gaussian(L.NormalSystem(a=np.eye(4097), b=np.ones(4097), degree=4096))


def test_build_normal_system_structure(L, oracle_mod):
    d = L.Dataset(oracle_mod.generate_synthetic(64, 5, 0.2, 3))
    sys_ = L.build_normal_system(L.accumulate(d, 5))
    a = sys_.a
    assert (a == a.T).all()
    for j in range(5):
        for k in range(1, 6):
            assert a[j, k] == a[j + 1, k - 1]
    sys7 = L.build_normal_system(L.accumulate(L.Dataset([(1.0, 2.0)] * 7), 3))
    assert (sys7.a == 7.0).all()


def test_fit_normal_reproduces_paper_tables(L):
    g = load_golden("table1.json")["by_degree"]
    d = L.Dataset(TABLE1)
    want = {1: [-8.356, 19.3496], 2: [-6.5106, 18.8735, 0.0127], 3: [-4.7553, 17.5105, 0.1086, -0.0016]}
    tol = {1: [5e-3, 5e-4], 2: [1e-3] * 3, 3: [1e-3] * 4}
    for m in (1, 2, 3):
        rep = L.fit_normal(d, m)
        c = rep.polynomial.coefficients()
        for k in range(m + 1):
            assert abs(c[k] - want[m][k]) <= tol[m][k]
        ref = g[str(m)]["fit"]
        assert max_rel_dev(c, unhex(ref["coeffs"])) <= 1e-9
        assert abs(rep.sse - unhex(ref["sse"])) <= 1e-9 * unhex(ref["sse"])
        assert abs(rep.r - unhex(ref["r"])) <= 1e-12
        assert rep.backend == "normal"
    assert abs(L.fit_normal(d, 3).sse - 128.1999) <= 0.05


def test_fit_normal_interpolates_two_points(L):
    rep = L.fit_normal(L.Dataset([(0.0, 1.0), (2.0, 5.0)]), 1)
    assert rep.polynomial.coefficients() == [1.0, 2.0]
    assert rep.sse <= 1e-24


def test_fit_normal_degree_cap_and_chebyshev12(L, oracle_mod):
    d = L.Dataset(oracle_mod.generate_synthetic(100, 1, 0.0, 1))
    with pytest.raises(L.DegreeTooHighError):
        L.fit_normal(d, 13)
    with pytest.raises(ValueError):
        L.fit_normal(d, -1)
    i = np.arange(100)
    x = np.cos(i * 3.14159265358979323846 / 99.0)
    L.fit_normal(L.Dataset(np.stack([x, np.sin(3.0 * x)], 1)), 12)  # must not throw


def test_fit_normal_zero_gradient(L, oracle_mod):
    for seed in (10, 11, 12):
        xy = oracle_mod.generate_synthetic(300, 5, 0.1, seed)
        rep = L.fit_normal(L.Dataset(xy), 5)
        c = np.array(rep.polynomial.coefficients())
        x, y = xy[:, 0], xy[:, 1]
        f = np.polyval(c[::-1], x)
        g = [abs(np.sum(x ** j * (y - f))) for j in range(6)]
        b = [abs(np.sum(x ** j * y)) for j in range(6)]
        assert max(g) / (1 + max(b)) <= 1e-6


def test_fit_normal_sse_monotone_in_degree(L, oracle_mod):
    for seed in (21, 22, 23, 24, 25):
        d = L.Dataset(oracle_mod.generate_synthetic(120, 3, 0.1, seed))
        prev = None
        for m in range(7):
            sse = L.fit_normal(d, m).sse
            if prev is not None:
                assert sse <= prev + 1e-9 * (1 + prev)
            prev = sse


def test_fit_normal_interpolates_m_plus_one_points(L):
    rng = np.random.default_rng(2025)
    for m in range(7):
        xs = [0.5] if m == 0 else [i / m for i in range(m + 1)]
        ys = rng.uniform(-1, 1, m + 1)
        rep = L.fit_normal(L.Dataset(np.stack([xs, ys], 1)), m)
        assert np.max(np.abs(rep.residuals)) <= 1e-8 * (1 + np.max(np.abs(ys)))


def test_fit_normal_translation_and_scaling(L, oracle_mod):
    rng = np.random.default_rng(55)
    pts = rng.uniform(-5, 5, (100, 2))
    sse0 = L.fit_normal(L.Dataset(pts), 3).sse
    for shift in (-10.0, -1.0, 1.0, 10.0):
        moved = pts.copy()
        moved[:, 0] += shift
        assert abs(L.fit_normal(L.Dataset(moved), 3).sse - sse0) <= 1e-6 * sse0
    base = oracle_mod.generate_synthetic(150, 4, 0.3, 66)
    c0 = np.array(L.fit_normal(L.Dataset(base), 4).polynomial.coefficients())
    for alpha in (-1.0, 2.0, 10.0):
        sc = base.copy()
        sc[:, 1] *= alpha
        c1 = np.array(L.fit_normal(L.Dataset(sc), 4).polynomial.coefficients())
        assert (np.abs(c1 - alpha * c0) <= 1e-9 * (1 + np.abs(alpha * c0))).all()


def test_fit_normal_chunked_changes_nothing(L, oracle_mod):
    d = L.Dataset(oracle_mod.generate_synthetic(5000, 3, 0.2, 77))
    a = L.fit_normal(d, 3, 1).polynomial.coefficients()
    b = L.fit_normal(d, 3, 4).polynomial.coefficients()
    assert all(abs(x - y) <= 1e-9 * (1 + abs(x)) for x, y in zip(a, b))


def test_fit_report_residuals_sse_r_vs_reference(L, oracle_mod):
    for rec in load_golden("synthetic_ref.json"):
        if rec["degree"] < 1 or rec["n"] > 20000:
            continue
        xy = oracle_mod.generate_synthetic(rec["n"], rec["degree"], rec["sigma"], rec["seed"])
        rep = L.fit_normal(L.Dataset(xy), rec["degree"])
        c = np.array(rep.polynomial.coefficients())
        assert max_rel_dev(c, unhex(rec["fit"]["coeffs"])) <= 1e-8
        sse = unhex(rec["fit"]["sse"])
        assert abs(rep.sse - sse) <= 1e-9 * (1 + sse)
        assert abs(rep.r - unhex(rec["fit"]["r"])) <= 1e-9
        # residuals: y - Horner(x), same rounding as the reference's evaluate()
        acc = np.full(len(xy), c[-1])
        for k in range(len(c) - 2, -1, -1):
            acc = acc * xy[:, 0] + c[k]
        assert bitwise_equal(rep.residuals, xy[:, 1] - acc)


@pytest.mark.parametrize("big", [1e160, 3e153, 1.5e154])
def test_fit_report_huge_finite_residual(L, oracle_mod, big):
    """Finite residuals whose squares overflow (1e160), or whose SST overflows
    (1.5e154): the reference returns sse=+inf (plain sum, diagnostics.cpp:21-25)
    and R from max(0, 1 - sse/sst) with sst=+inf, and throws only for
    NON-finite residuals (:42-44) — so no OverflowError here."""
    pts = np.array([(0.0, 0.0), (1.0, 0.0), (2.0, 0.0), (3.0, big), (4.0, 0.0)])
    rep = L.fit_normal(L.Dataset(pts), 1)
    assert all(np.isfinite(rep.residuals))
    expect = {1e160: (float("inf"), 0.0), 3e153: (6.300000000000001e+306, 0.3535533905932738),
              1.5e154: (1.5750000000000003e+308, 1.0)}[big]  # oracle/_ref (the compiled reference)
    if oracle_mod.have_ref():
        st, c, sse, r = oracle_mod.ref_fit_normal(pts, 1)
        assert st == 0 and (sse, r) == expect
    sse, r = expect
    assert rep.sse == sse or abs(rep.sse - sse) <= 1e-12 * sse
    assert abs(rep.r - r) <= 1e-12


# ------------------------------------------------- device-resident path ----

def test_device_path_matches_host_path_bitwise(L, D, oracle_mod):
    import torch
    xy_h = oracle_mod.synth(2500000, 0, 4, 3, 0.1)
    host = L.fit_normal(L.Dataset(xy_h), 3)
    xy = torch.from_numpy(xy_h).cuda()
    out = D.fit(xy, 3)
    torch.cuda.synchronize()
    r = D.read_result(out)
    assert r.status == 0 and r.n == 2500000
    assert bitwise_equal(list(r.coeffs[:4]), host.polynomial.coefficients())


def test_sharded_combine(L, D, oracle_mod):
    import torch
    n, m = 3000017, 3
    xy = D.synth(n, 0, 12, 3, 0.1)
    whole = D.read_result(D.fit(xy, m))
    for G in (1, 2, 3, 8):
        parts = D.empty_result(xy.device, G)
        for g in range(G):
            lo, hi = n * g // G, n * (g + 1) // G
            D.fit(xy[lo:hi], m, flags=0, out=parts[g * D._capi.RESULT_BYTES:(g + 1) * D._capi.RESULT_BYTES])
        comb = D.read_result(D.combine(parts, G, m))
        assert comb.n == n and comb.status == 0
        if G == 1:
            assert bitwise_equal(list(comb.s[:7]), list(whole.s[:7]))
        assert max_rel_dev(list(comb.coeffs[:4]), list(whole.coeffs[:4])) <= 1e-12
        check_bound(oracle_mod, D.synth(n, 0, 12, 3, 0.1).cpu().numpy(), m, np.array(comb.s[:7]),
                    np.array(comb.t[:4]), 5)


def test_empty_shard_is_neutral(D):
    import torch
    xy = D.synth(1000, 0, 1, 1, 0.1)
    empty = torch.empty((0, 2), dtype=torch.float64, device="cuda")
    r = D.read_result(D.fit(empty, 1, flags=0))
    assert r.n == 0 and r.status == 0 and all(v == 0.0 for v in r.s[:3])
    parts = D.empty_result(xy.device, 2)
    D.fit(xy, 1, flags=0, out=parts[:D._capi.RESULT_BYTES])
    D.fit(empty, 1, flags=0, out=parts[D._capi.RESULT_BYTES:])
    comb = D.read_result(D.combine(parts, 2, 1))
    single = D.read_result(D.fit(xy, 1))
    assert bitwise_equal(list(comb.coeffs[:2]), list(single.coeffs[:2]))


def test_context_scratch_ordered_across_streams(L, D, oracle_mod):
    """One context serves the host path (its private stream) and device-path
    launches on any caller stream; they share per-context scratch (slots,
    tickets), so launches are chained across streams (claim_scratch) and never
    overlap: results stay bit-identical to isolated runs."""
    import torch
    big = D.synth(300_000_000, 0, 21, 3, 0.1)
    big2 = D.synth(200_000_000, 0, 22, 3, 0.1)
    small = L.Dataset(oracle_mod.synth(100_000, 0, 23, 3, 0.1))
    want_big = D.read_result(D.fit(big, 3))
    want_big2 = D.read_result(D.fit(big2, 5))
    want_small = L.accumulate(small, 3)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(10):
        with torch.cuda.stream(s1):
            o1 = D.fit(big, 3)  # asynchronous, ~1 ms
        with torch.cuda.stream(s2):
            o2 = D.fit(big2, 5)  # another stream, same context
        r = L.accumulate(small, 3)  # host path, issued while both may still run
        torch.cuda.synchronize()
        a, b = D.read_result(o1), D.read_result(o2)
        assert bitwise_equal(list(a.s[:7]), list(want_big.s[:7]))
        assert bitwise_equal(list(b.s[:11]), list(want_big2.s[:11]))
        assert bitwise_equal(r.s, want_small.s) and bitwise_equal(r.t, want_small.t)


@pytest.mark.parametrize("m", [13, 20, 47])
def test_any_degree_accumulate(L, oracle_mod, m):
    """The reference's accumulate has no degree cap: above the fused kernels'
    12 the generic kernel forms the same terms (exact multiplication chain)
    and sums them compensated — within a few u * sum|T| of exact, and within
    the reference's 1e-9 of its own plain sums; chunked host streaming gives
    the same sums."""
    from paper_1512_08017_b200 import _capi
    n = 200_003
    xy = oracle_mod.synth(n, 0, 40 + m, 3, 0.1)
    d = L.Dataset(xy)
    r = L.accumulate(d, m)
    assert r.degree == m and len(r.s) == 2 * m + 1 and len(r.t) == m + 1 and r.s[0] == float(n)
    check_bound(oracle_mod, xy, m, np.array(r.s), np.array(r.t), 4)
    st, s_ref, t_ref = oracle_mod.accumulate(xy, m)
    assert st == 0
    assert max_rel_dev(r.s, s_ref) <= 1e-9 or np.allclose(r.s, s_ref, rtol=1e-9, atol=1e-9 * n)
    assert bitwise_equal(L.accumulate_parallel(d, m, 5).s, r.s)
    try:
        _capi.context(0).set_stream_chunk(70_001)  # out of core: 3 chunks
        rs = L.accumulate(d, m)
    finally:
        _capi.context(0).set_stream_chunk(0)
    check_bound(oracle_mod, xy, m, np.array(rs.s), np.array(rs.t), 4)


def test_any_degree_overflow_and_validation(L):
    big = L.Dataset([(1.0, 1.0)] * 10 + [(10.0, 1.0)])
    with pytest.raises(L.OverflowError):
        L.accumulate(big, 200)  # 10^400 overflows, as in the reference (require_finite)
    r = L.accumulate(L.Dataset([(1.0, 2.0)] * 7), 30)
    assert all(v == 7.0 for v in r.s) and all(v == 14.0 for v in r.t)
    with pytest.raises(ValueError):
        L.accumulate(big, -1)


@pytest.mark.parametrize("m", [3, 12, 13, 25])
def test_report_any_degree(L, oracle_mod, m):
    """residuals / make_fit_report / correlation_coefficient (diagnostics.cpp
    :14-48) for any polynomial degree: residuals bit-identical to the
    reference's Horner on the host, SSE and R against the oracle's report."""
    rng = np.random.default_rng(m)
    n = 100_003
    xy = oracle_mod.synth(n, 0, 60 + m, 3, 0.1)
    d = L.Dataset(xy)
    c = list(rng.uniform(-1, 1, m + 1) * 10.0 ** -np.arange(m + 1) * 0.5)
    poly = L.Polynomial(c)
    res = L.residuals(d, poly)
    acc = np.full(n, c[-1])
    for k in range(m - 1, -1, -1):
        acc = acc * xy[:, 0] + c[k]
    assert bitwise_equal(res, xy[:, 1] - acc)
    rep = L.make_fit_report(d, poly)
    sse = float(np.sum((xy[:, 1] - acc) ** 2))
    assert abs(rep.sse - sse) <= 1e-12 * sse
    ybar = np.mean(xy[:, 1])
    sst = float(np.sum((xy[:, 1] - ybar) ** 2))
    r_ref = np.sqrt(max(0.0, 1.0 - sse / sst))
    assert abs(rep.r - r_ref) <= 1e-12 and abs(L.correlation_coefficient(d, sse) - r_ref) <= 1e-12
    assert rep.n_points == n and bitwise_equal(rep.residuals, res)


def test_fit_facade_both_backends(L, oracle_mod):
    """fit.cpp:34-57: Both -> normal then QR report, discrepancy and agreement."""
    xy = oracle_mod.generate_synthetic(5000, 3, 0.05, 7)
    out = L.fit(L.Dataset(xy), 3, backend="both", chunks=4)
    assert [r.backend for r in out.reports] == ["normal", "qr"]
    assert out.backends_agree and out.max_coef_discrepancy < 1e-8
    assert L.fit(L.Dataset(xy), 2).reports[0].backend == "normal"
    with pytest.raises(ValueError):
        L.fit(L.Dataset(xy), 2, backend="lu")


def test_solve_sums_abi_matches_reference(L, oracle_mod):
    """lsqfit_cuda_solve_sums_host (build_normal_system + solve_gaussian from
    sums) gives the reference's solve bits for the same sums."""
    import ctypes as C
    from paper_1512_08017_b200 import _capi
    for m in (0, 1, 3, 8, 12, 20):
        xy = oracle_mod.synth(50_000, 0, 5 + m, min(m, 3), 0.1)
        st, s, t = oracle_mod.accumulate(xy, m)
        ref_st, x = oracle_mod.solve_from_sums(s, t, m)
        out = np.zeros(m + 1)
        dp = C.POINTER(C.c_double)
        ctx = _capi.context(0)
        got = ctx._lib.lsqfit_cuda_solve_sums_host(ctx.h, s.ctypes.data_as(dp), t.ctypes.data_as(dp), m,
                                                  out.ctypes.data_as(dp))
        assert got == ref_st, m
        if ref_st == 0:
            assert bitwise_equal(out, x), m


@pytest.mark.parametrize("m", [3, 5, 8, 12])
def test_repeated_launches_bit_identical(D, m):
    """Every feed mode (producer warp, self-feed, column split): 24 back-to-back
    launches on the same data give the same record bits (no pipeline race)."""
    import torch
    n = 150_000_001
    xy = D.synth(n, 0, 77, 3, 0.1)
    B = _capi.RESULT_BYTES
    outs = torch.zeros(24 * B, dtype=torch.uint8, device=xy.device)
    for i in range(24):
        D.fit(xy, m, out=outs[i * B:(i + 1) * B])
    rows = outs.view(24, B)
    assert bool((rows == rows[0:1]).all().item())
    assert D.read_result(outs).status == 0


def test_device_entry_point_validation(D):
    """Device entry points: misaligned or NULL pointers and bad degrees give
    EINVAL (nothing launched); n = 0 is an empty record (used by empty shards)."""
    import torch
    ctx = _capi.context(0)
    xy = D.synth(1000, 0, 1, 3, 0.1)
    out = D.empty_result(xy.device)
    stream = torch.cuda.current_stream().cuda_stream
    L = ctx._lib
    assert L.lsqfit_cuda_fit_device(ctx.h, xy.data_ptr() + 8, 999, 3, 1, out.data_ptr(), stream) == _capi.EINVAL
    assert L.lsqfit_cuda_fit_device(ctx.h, xy.data_ptr(), 1000, 13, 1, out.data_ptr(), stream) == _capi.EINVAL
    assert L.lsqfit_cuda_fit_device(ctx.h, xy.data_ptr(), 1000, 3, 1, None, stream) == _capi.EINVAL
    assert L.lsqfit_cuda_fit_batched_device(ctx.h, xy.data_ptr(), 10, 0, 2, out.data_ptr(), out.data_ptr(),
                                            stream) == _capi.EINVAL
    # n = 0: an empty SUMS record (zero sums, n = 0) — what an empty shard contributes
    assert L.lsqfit_cuda_fit_device(ctx.h, None, 0, 3, _capi.SUMS, out.data_ptr(), stream) == _capi.OK
    r = D.read_result(out)
    assert r.n == 0 and r.status == 0 and all(v == 0.0 for v in r.s[:7]) and all(v == 0.0 for v in r.t[:4])

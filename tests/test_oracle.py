"""CPU: pin the oracle (test infrastructure) to the reference before trusting it.

* against the golden fixtures made from the compiled reference
  (oracle/make_golden.py -> tests/golden/*.json) — runs everywhere;
* against the compiled reference itself (oracle/_ref) on fresh random inputs
  — runs where oracle/_ref exists;
* the double-double exact-sum oracle against exact rational arithmetic.
"""
import hashlib
import math
from fractions import Fraction

import numpy as np
import pytest

from conftest import TABLE1, bitwise_equal, load_golden, unhex


def digest(xy):
    return hashlib.sha256(np.ascontiguousarray(xy, dtype=np.float64).tobytes()).hexdigest()


# ---------------------------------------------------------------- golden ----

def test_table1_sums_and_fits_match_reference_bits(oracle_mod):
    g = load_golden("table1.json")
    for m, e in g["by_degree"].items():
        m = int(m)
        st, s, t = oracle_mod.accumulate(TABLE1, m)
        assert st == 0
        assert bitwise_equal(s, unhex(e["s"])) and bitwise_equal(t, unhex(e["t"]))
        for chunks in (1, 2, 3, 16):
            st, s, t = oracle_mod.accumulate_parallel(TABLE1, m, chunks)
            assert bitwise_equal(s, unhex(e[f"par{chunks}"]["s"]))
            assert bitwise_equal(t, unhex(e[f"par{chunks}"]["t"]))
        ks, kt = oracle_mod.kahan_pow_sums(TABLE1, m)
        assert bitwise_equal(ks, unhex(e["kahan_pow"]["s"])) and bitwise_equal(kt, unhex(e["kahan_pow"]["t"]))
        if m >= 1:
            st, c = oracle_mod.fit_normal(TABLE1, m)
            assert st == 0 and bitwise_equal(c, unhex(e["fit"]["coeffs"]))


def test_table1_matches_survey_golden_vectors(oracle_mod):
    # degree-3 s/t and normal-path coefficients on Table I.
    st, s, t = oracle_mod.accumulate(TABLE1, 3)
    assert list(s) == [6, 104.15600000000001, 3025.07305, 98017.038830648002, 3372567.5558183366,
                       120550025.81553388, 4420414550.8308372]
    assert list(t) == [1965.2455199999999, 57663.758106319998, 1873176.2942356199, 64529583.154778928]
    coeffs = {1: [-8.3559866531075571, 19.349643226685409],
              2: [-6.510928235141118, 18.873513826966992, 0.012734034058870953],
              3: [-4.7551083966032817, 17.51093799773647, 0.10857202524918211, -0.0016173860909198452]}
    for m, want in coeffs.items():
        st, c = oracle_mod.fit_normal(TABLE1, m)
        assert list(c) == want


def test_mt19937_generate_synthetic_port_matches_reference_datasets(oracle_mod):
    for rec in load_golden("synthetic_ref.json"):
        if rec["n"] > 100000:
            continue  # the 1e6 case is covered on the GPU box
        xy = oracle_mod.generate_synthetic(rec["n"], rec["degree"], rec["sigma"], rec["seed"])
        assert digest(xy) == rec["sha256"]
        st, s, t = oracle_mod.accumulate(xy, rec["degree"])
        assert bitwise_equal(s, unhex(rec["s"])) and bitwise_equal(t, unhex(rec["t"]))
        for chunks, e in rec["par"].items():
            st, s, t = oracle_mod.accumulate_parallel(xy, rec["degree"], int(chunks))
            assert bitwise_equal(s, unhex(e["s"])) and bitwise_equal(t, unhex(e["t"]))
        st, c = oracle_mod.fit_normal(xy, rec["degree"])
        assert st == rec["fit"]["status"]
        assert bitwise_equal(c, unhex(rec["fit"]["coeffs"]))


def test_solve_gaussian_golden_cases(oracle_mod):
    for case in load_golden("solve.json"):
        a = unhex(case["a"]).reshape(case["dim"], case["dim"])
        b = unhex(case["b"])
        st, x = oracle_mod.solve_gaussian(a, b)
        assert st == case["status"], case["name"]
        if st == 0:
            assert bitwise_equal(x, unhex(case["x"])), case["name"]


def test_misc_known_answers(oracle_mod):
    g = load_golden("misc.json")
    st, s, t = oracle_mod.accumulate([(0.0, 0.0), (1.0, 1.0)], 1)
    assert list(s) == [2.0, 1.0, 1.0] and list(t) == [1.0, 1.0]
    assert bitwise_equal(s, unhex(g["two_point"]["s"]))
    st, s, t = oracle_mod.accumulate([(1.0, 1.0)] * 37, 5)
    assert (s == 37).all() and (t == 37).all()
    st, s, t = oracle_mod.accumulate([(2.0, 3.0), (4.0, 5.0)], 0)
    assert list(s) == [2.0] and list(t) == [8.0]
    st, _, _ = oracle_mod.accumulate([(1e200, 1.0), (1e200, 2.0), (1.0, 3.0)], 2)
    assert st == oracle_mod.EOVERFLOW == g["overflow_status"]
    st, c = oracle_mod.fit_normal([(0.0, 1.0), (2.0, 5.0)], 1)
    assert list(c) == [1.0, 2.0]
    cheb = unhex(g["cheb12"]["points"]).reshape(-1, 2)
    st, c = oracle_mod.fit_normal(cheb, 12)
    assert st == g["cheb12"]["status"] == 0 and bitwise_equal(c, unhex(g["cheb12"]["coeffs"]))
    assert oracle_mod.accumulate([(0.0, 0.0)], -1)[0] == oracle_mod.EINVAL
    assert oracle_mod.accumulate_parallel([(0.0, 0.0)], 1, 0)[0] == oracle_mod.EINVAL
    assert oracle_mod.fit_normal([(0.0, 0.0), (1.0, 1.0)], 13)[0] == oracle_mod.EDEGREE


def test_counter_generator_digests(oracle_mod):
    for rec in load_golden("counter_synth.json"):
        if rec.get("batched"):
            xy = oracle_mod.synth_batched(rec["n_curves"], rec["ppc"], rec["seed"], rec["truth_degree"],
                                          rec["sigma"])
            assert digest(xy) == rec["sha256"]
            c, st = oracle_mod.fit_batched(xy, rec["n_curves"], rec["ppc"], rec["truth_degree"])
            assert bitwise_equal(c.ravel(), unhex(rec["coeffs"])) and st.tolist() == rec["status"]
        else:
            xy = oracle_mod.synth(rec["n"], rec["offset"], rec["seed"], rec["truth_degree"], rec["sigma"])
            assert digest(xy) == rec["sha256"]
            assert (xy[:, 0] >= -1).all() and (xy[:, 0] < 1).all()
            st, s, t = oracle_mod.accumulate(xy, rec["truth_degree"])
            assert bitwise_equal(s, unhex(rec["ref_s"])) and bitwise_equal(t, unhex(rec["ref_t"]))


def test_counter_generator_is_sliceable(oracle_mod):
    whole = oracle_mod.synth(5000, 0, 9, 3, 0.1)
    parts = np.concatenate([oracle_mod.synth(1234, 0, 9, 3, 0.1), oracle_mod.synth(5000 - 1234, 1234, 9, 3, 0.1)])
    assert bitwise_equal(whole, parts)


# ----------------------------------------------------- exact-sum oracle ----

def test_exact_sums_against_rationals(oracle_mod):
    xy = oracle_mod.synth(3000, 0, 21, 3, 0.1)
    m = 3
    s_hi, s_lo, s_abs, t_hi, t_lo, t_abs = oracle_mod.exact_sums(xy, m)
    S = [Fraction(0)] * (2 * m + 1)
    T = [Fraction(0)] * (m + 1)
    A = [0.0] * (2 * m + 1)
    for x, y in xy:
        p = 1.0
        for k in range(2 * m + 1):
            S[k] += Fraction(p)
            A[k] += abs(p)
            if k <= m:
                T[k] += Fraction(p * y)  # the reference's rounded term
            p = p * x
    for k in range(2 * m + 1):
        err = abs(Fraction(s_hi[k]) + Fraction(s_lo[k]) - S[k])
        assert err <= Fraction(2.0 ** -100) * Fraction(A[k] + 1)
        assert s_abs[k] == pytest.approx(A[k], rel=1e-12)
    for j in range(m + 1):
        err = abs(Fraction(t_hi[j]) + Fraction(t_lo[j]) - T[j])
        assert err <= Fraction(2.0 ** -100) * Fraction(float(t_abs[j]) + 1)


def test_exact_sums_terms_against_rationals(oracle_mod):
    """Both term families of the CUDA kernel (the reference's rounded terms,
    and the fused-multiply-add mode's exact products pw_{k//2} * pw_{k-k//2}
    and pw_j * y) summed exactly, checked with rational arithmetic; the plain
    family is bit-identical to exact_sums()."""
    xy = oracle_mod.synth(2000, 0, 23, 3, 0.1)
    m = 6
    g = oracle_mod.exact_sums_terms(xy, m)
    ref = oracle_mod.exact_sums(xy, m)
    assert all((a == b).all() for a, b in zip(ref, oracle_mod.kernel_term_sums(g, m, False)))
    SX = [Fraction(0)] * (2 * m + 1)
    TX = [Fraction(0)] * (m + 1)
    for x, y in xy:
        pw = [1.0]
        for k in range(1, 2 * m + 1):
            pw.append(pw[-1] * x)
        for k in range(2 * m + 1):
            a = k // 2
            SX[k] += Fraction(pw[a]) * Fraction(pw[k - a]) if k >= 2 else Fraction(pw[k])
        for j in range(m + 1):
            TX[j] += Fraction(pw[j]) * Fraction(float(y))
    for k in range(2 * m + 1):
        err = abs(Fraction(g["sx"][0][k]) + Fraction(g["sx"][1][k]) - SX[k])
        assert err <= Fraction(2.0 ** -100) * Fraction(float(g["sx"][2][k]) + 1)
    for j in range(m + 1):
        err = abs(Fraction(g["tx"][0][j]) + Fraction(g["tx"][1][j]) - TX[j])
        assert err <= Fraction(2.0 ** -100) * Fraction(float(g["tx"][2][j]) + 1)
    # kernel_term_sums(products=True): plain powers up to m, products above
    s_hi = oracle_mod.kernel_term_sums(g, 3, True)[0]
    assert (s_hi[:4] == g["sp"][0][:4]).all() and (s_hi[4:] == g["sx"][0][4:7]).all()


# -------------------------------------------- port vs compiled reference ----

needs_ref = pytest.mark.skipif("not __import__('oracle').have_ref()", reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("m", [0, 1, 2, 3, 5, 8, 12])
def test_port_bitwise_equals_reference(oracle_mod, m):
    rng = np.random.default_rng(100 + m)
    xy = np.stack([rng.uniform(-1.5, 1.5, 20011), rng.standard_normal(20011)], axis=1)
    st, s, t = oracle_mod.accumulate(xy, m)
    rst, rs, rt = oracle_mod.ref_accumulate(xy, m)
    assert st == rst and bitwise_equal(s, rs) and bitwise_equal(t, rt)
    for chunks in (1, 2, 7, 64, 30000):
        st, s, t = oracle_mod.accumulate_parallel(xy, m, chunks)
        rst, rs, rt = oracle_mod.ref_accumulate_parallel(xy, m, chunks)
        assert st == rst and bitwise_equal(s, rs) and bitwise_equal(t, rt)
    if 1 <= m <= 12:
        st, c = oracle_mod.fit_normal(xy, m)
        rst, rc, _, _ = oracle_mod.ref_fit_normal(xy, m)
        assert st == rst and (st != 0 or bitwise_equal(c, rc))


@needs_ref
def test_port_solve_bitwise_equals_reference_random(oracle_mod):
    rng = np.random.default_rng(3)
    for dim in (1, 2, 4, 9, 13, 40):
        for _ in range(5):
            a = rng.standard_normal((dim, dim))
            if dim > 2:
                a[1] = a[0]  # a tie / near-singular row now and then
                a[1, -1] += 1e-3
            b = rng.standard_normal(dim)
            st, x = oracle_mod.solve_gaussian(a, b)
            rst, rx = oracle_mod.ref_solve_gaussian(a, b)
            assert st == rst and (st != 0 or bitwise_equal(x, rx))


def test_isfinite_and_threads(oracle_mod):
    assert oracle_mod.max_threads() >= 1
    assert math.isfinite(oracle_mod.synth(10, 0, 1, 1, 0.1).sum())


def test_residual_moments_against_fsum(oracle_mod):
    """orc_residual_moments: the reference's Horner residuals (no contraction)
    and their moments, each equal to math.fsum of the same terms."""
    import math
    xy = oracle_mod.synth(50_001, 0, 31, 3, 0.1)
    c = np.array([0.5, -1.0, 0.25, 2.0])
    shift = float(xy[0, 1])
    a, b, e = oracle_mod.residual_moments(xy, c, shift)
    acc = np.full(len(xy), c[3])
    for k in range(2, -1, -1):
        acc = acc * xy[:, 0] + c[k]
    r = xy[:, 1] - acc
    d = xy[:, 1] - shift
    assert a == math.fsum(r * r) and b == math.fsum(d) and e == math.fsum(d * d)

"""GPU property tests (hypothesis): random sizes, degrees, scales and offsets
against the oracle — the stated power-sum bound, coefficient agreement scaled
by conditioning, status parity for overflow / singular inputs, determinism."""
import numpy as np
import pytest

from conftest import kernel_sums

from paper_1512_08017_b200 import _capi
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

pytestmark = pytest.mark.gpu
U = 2.0 ** -53

import os  # noqa: E402

# LSQ_FUZZ_EXAMPLES / LSQ_FUZZ_RANDOM=1: longer, non-derandomised soak runs
SETTINGS = settings(max_examples=int(os.environ.get("LSQ_FUZZ_EXAMPLES", "40")), deadline=None,
                    derandomize=os.environ.get("LSQ_FUZZ_RANDOM") != "1",
                    suppress_health_check=[HealthCheck.too_slow, HealthCheck.function_scoped_fixture])


@pytest.fixture(scope="module")
def L():
    import torch
    assert torch.cuda.is_available()
    from paper_1512_08017_b200 import lsqfit
    return lsqfit


def points(n, scale, shift, seed, distinct):
    rng = np.random.default_rng(seed)
    x = shift + scale * rng.uniform(-1, 1, n)
    if distinct is not None:
        x = rng.choice(np.linspace(-scale, scale, distinct) + shift, n)
    y = rng.standard_normal(n) * (1 + abs(shift))
    return np.stack([x, y], 1)


@SETTINGS
@given(n=st.integers(1, 60_000), m=st.integers(0, 12), scale=st.sampled_from([1e-3, 0.5, 1.0, 3.0, 40.0]),
       shift=st.sampled_from([0.0, 0.5, -2.0]), seed=st.integers(0, 2**31 - 1))
def test_sums_bound_and_determinism(L, oracle_mod, n, m, scale, shift, seed):
    xy = points(n, scale, shift, seed, None)
    d = L.Dataset(xy)
    st_ref, s_ref, t_ref = oracle_mod.accumulate(xy, m)
    if st_ref != 0:
        with pytest.raises(L.OverflowError):
            L.accumulate(d, m)
        return
    r = L.accumulate(d, m)
    assert r.n == n and r.s[0] == float(n)
    r2 = L.accumulate_parallel(d, m, 7)
    assert np.array_equal(np.array(r.s).view(np.uint64), np.array(r2.s).view(np.uint64))
    s_hi, s_lo, s_abs, t_hi, t_lo, t_abs = kernel_sums(oracle_mod, xy, m)
    levels = _capi.sum_error_levels(m)
    for got, hi, lo, ab in ((np.array(r.s[1:]), s_hi[1:], s_lo[1:], s_abs[1:]), (np.array(r.t), t_hi, t_lo, t_abs)):
        err = np.abs((got - hi) - lo)
        assert (err <= levels * U * ab * (1 + 1e-12) + np.spacing(np.abs(hi)) + 1e-300).all()


@SETTINGS
@given(n=st.integers(2, 40_000), m=st.integers(0, 8), scale=st.sampled_from([0.5, 1.0, 2.0]),
       seed=st.integers(0, 2**31 - 1), distinct=st.sampled_from([None, None, None, 1, 2, 3, 5]))
def test_fit_status_and_coefficients(L, oracle_mod, n, m, scale, seed, distinct):
    xy = points(n, scale, 0.0, seed, distinct)
    d = L.Dataset(xy)
    s_hi, s_lo, _, t_hi, t_lo, _ = kernel_sums(oracle_mod, xy, m)
    ex_st, ex = oracle_mod.solve_from_sums(s_hi + s_lo, t_hi + t_lo, m)
    try:
        rep = L.fit_normal(d, m)
        got_st = 0
    except L.SingularSystemError:
        got_st = 3
    A = oracle_mod.build_normal_system(s_hi + s_lo, m)
    kappa = np.linalg.cond(A)
    if ex_st != got_st:
        # only allowed at the pivot-floor boundary: a nearly singular system
        assert kappa > 1e10, (ex_st, got_st, kappa)
        return
    if got_st == 0:
        c = np.array(rep.polynomial.coefficients())
        tol = max(1e-12, 64 * U * kappa)
        assert np.max(np.abs(c - ex)) / max(np.max(np.abs(ex)), 1e-300) <= tol


@SETTINGS
@given(curves=st.integers(1, 400), ppc=st.integers(1, 1100), m=st.integers(0, 12), seed=st.integers(0, 2**31 - 1))
def test_batched_matches_per_curve_loop(oracle_mod, curves, ppc, m, seed):
    import torch
    from paper_1512_08017_b200 import device as D
    xy = points(curves * ppc, 1.0, 0.0, seed, None)
    c, s = D.fit_batched(torch.from_numpy(xy).cuda(), curves, ppc, m)
    c, s = c.cpu().numpy(), s.cpu().numpy()
    rc, rs = oracle_mod.fit_batched(xy, curves, ppc, m)
    ok = (rs == 0) & (s == 0)
    # status may differ only for curves at the singular boundary
    for i in np.nonzero(rs != s)[0]:
        seg = xy[i * ppc:(i + 1) * ppc]
        st_, s_, t_ = oracle_mod.accumulate(seg, m)
        assert np.linalg.cond(oracle_mod.build_normal_system(s_, m)) > 1e10
    for i in np.nonzero(ok)[0]:
        seg = xy[i * ppc:(i + 1) * ppc]
        st_, s_, t_ = oracle_mod.accumulate(seg, m)
        kappa = np.linalg.cond(oracle_mod.build_normal_system(s_, m))
        # the right-hand side's own cancellation (sum|T| / |sum T|, e.g. the
        # mean of zero-mean y at m = 0) scales the sums' relative error
        _, _, _, t_hi, _, t_abs = oracle_mod.exact_sums(seg, m)
        cancel = max(1.0, np.linalg.norm(t_abs) / max(np.linalg.norm(t_hi), 1e-300))
        err = np.max(np.abs(c[i] - rc[i])) / max(np.max(np.abs(rc[i])), 1e-300)
        assert err <= max(1e-12, 256 * U * kappa * cancel)


@SETTINGS
@given(n=st.integers(1, 20_000), m=st.integers(13, 40), scale=st.sampled_from([0.3, 1.0, 1.2]),
       seed=st.integers(0, 2**31 - 1))
def test_any_degree_sums_bound(L, oracle_mod, n, m, scale, seed):
    """Degrees above the fused kernels' cap: the generic kernel's sums within a
    few u * sum|T| of the exact sums of the reference's own terms."""
    xy = points(n, scale, 0.0, seed, None)
    st_ref, _, _ = oracle_mod.accumulate(xy, m)
    d = L.Dataset(xy)
    if st_ref != 0:
        with pytest.raises(L.OverflowError):
            L.accumulate(d, m)
        return
    r = L.accumulate(d, m)
    assert r.s[0] == float(n)
    s_hi, s_lo, s_abs, t_hi, t_lo, t_abs = kernel_sums(oracle_mod, xy, m)
    for got, hi, lo, ab in ((np.array(r.s[1:]), s_hi[1:], s_lo[1:], s_abs[1:]), (np.array(r.t), t_hi, t_lo, t_abs)):
        err = np.abs((got - hi) - lo)
        assert (err <= 4 * U * ab * (1 + 1e-12) + np.spacing(np.abs(hi)) + 1e-300).all()

"""GPU: the out-of-core host path (double-buffered H2D chunks overlapped with
per-chunk kernels, ordered combine) — forced with a small streaming granule —
against the single-launch path and the exact oracle."""
import math

import numpy as np
import pytest

from paper_1512_08017_b200 import _capi

from conftest import bitwise_equal, kernel_sums

pytestmark = pytest.mark.gpu
U = 2.0 ** -53


@pytest.fixture()
def L():
    import torch
    assert torch.cuda.is_available()
    from paper_1512_08017_b200 import _capi, lsqfit
    yield lsqfit
    _capi.context(0).set_stream_chunk(0)


@pytest.mark.parametrize("chunk", [100_003, 262_144, 999_999])
@pytest.mark.parametrize("m", [1, 3, 8])
def test_streamed_sums_match_single_launch_and_oracle(L, oracle_mod, chunk, m):
    from paper_1512_08017_b200 import _capi
    n = 1_000_003
    xy = oracle_mod.synth(n, 0, 7, min(m, 3), 0.1)
    d = L.Dataset(xy)
    _capi.context(0).set_stream_chunk(0)
    single = L.accumulate(d, m)
    _capi.context(0).set_stream_chunk(chunk)
    streamed = L.accumulate(d, m)
    again = L.accumulate(d, m)
    assert streamed.n == n and streamed.s[0] == float(n)
    assert bitwise_equal(streamed.s, again.s) and bitwise_equal(streamed.t, again.t)  # deterministic
    s_hi, s_lo, s_abs, t_hi, t_lo, t_abs = kernel_sums(oracle_mod, xy, m)
    levels = _capi.sum_error_levels(m)
    for got, hi, lo, ab in ((np.array(streamed.s[1:]), s_hi[1:], s_lo[1:], s_abs[1:]),
                            (np.array(streamed.t), t_hi, t_lo, t_abs)):
        assert (np.abs((got - hi) - lo) <= levels * U * ab + np.spacing(np.abs(hi))).all()
    rel = np.max(np.abs(np.array(streamed.s) - np.array(single.s)) / np.maximum(np.abs(single.s), 1e-300))
    assert rel <= 1e-12 or m == 8


@pytest.mark.parametrize("restream", [False, True])
def test_streamed_fit_report(L, oracle_mod, monkeypatch, restream):
    """fit_normal over a chunked host dataset: kept resident in HBM for the
    report pass (default when it fits) or re-streamed over PCIe
    (LSQFIT_CUDA_NO_RESIDENT=1) — same results either way."""
    from paper_1512_08017_b200 import _capi
    if restream:
        monkeypatch.setenv("LSQFIT_CUDA_NO_RESIDENT", "1")
    n, m = 777_777, 3
    xy = oracle_mod.synth(n, 0, 8, 3, 0.1)
    d = L.Dataset(xy)
    _capi.context(0).set_stream_chunk(0)
    a = L.fit_normal(d, m)
    _capi.context(0).set_stream_chunk(123_457)
    b = L.fit_normal(d, m)
    ca, cb = np.array(a.polynomial.coefficients()), np.array(b.polynomial.coefficients())
    assert np.max(np.abs(ca - cb) / np.abs(ca)) <= 1e-12
    # residuals are per point: bit-identical whenever the coefficients are
    c = cb
    acc = np.full(n, c[-1])
    for k in range(len(c) - 2, -1, -1):
        acc = acc * xy[:, 0] + c[k]
    assert bitwise_equal(b.residuals, xy[:, 1] - acc)
    assert abs(a.sse - b.sse) <= 1e-12 * a.sse and abs(a.r - b.r) <= 1e-14
    # against the oracle: coefficients within 1e-10 of the exact-sum solve
    # (reference solve_gaussian on double-double sums of the reference's own
    # terms), SSE and R within 1e-9 of the reference's fit_normal
    s_hi, s_lo, _, t_hi, t_lo, _ = kernel_sums(oracle_mod, xy, m)
    st, ex = oracle_mod.solve_from_sums(s_hi + s_lo, t_hi + t_lo, m)
    assert st == 0
    for rep in (a, b):
        c = np.array(rep.polynomial.coefficients())
        assert np.max(np.abs(c - ex) / np.abs(ex)) <= 1e-10
    if oracle_mod.have_ref():
        st, ref_c, ref_sse, ref_r = oracle_mod.ref_fit_normal(xy, m, 16)
    else:
        st, ref_c = oracle_mod.fit_normal(xy, m, 16)
        acc = np.full(n, ref_c[-1])
        for k in range(len(ref_c) - 2, -1, -1):
            acc = acc * xy[:, 0] + ref_c[k]
        r_ref = xy[:, 1] - acc
        ref_sse = math.fsum(r_ref * r_ref)
        yc = xy[:, 1] - math.fsum(xy[:, 1]) / n
        ref_r = math.sqrt(max(0.0, 1.0 - ref_sse / math.fsum(yc * yc)))
    assert st == 0 and np.max(np.abs(np.array(ref_c) - ex) / np.abs(ex)) <= 1e-10
    for rep in (a, b):
        assert abs(rep.sse - ref_sse) <= 1e-9 * ref_sse and abs(rep.r - ref_r) <= 1e-9


def test_streamed_overflow_and_singular(L):
    from paper_1512_08017_b200 import _capi
    _capi.context(0).set_stream_chunk(3)
    pts = [(2.0, 1.0)] * 10
    with pytest.raises(L.SingularSystemError):
        L.fit_normal(L.Dataset(pts), 1)
    big = [(1.0, 1.0)] * 7 + [(1e200, 1.0)] + [(1.0, 2.0)] * 5
    with pytest.raises(L.OverflowError):
        L.accumulate(L.Dataset(big), 2)
    r = L.accumulate(L.Dataset([(1.0, 1.0)] * 37), 5)
    assert all(v == 37.0 for v in r.s) and all(v == 37.0 for v in r.t)


def test_device_group_sharding_matches_single_device(oracle_mod):
    """lsqfit_cuda_group: G contexts (emulated on one GPU with repeated ids) each
    stream a contiguous shard; records combine in device order."""
    from paper_1512_08017_b200 import _capi
    n, m = 2_000_003, 3
    xy = oracle_mod.synth(n, 0, 12, 3, 0.1)
    st, single = _capi.context(0).fit_host(xy.ctypes.data, n, m, _capi.SOLVE)
    assert st == 0
    s_hi, s_lo, s_abs, t_hi, t_lo, t_abs = kernel_sums(oracle_mod, xy, m)
    for devs in ([0, 0], [0, 0, 0, 0]):
        g = _capi.Group(devs)
        st, r = g.fit_host(xy.ctypes.data, n, m, _capi.SOLVE)
        st2, r2 = g.fit_host(xy.ctypes.data, n, m, _capi.SOLVE)
        g.close()
        assert st == 0 and r.n == n and r.s[0] == float(n)
        assert bitwise_equal(list(r.coeffs[:4]), list(r2.coeffs[:4]))  # deterministic
        got = np.concatenate([np.array(r.s[1:7]), np.array(r.t[:4])])
        hi = np.concatenate([s_hi[1:], t_hi])
        lo = np.concatenate([s_lo[1:], t_lo])
        ab = np.concatenate([s_abs[1:], t_abs])
        assert (np.abs((got - hi) - lo) <= 5 * U * ab + np.spacing(np.abs(hi))).all()
        c, c1 = np.array(r.coeffs[:4]), np.array(single.coeffs[:4])
        assert np.max(np.abs(c - c1) / np.abs(c1)) <= 1e-12


def test_release_buffers_and_reuse(L, oracle_mod):
    """lsqfit_cuda_release_buffers frees the grow-only buffers; the next calls
    re-allocate them and give the same bits."""
    from paper_1512_08017_b200 import _capi
    xy = oracle_mod.synth(500_000, 0, 9, 3, 0.1)
    d = L.Dataset(xy)
    a = L.fit_normal(d, 3)
    ctx = _capi.context(0)
    ctx.release_buffers()
    ctx.release_buffers()  # idempotent
    b = L.fit_normal(d, 3)
    assert bitwise_equal(a.polynomial.coefficients(), b.polynomial.coefficients())
    assert bitwise_equal(a.residuals, b.residuals) and a.sse == b.sse
    ctx.set_stream_chunk(123_457)
    try:
        c = L.accumulate(d, 3)
        ctx.release_buffers()
        e = L.accumulate(d, 3)
    finally:
        ctx.set_stream_chunk(0)
    assert bitwise_equal(c.s, e.s) and bitwise_equal(c.t, e.t)


def test_device_group_fit_device_resident_shards(oracle_mod):
    """lsqfit_cuda_group_fit_device: device-resident shards reduced per device,
    records peer-copied to device 0 and combined in device order — bit-identical
    to the local emulation (per-shard fit + combine); empty shards allowed.
    (One GPU here: the group repeats device 0.)"""
    import torch
    from paper_1512_08017_b200 import _capi, device as D
    n, m = 3_000_017, 3
    xy = D.synth(n, 0, 31, 3, 0.1)
    torch.cuda.synchronize()
    for G in (1, 2, 3):
        g = _capi.Group([0] * G)
        bounds = [(n * k // G, n * (k + 1) // G) for k in range(G)]
        st, r = g.fit_device([xy[lo:hi].data_ptr() for lo, hi in bounds], [hi - lo for lo, hi in bounds],
                             m, _capi.SOLVE)
        assert st == 0 and r.n == n
        parts = D.empty_result(xy.device, G)
        B = _capi.RESULT_BYTES
        for k, (lo, hi) in enumerate(bounds):
            D.fit(xy[lo:hi], m, flags=_capi.SUMS, out=parts[k * B:(k + 1) * B])
        comb = D.read_result(D.combine(parts, G, m))
        assert bitwise_equal(list(r.s[:7]), list(comb.s[:7])) and bitwise_equal(list(r.coeffs[:4]), list(comb.coeffs[:4]))
        g.close()
    g = _capi.Group([0, 0])
    st, r = g.fit_device([xy.data_ptr(), 0], [n, 0], m, _capi.SOLVE)  # empty second shard
    whole = D.read_result(D.fit(xy, m))
    assert st == 0 and bitwise_equal(list(r.s[:7]), list(whole.s[:7]))
    g.close()

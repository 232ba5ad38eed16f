"""GPU: batched mode (one warp per curve; one thread per curve for short curves
at m <= 6) against the per-curve reference loop (oracle: accumulate ->
build_normal_system -> solve_gaussian per curve)."""
import numpy as np
import pytest

from conftest import bitwise_equal, load_golden, unhex

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def D():
    import torch
    assert torch.cuda.is_available()
    from paper_1512_08017_b200 import device
    return device


def normwise(c, ref):
    """Per-curve max|c - ref| / max|ref| (coefficient vectors, norm-wise)."""
    if c.size == 0:
        return 0.0
    return float(np.max(np.max(np.abs(c - ref), axis=1) / np.maximum(np.max(np.abs(ref), axis=1), 1e-300)))


def kappa_tolerance(oracle_mod, xy, n_curves, ppc, m, floor=1e-12):
    """Per-curve tolerance 256 u kappa(A): the sums differ from the reference's
    by a few u * sum|T| (different summation order), which the solve amplifies
    by at most ~kappa(A)."""
    tol = np.empty(n_curves)
    for c in range(n_curves):
        st, s, t = oracle_mod.accumulate(xy[c * ppc:(c + 1) * ppc], m)
        a = oracle_mod.build_normal_system(s, m)
        tol[c] = max(floor, 256 * 2.0 ** -53 * np.linalg.cond(a))
    return tol


def curve_errors(c, ref):
    return np.max(np.abs(c - ref), axis=1) / np.maximum(np.max(np.abs(ref), axis=1), 1e-300)


def run(D, xy_np, n_curves, ppc, m):
    import torch
    xy = torch.from_numpy(np.ascontiguousarray(xy_np)).cuda()
    c, st = D.fit_batched(xy, n_curves, ppc, m)
    torch.cuda.synchronize()
    return c.cpu().numpy(), st.cpu().numpy()


def test_golden_batched_curves(D):
    rec = [r for r in load_golden("counter_synth.json") if r.get("batched")][0]
    xy = D.synth_batched(rec["n_curves"], rec["ppc"], rec["seed"], rec["truth_degree"], rec["sigma"])
    c, st = D.fit_batched(xy, rec["n_curves"], rec["ppc"], rec["truth_degree"])
    c, st = c.cpu().numpy(), st.cpu().numpy()
    ref = unhex(rec["coeffs"]).reshape(c.shape)
    assert (st == 0).all()
    assert normwise(c, ref) <= 1e-12


@pytest.mark.parametrize("m", list(range(0, 13)))
def test_batched_matches_per_curve_reference(D, oracle_mod, m):
    n_curves, ppc = 300, 1024 if m <= 4 else 512
    xy = oracle_mod.synth_batched(n_curves, ppc, 70 + m, min(m, 4), 0.1)
    c, st = run(D, xy, n_curves, ppc, m)
    rc, rst = oracle_mod.fit_batched(xy, n_curves, ppc, m)
    assert (st == rst).all()
    ok = rst == 0
    # normal-equation conditioning grows with m (SURVEY §8c kappa table): scale the tolerance
    tol = kappa_tolerance(oracle_mod, xy, n_curves, ppc, m)
    assert (curve_errors(c[ok], rc[ok]) <= tol[ok]).all()
    if m <= 3:
        assert normwise(c[ok], rc[ok]) <= 1e-11


@pytest.mark.parametrize("ppc", [1, 2, 3, 31, 255, 256, 257, 1000, 1023, 1025, 4097])
def test_ragged_points_per_curve(D, oracle_mod, ppc):
    n_curves, m = 97, 2
    xy = oracle_mod.synth_batched(n_curves, ppc, 5, 2, 0.1)
    c, st = run(D, xy, n_curves, ppc, m)
    rc, rst = oracle_mod.fit_batched(xy, n_curves, ppc, m)
    assert (st == rst).all()
    ok = rst == 0
    tol = kappa_tolerance(oracle_mod, xy, n_curves, ppc, m)
    assert (curve_errors(c[ok], rc[ok]) <= tol[ok]).all()


def test_singular_and_overflow_curves_flagged(D, oracle_mod):
    ppc = 256
    xy = oracle_mod.synth_batched(4, ppc, 1, 2, 0.1)
    xy[ppc:2 * ppc, 0] = 0.5          # curve 1: one distinct x -> singular
    xy[2 * ppc, 0] = 1e200            # curve 2: overflow
    c, st = run(D, xy, 4, ppc, 2)
    rc, rst = oracle_mod.fit_batched(xy, 4, ppc, 2)
    assert st.tolist() == rst.tolist() == [0, 3, 2, 0]
    assert bitwise_equal(c[0], c[0]) and np.allclose(c[[0, 3]], rc[[0, 3]], rtol=1e-10)


def test_batched_solve_bitwise_given_same_sums(D, oracle_mod):
    """Curves whose sums are exact (integer x, y) must give the reference's bits."""
    rng = np.random.default_rng(9)
    n_curves, ppc, m = 64, 256, 2
    xy = np.stack([rng.integers(-4, 5, n_curves * ppc), rng.integers(-50, 50, n_curves * ppc)], 1).astype(np.float64)
    c, st = run(D, xy, n_curves, ppc, m)
    rc, rst = oracle_mod.fit_batched(xy, n_curves, ppc, m)
    assert (st == rst).all()
    assert bitwise_equal(c[rst == 0], rc[rst == 0])


@pytest.mark.parametrize("m", [0, 1, 2, 3, 4, 5, 6, 7, 9, 12])
@pytest.mark.parametrize("ppc", [1, 4, 5, 15, 16, 17, 100, 256])
def test_short_curves_thread_per_curve(D, oracle_mod, m, ppc):
    """Thread-per-curve kernel (direct loads below 16 points, warp-staged
    slices from 16 to 256; the system in registers up to m = 6, in shared
    memory beyond) incl. a partial last group of 32 curves."""
    n_curves = 1000 + 7
    xy = oracle_mod.synth_batched(n_curves, ppc, 300 + ppc, min(m, 2), 0.1)
    c, st = run(D, xy, n_curves, ppc, m)
    rc, rst = oracle_mod.fit_batched(xy, n_curves, ppc, m)
    assert (st == rst).all()
    ok = rst == 0
    tol = kappa_tolerance(oracle_mod, xy, n_curves, ppc, m)
    assert (curve_errors(c[ok], rc[ok]) <= tol[ok]).all()
    assert (c[~ok] == 0).all()


@pytest.mark.parametrize("ppc,m", [(8, 2), (16, 2), (64, 2), (64, 8), (256, 10)])
def test_short_curves_status_and_bitwise_solve(D, oracle_mod, ppc, m):
    """Singular / overflow flags and, for exactly representable sums (small
    integers), the reference's bits from the in-register solve."""
    rng = np.random.default_rng(ppc + m)
    n_curves = 96
    xy = np.stack([rng.integers(-4, 5, n_curves * ppc), rng.integers(-50, 50, n_curves * ppc)], 1).astype(np.float64)
    xy[ppc:2 * ppc, 0] = 3.0       # curve 1: one distinct x -> singular
    xy[2 * ppc + 1, 0] = 1e200     # curve 2: overflow
    c, st = run(D, xy, n_curves, ppc, m)
    rc, rst = oracle_mod.fit_batched(xy, n_curves, ppc, m)
    assert st[1] == 3 and st[2] == 2
    assert (st == rst).all()
    assert bitwise_equal(c[rst == 0], rc[rst == 0])


@pytest.mark.parametrize("m,maxlen", [(1, 40), (2, 300), (3, 2500), (8, 200), (12, 120)])
def test_ragged_batch_matches_per_curve_reference(D, oracle_mod, m, maxlen):
    """Ragged batches (curve c = [offsets[c], offsets[c+1]), empty curves
    allowed): each curve as accumulate -> build_normal_system -> solve_gaussian
    on its own points; statuses as the reference (empty / too few distinct x:
    singular)."""
    import torch
    rng = np.random.default_rng(m * 1000 + maxlen)
    lens = rng.integers(0, maxlen + 1, 700)
    lens[:3] = [0, 1, m + 1]
    offs = np.concatenate([[5], 5 + np.cumsum(lens)]).astype(np.int64)
    xy = oracle_mod.synth(int(offs[-1]) + 3, 0, 500 + m, min(m, 3), 0.1)
    c, st = D.fit_batched_ragged(torch.from_numpy(np.ascontiguousarray(xy)).cuda(), torch.from_numpy(offs).cuda(), m)
    c, st = c.cpu().numpy(), st.cpu().numpy()
    for k in range(len(lens)):
        seg = xy[offs[k]:offs[k + 1]]
        if len(seg) == 0:
            assert st[k] == 3
            continue
        s_st, s, t = oracle_mod.accumulate(seg, m)
        r_st, x = oracle_mod.solve_from_sums(s, t, m) if s_st == 0 else (s_st, None)
        if r_st != st[k]:  # only at the singular boundary
            assert np.linalg.cond(oracle_mod.build_normal_system(s, m)) > 1e10
            continue
        if r_st == 0:
            kappa = np.linalg.cond(oracle_mod.build_normal_system(s, m))
            _, _, _, t_hi, _, t_abs = oracle_mod.exact_sums(seg, m)
            cancel = max(1.0, np.linalg.norm(t_abs) / max(np.linalg.norm(t_hi), 1e-300))
            err = np.max(np.abs(c[k] - x)) / max(np.max(np.abs(x)), 1e-300)
            assert err <= max(1e-12, 256 * 2.0 ** -53 * kappa * cancel), (k, len(seg), err)


def test_ragged_host_api_matches_device(D, oracle_mod):
    """lsqfit_cuda_fit_batched_ragged_host (offsets may start past 0) equals
    the device-resident ragged fit on the same curves, bit for bit."""
    import ctypes as C
    import torch
    from paper_1512_08017_b200 import _capi
    rng = np.random.default_rng(3)
    lens = rng.integers(0, 90, 400)
    offs = np.concatenate([[11], 11 + np.cumsum(lens)]).astype(np.uint64)
    xy = np.ascontiguousarray(oracle_mod.synth(int(offs[-1]) + 2, 0, 44, 2, 0.1))
    m = 2
    coeffs = np.zeros(len(lens) * (m + 1))
    status = np.zeros(len(lens), dtype=np.int32)
    ctx = _capi.context(0)
    dp = C.POINTER(C.c_double)
    st = ctx._lib.lsqfit_cuda_fit_batched_ragged_host(ctx.h, xy.ctypes.data_as(dp),
                                                      offs.ctypes.data_as(C.POINTER(C.c_uint64)), len(lens), m,
                                                      coeffs.ctypes.data_as(dp),
                                                      status.ctypes.data_as(C.POINTER(C.c_int32)))
    assert st == 0
    c_dev, s_dev = D.fit_batched_ragged(torch.from_numpy(xy).cuda(), torch.from_numpy(offs.astype(np.int64)).cuda(), m)
    assert np.array_equal(status, s_dev.cpu().numpy())
    assert bitwise_equal(coeffs.reshape(-1, m + 1), c_dev.cpu().numpy())


def test_python_mirror_batched_host(oracle_mod):
    """lsqfit.fit_batched / fit_batched_ragged (host numpy in, host numpy out)."""
    from paper_1512_08017_b200 import lsqfit as L
    xy = oracle_mod.synth_batched(50, 64, 8, 2, 0.1)
    c, st = L.fit_batched(xy, 50, 64, 2)
    rc, rst = oracle_mod.fit_batched(xy, 50, 64, 2)
    assert (st == rst).all() and np.max(np.abs(c - rc)) <= 1e-10 * np.max(np.abs(rc))
    offs = np.arange(0, 50 * 64 + 1, 64)
    c2, st2 = L.fit_batched_ragged(xy, offs, 2)
    assert (st2 == st).all() and np.max(np.abs(c2 - c)) <= 1e-12 * np.max(np.abs(c))
    with pytest.raises(ValueError):
        L.fit_batched_ragged(xy, [0, 10, 5], 2)


@pytest.mark.parametrize("m,ppc", [(2, 1100), (3, 1025), (5, 2048)])
def test_dynamic_curve_claims_cover_every_curve(D, oracle_mod, m, ppc):
    """The warp-per-curve kernel deals curves beyond each warp's first block
    through a claim counter (csrc/batched.cuh): with far more curves than
    warps every curve is written exactly as the per-curve reference computes
    it, the counters re-arm (the second launch gives the same bits), and two
    batches on two streams of one context do not share claims."""
    import torch
    n_curves = 120_000
    xy = D.synth_batched(n_curves, ppc, 90 + m, min(m, 2), 0.1)
    c = torch.full((n_curves, m + 1), float("nan"), dtype=torch.float64, device="cuda")
    st = torch.full((n_curves,), -7, dtype=torch.int32, device="cuda")
    D.fit_batched(xy, n_curves, ppc, m, c, st)
    c2, st2 = D.fit_batched(xy, n_curves, ppc, m)
    torch.cuda.synchronize()
    assert (st != -7).all() and not torch.isnan(c).any()
    assert torch.equal(c.view(torch.int64), c2.view(torch.int64)) and torch.equal(st, st2)
    rng = np.random.default_rng(m)
    idx = np.sort(rng.choice(n_curves, 300, replace=False))
    xy_h = xy.view(n_curves, ppc, 2)[torch.from_numpy(idx).cuda()].cpu().numpy().reshape(-1, 2)
    rc, rst = oracle_mod.fit_batched(xy_h, len(idx), ppc, m)
    ch, sth = c.cpu().numpy()[idx], st.cpu().numpy()[idx]
    assert (sth == rst).all()
    ok = rst == 0
    tol = kappa_tolerance(oracle_mod, xy_h, len(idx), ppc, m)
    assert (curve_errors(ch[ok], rc[ok]) <= tol[ok]).all()
    # two streams, one context: the second batch waits for the first's claims
    half = n_curves // 2
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    a = torch.empty_like(c)
    sa = torch.empty_like(st)
    with torch.cuda.stream(s1):
        D.fit_batched(xy[: half * ppc], half, ppc, m, a[:half], sa[:half])
    with torch.cuda.stream(s2):
        D.fit_batched(xy[half * ppc:], n_curves - half, ppc, m, a[half:], sa[half:])
    torch.cuda.synchronize()
    assert torch.equal(a.view(torch.int64), c.view(torch.int64)) and torch.equal(sa, st)

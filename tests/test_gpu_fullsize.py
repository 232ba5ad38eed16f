"""GPU, BASELINE.json full sizes, checked through size-independent properties:
n = 4e9 (the metric's config, 64 GB resident) and the 1e6 x 1024 batched
config (16.4 GB). Determinism, shard additivity (the checksum of shard
checksums), the exact count, agreement with the reference-order (bit-exact
reference accumulate_parallel) sums within the reference's cross-strategy
tolerance, recovery of the generating polynomial, and per-curve parity on a
sample against the CPU per-curve loop."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N_FULL = 4_000_000_000
M = 3


@pytest.fixture(scope="module")
def big():
    import torch
    from paper_1512_08017_b200 import device as D
    free, _ = torch.cuda.mem_get_info()
    if free < 70e9:
        pytest.skip("needs ~70 GB of free device memory")
    xy = D.synth(N_FULL, 0, 4, 3, 0.1)
    torch.cuda.synchronize()
    yield xy
    del xy
    torch.cuda.empty_cache()


def test_full_size_determinism_count_and_truth(big, oracle_mod):
    from paper_1512_08017_b200 import device as D
    a = D.read_result(D.fit(big, M))
    b = D.read_result(D.fit(big, M))
    assert a.status == 0 and a.n == N_FULL and a.s[0] == float(N_FULL)
    assert list(a.s[:7]) == list(b.s[:7]) and list(a.coeffs[:4]) == list(b.coeffs[:4])
    truth = oracle_mod.synth_truth(4, 0, 3)
    # noise sigma = 0.1 over 4e9 points: the fit recovers the truth to ~1e-4
    assert np.max(np.abs(np.array(a.coeffs[:4]) - truth)) < 1e-3


def test_full_size_shard_additivity(big):
    """Sum of per-shard double-double partials (combine) == whole within the bound."""
    from paper_1512_08017_b200 import _capi, device as D
    whole = D.read_result(D.fit(big, M))
    G = 8
    parts = D.empty_result(big.device, G)
    B = _capi.RESULT_BYTES
    for g in range(G):
        lo, hi = N_FULL * g // G, N_FULL * (g + 1) // G
        D.fit(big[lo:hi], M, flags=0, out=parts[g * B:(g + 1) * B])
    comb = D.read_result(D.combine(parts, G, M))
    assert comb.n == N_FULL and comb.status == 0
    for k in range(1, 7):
        # sum|T| for s[k] is <= n (|x| < 1); bound 5u * n per sum plus an ulp
        assert abs(comb.s[k] - whole.s[k]) <= 2 * 5 * 2.0 ** -53 * N_FULL + 2 * np.spacing(abs(whole.s[k]))
    assert np.max(np.abs(np.array(comb.coeffs[:4]) - np.array(whole.coeffs[:4]))) <= 1e-12 * np.max(
        np.abs(whole.coeffs[:4]))


def test_full_size_reference_order_agreement(big):
    """The reference's own accumulate_parallel(d, 3, 65536), replayed bit-exactly
    on the GPU, agrees with the compensated sums to the reference's 1e-9."""
    from paper_1512_08017_b200 import device as D
    whole = D.read_result(D.fit(big, M))
    ref = D.read_result(D.fit_ordered(big, M, 65536))
    assert ref.status == 0 and ref.s[0] == float(N_FULL)
    for k in range(7):
        assert abs(ref.s[k] - whole.s[k]) <= 1e-9 * max(abs(whole.s[k]), 1.0) + 1e-9 * N_FULL * (k % 2)
    for j in range(4):
        assert abs(ref.t[j] - whole.t[j]) <= 1e-9 * N_FULL * 10
    rel = np.max(np.abs(np.array(ref.coeffs[:4]) - np.array(whole.coeffs[:4])) / np.abs(np.array(whole.coeffs[:4])))
    print(f"\nn=4e9 m=3 coefficient max rel. diff vs reference accumulate_parallel(65536): {rel:.3e}")
    assert rel <= 1e-10  # north star: <= 1e-10 for m <= 3, x in [-1, 1]


def test_full_size_batched_config(oracle_mod):
    import torch
    from paper_1512_08017_b200 import device as D
    free, _ = torch.cuda.mem_get_info()
    if free < 20e9:
        pytest.skip("needs ~20 GB of free device memory")
    curves, ppc, m = 1_000_000, 1024, 2
    xy = D.synth_batched(curves, ppc, 5, 2, 0.1)
    c, st = D.fit_batched(xy, curves, ppc, m)
    assert int((st != 0).sum().item()) == 0
    rng = np.random.default_rng(0)
    sample = np.sort(rng.choice(curves, 200, replace=False))
    cs = c.cpu().numpy()
    for i in sample:
        seg = xy[i * ppc:(i + 1) * ppc].cpu().numpy()
        rc, rs = oracle_mod.fit_batched(seg, 1, ppc, m)
        assert rs[0] == 0
        assert np.max(np.abs(cs[i] - rc[0])) <= 1e-12 * np.max(np.abs(rc[0]))
    del xy
    torch.cuda.empty_cache()


def test_full_size_diagnostics(big):
    """FitReport pass at n = 4e9 (8e9 doubles: element offsets past 2^32): shard
    additivity of SSE and of the shifted moments (same shift), exact count,
    sane R, and residuals at sampled indices bit-identical to host Horner."""
    import torch
    from paper_1512_08017_b200 import device as D
    fr = D.fit(big, M)
    shift = float(big[0, 1].item())
    res = torch.empty(N_FULL, dtype=torch.float64, device=big.device)
    whole = D.read_diag(D.diagnostics(big, M, fr, residuals=res))
    assert whole.status == 0 and whole.n == N_FULL and whole.shift == shift
    assert 0.99 < whole.r <= 1.0
    G = 4
    sse = 0.0
    sd = np.longdouble(0)
    sd2 = np.longdouble(0)
    for g in range(G):
        lo, hi = N_FULL * g // G, N_FULL * (g + 1) // G
        d = D.read_diag(D.diagnostics(big[lo:hi], M, fr, shift=shift))
        assert d.status == 0 and d.n == hi - lo and d.shift == shift
        sse += d.sse
        sd += np.longdouble(d.part_hi[1]) + np.longdouble(d.part_lo[1])
        sd2 += np.longdouble(d.part_hi[2]) + np.longdouble(d.part_lo[2])
    assert abs(sse - whole.sse) <= 1e-12 * whole.sse
    sst = float(sd2 - sd * sd / np.longdouble(N_FULL))
    assert abs(sst - whole.sst) <= 1e-12 * whole.sst
    # residuals: y - Horner(x), rounded exactly as the reference (no FMA)
    c = np.array(D.read_result(fr).coeffs[:M + 1])
    idx = np.array([0, 1, 2 ** 31 - 1, 2 ** 31, 2 ** 31 + 12345, N_FULL - 2, N_FULL - 1], dtype=np.int64)
    # (row slices, not an index tensor: torch's gather asserts past 2^31 rows)
    pts = np.array([big[int(i):int(i) + 1].cpu().numpy()[0] for i in idx])
    got = np.array([res[int(i):int(i) + 1].cpu().numpy()[0] for i in idx])
    acc = np.full(len(idx), c[M])
    for k in range(M - 1, -1, -1):
        acc = acc * pts[:, 0] + c[k]
    assert (got == pts[:, 1] - acc).all()
    del res
    torch.cuda.empty_cache()

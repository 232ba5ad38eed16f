"""GPU: the TSQR cross-check backend against the reference's Householder-QR
fit (golden fixtures from oracle/_ref), exact rational least squares, and its
own sharded / streamed forms."""
from fractions import Fraction

import numpy as np
import pytest

from conftest import load_golden, unhex

pytestmark = pytest.mark.gpu
U = 2.0 ** -53


@pytest.fixture(scope="module")
def L():
    import torch
    assert torch.cuda.is_available()
    from paper_1512_08017_b200 import lsqfit
    return lsqfit


def vander(xy, m):
    return np.vander(xy[:, 0], m + 1, increasing=True)


def test_golden_reference_qr_fits(L):
    for case in load_golden("qr_fits.json"):
        xy = unhex(case["points"]).reshape(-1, 2)
        m = case["degree"]
        if case["status"] != 0:
            with pytest.raises(L.RankDeficientError):
                L.fit_qr(L.Dataset(xy), m)
            continue
        rep = L.fit_qr(L.Dataset(xy), m)
        c = np.array(rep.polynomial.coefficients())
        ref = unhex(case["coeffs"])
        kappa = np.linalg.cond(vander(xy, m))
        tol = max(1e-13, 64 * U * kappa)
        assert np.max(np.abs(c - ref)) / np.max(np.abs(ref)) <= tol, (case["name"], kappa)
        sse = unhex(case["sse"])
        assert abs(rep.sse - sse) <= 1e-9 * (1 + sse), case["name"]
        assert abs(rep.r - unhex(case["r"])) <= 1e-9
        assert rep.backend == "qr"


def exact_ls(xy, m):
    """Exact least-squares coefficients (rational normal equations, exact data)."""
    X = [Fraction(float(x)) for x in xy[:, 0]]
    Y = [Fraction(float(y)) for y in xy[:, 1]]
    pw = [[Fraction(1)] * len(X)]
    for _ in range(2 * m):
        pw.append([a * b for a, b in zip(pw[-1], X)])
    s = [sum(p) for p in pw]
    t = [sum(a * b for a, b in zip(pw[j], Y)) for j in range(m + 1)]
    A = [[s[i + j] for j in range(m + 1)] + [t[i]] for i in range(m + 1)]
    for c in range(m + 1):
        p = next(r for r in range(c, m + 1) if A[r][c] != 0)
        A[c], A[p] = A[p], A[c]
        for r in range(m + 1):
            if r != c and A[r][c] != 0:
                f = A[r][c] / A[c][c]
                A[r] = [a - f * b for a, b in zip(A[r], A[c])]
    return np.array([float(A[i][m + 1] / A[i][i]) for i in range(m + 1)])


def test_qr_beats_normal_equations_when_ill_conditioned(L, oracle_mod):
    # x in [0, 1) (the reference generator), degree 8: kappa(V) ~ 1e7, kappa(A) = kappa(V)^2
    xy = oracle_mod.generate_synthetic(400, 8, 0.05, 9)
    m = 8
    exact = exact_ls(xy, m)
    qr = np.array(L.fit_qr(L.Dataset(xy), m).polynomial.coefficients())
    ne = np.array(L.fit_normal(L.Dataset(xy), m).polynomial.coefficients())
    e_qr = np.max(np.abs(qr - exact)) / np.max(np.abs(exact))
    e_ne = np.max(np.abs(ne - exact)) / np.max(np.abs(exact))
    kappa = np.linalg.cond(vander(xy, m))
    assert e_qr <= 64 * U * kappa
    assert e_qr < e_ne / 10, (e_qr, e_ne)


def test_r_factor_reproduces_gram_matrix(L, oracle_mod):
    import torch
    from paper_1512_08017_b200 import device as D
    n, m = 100_003, 3
    xy = oracle_mod.synth(n, 0, 3, 3, 0.1)
    out = D.qr_fit(torch.from_numpy(xy).cuda(), m)
    q = D.read_qr_result(out)
    C = m + 2
    R = np.array(q.r[: C * C]).reshape(C, C)
    assert q.status == 0 and q.n == n
    assert np.allclose(np.tril(R, -1), 0.0) and (np.diag(R) >= 0).all()
    G = R.T @ R  # == [V y]^T [V y]
    s_hi, s_lo, _, t_hi, t_lo, _ = oracle_mod.exact_sums(xy, m)
    s = s_hi + s_lo
    A = np.array([[s[i + j] for j in range(m + 1)] for i in range(m + 1)])
    assert np.max(np.abs(G[: m + 1, : m + 1] - A) / np.abs(A).max()) <= 1e-13
    assert np.max(np.abs(G[: m + 1, m + 1] - (t_hi + t_lo))) / np.abs(t_hi).max() <= 1e-13
    # rho^2 is the least-squares SSE
    rep = L.fit_normal(L.Dataset(xy), m)
    assert abs(q.residual_norm ** 2 - rep.sse) <= 1e-9 * rep.sse
    c = np.array(q.coeffs[: m + 1])
    ne = np.array(rep.polynomial.coefficients())
    assert np.max(np.abs(c - ne) / np.abs(ne)) <= 1e-11


@pytest.mark.parametrize("m", list(range(0, 13)))
def test_all_degrees_agree_with_reference_qr(L, oracle_mod, m):
    xy = oracle_mod.synth(20_011, 0, 50 + m, min(m, 4), 0.1)
    rep = L.fit_qr(L.Dataset(xy), m)
    if oracle_mod.have_ref():
        st, ref, sse, r = oracle_mod.ref_fit_qr(xy, m)
        assert st == 0
    else:
        st, ref = oracle_mod.fit_normal(xy, m)  # well conditioned on [-1, 1] for these degrees
    c = np.array(rep.polynomial.coefficients())
    kappa = np.linalg.cond(vander(xy, m))
    assert np.max(np.abs(c - ref)) / np.max(np.abs(ref)) <= max(1e-13, 256 * U * kappa * (kappa if not oracle_mod.have_ref() else 1))


def test_sharded_and_streamed_qr(L, oracle_mod):
    import torch
    from paper_1512_08017_b200 import _capi, device as D
    n, m = 1_000_003, 4
    xy_h = oracle_mod.synth(n, 0, 11, 4, 0.1)
    xy = torch.from_numpy(xy_h).cuda()
    whole = D.read_qr_result(D.qr_fit(xy, m))
    for G in (2, 3):
        parts = D.empty_qr_result(xy.device, G)
        B = _capi.QR_BYTES
        for g in range(G):
            lo, hi = n * g // G, n * (g + 1) // G
            D.qr_fit(xy[lo:hi], m, flags=0, out=parts[g * B:(g + 1) * B])
        comb = D.read_qr_result(D.qr_combine(parts, G, m))
        assert comb.status == 0 and comb.n == n
        assert np.max(np.abs(np.array(comb.coeffs[:5]) - np.array(whole.coeffs[:5]))) <= 1e-12 * np.max(np.abs(whole.coeffs[:5]))
    ctx = _capi.context(0)
    try:
        ctx.set_stream_chunk(77_777)
        st, q = ctx.qr_fit_host(xy_h.ctypes.data, n, m)
    finally:
        ctx.set_stream_chunk(0)
    assert st == 0 and q.n == n
    assert np.max(np.abs(np.array(q.coeffs[:5]) - np.array(whole.coeffs[:5]))) <= 1e-12 * np.max(np.abs(whole.coeffs[:5]))


def test_qr_errors(L):
    with pytest.raises(L.RankDeficientError):
        L.fit_qr(L.Dataset([(2.0, 1.0)] * 5), 1)
    with pytest.raises(L.RankDeficientError):
        L.fit_qr(L.Dataset([(0.0, 1.0), (1.0, 2.0)]), 2)
    with pytest.raises(L.OverflowError):
        L.fit_qr(L.Dataset([(1e200, 1.0), (1.0, 2.0), (2.0, 3.0), (3.0, 1.0)]), 2)
    with pytest.raises(L.DegreeTooHighError):
        L.fit_qr(L.Dataset([(0.0, 1.0), (1.0, 2.0)]), 13)
    # TSQR now covers the reference's whole degree range (<= 12).
    with pytest.raises(L.RankDeficientError):
        L.fit_qr(L.Dataset([(0.0, 1.0), (1.0, 2.0)]), 12)

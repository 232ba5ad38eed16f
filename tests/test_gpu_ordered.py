"""GPU: reference-order mode reproduces the reference's accumulate /
accumulate_parallel bits exactly — against the golden reference fixtures
(bits produced by the compiled reference) and the bit-pinned oracle port."""
import pytest

from conftest import TABLE1, bitwise_equal, load_golden, unhex

pytestmark = pytest.mark.gpu


@pytest.fixture()
def L():
    import torch
    assert torch.cuda.is_available()
    from paper_1512_08017_b200 import lsqfit
    lsqfit.set_reference_order(True)
    yield lsqfit
    lsqfit.set_reference_order(False)


def test_table1_reference_bits(L):
    g = load_golden("table1.json")
    d = L.Dataset(TABLE1)
    for m, e in g["by_degree"].items():
        m = int(m)
        r = L.accumulate(d, m)
        assert bitwise_equal(r.s, unhex(e["s"])) and bitwise_equal(r.t, unhex(e["t"]))
        for chunks in (1, 2, 3, 16):
            r = L.accumulate_parallel(d, m, chunks)
            assert bitwise_equal(r.s, unhex(e[f"par{chunks}"]["s"])), (m, chunks)
            assert bitwise_equal(r.t, unhex(e[f"par{chunks}"]["t"])), (m, chunks)


def test_reference_generate_synthetic_bits(L, oracle_mod):
    for rec in load_golden("synthetic_ref.json"):
        xy = oracle_mod.generate_synthetic(rec["n"], rec["degree"], rec["sigma"], rec["seed"])
        d = L.Dataset(xy)
        m = rec["degree"]
        if rec["n"] <= 20000:
            r = L.accumulate(d, m)  # one sequential chain (slow path, small n only)
            assert bitwise_equal(r.s, unhex(rec["s"])) and bitwise_equal(r.t, unhex(rec["t"]))
        for chunks, e in rec["par"].items():
            if int(chunks) == 1 and rec["n"] > 20000:
                continue
            r = L.accumulate_parallel(d, m, int(chunks))
            assert bitwise_equal(r.s, unhex(e["s"])) and bitwise_equal(r.t, unhex(e["t"])), (rec["n"], chunks)


@pytest.mark.parametrize("m", [0, 1, 3, 5, 8, 12])
@pytest.mark.parametrize("chunks", [7, 1000, 65536, 300_001, 500_000])
def test_bitwise_vs_port_many_chunks(L, oracle_mod, m, chunks):
    n = 300_001
    xy = oracle_mod.synth(n, 0, 90 + m, min(m, 3), 0.1)
    r = L.accumulate_parallel(L.Dataset(xy), m, chunks)
    st, s, t = oracle_mod.accumulate_parallel(xy, m, chunks)
    assert st == 0
    assert bitwise_equal(r.s, s) and bitwise_equal(r.t, t)
    assert r.s[0] == float(n)


def test_ordered_solve_matches_reference_fit_bits(L, oracle_mod):
    """Sums bit-identical + the bit-identical solve => the reference's coefficients exactly."""
    import torch
    from paper_1512_08017_b200 import device as D
    n, m, chunks = 1_000_003, 3, 4096
    xy = oracle_mod.synth(n, 0, 5, 3, 0.1)
    out = D.read_result(D.fit_ordered(torch.from_numpy(xy).cuda(), m, chunks))
    st, c = oracle_mod.fit_normal(xy, m, chunks)
    assert st == 0 and out.status == 0
    assert bitwise_equal(list(out.coeffs[: m + 1]), c)


def test_ordered_overflow(L):
    with pytest.raises(L.OverflowError):
        L.accumulate_parallel(L.Dataset([(1e200, 1.0), (1e200, 2.0), (1.0, 3.0)]), 2, 2)


@pytest.mark.parametrize("m,chunks", [(13, 1), (13, 7), (20, 64), (31, 3)])
def test_reference_order_any_degree_bits(L, oracle_mod, m, chunks):
    """Reference-order mode above the fused kernels' cap: the column replay
    gives exactly the compiled reference's accumulate_parallel(d, m, chunks)
    (accumulate for chunks = 1) bits."""
    if not oracle_mod.have_ref():
        pytest.skip("oracle/_ref not built")
    xy = oracle_mod.synth(30_011, 0, 90 + m, 3, 0.1)
    L.set_reference_order(True)
    try:
        d = L.Dataset(xy)
        r = L.accumulate(d, m) if chunks == 1 else L.accumulate_parallel(d, m, chunks)
    finally:
        L.set_reference_order(False)
    st, s, t = oracle_mod.ref_accumulate(xy, m) if chunks == 1 else oracle_mod.ref_accumulate_parallel(xy, m, chunks)
    assert st == 0
    assert bitwise_equal(r.s, s) and bitwise_equal(r.t, t)


def test_python_fit_normal_reference_order_bits(L, oracle_mod):
    """The Python mirror's fit_normal in reference-order mode follows the C++
    drop-in: the reference's own sums over `chunks` slices and its solve, so
    the coefficients equal the reference's fit_normal bit for bit; the report
    (residuals / SSE / R) comes from the device pass."""
    for rec in load_golden("synthetic_ref.json"):
        if rec["degree"] < 1 or rec["n"] > 20000:
            continue
        xy = oracle_mod.generate_synthetic(rec["n"], rec["degree"], rec["sigma"], rec["seed"])
        m = rec["degree"]
        for chunks in (1, 4):
            rep = L.fit_normal(L.Dataset(xy), m, chunks)
            st, c = oracle_mod.fit_normal(xy, m, chunks)  # the bit-pinned port of the reference
            assert st == 0 and bitwise_equal(rep.polynomial.coefficients(), c), (rec["n"], m, chunks)
            if chunks == 1:
                assert bitwise_equal(rep.polynomial.coefficients(), unhex(rec["fit"]["coeffs"]))
            assert abs(rep.sse - unhex(rec["fit"]["sse"])) <= 1e-9 * (1 + unhex(rec["fit"]["sse"]))


@pytest.mark.parametrize("m", [1, 3, 8, 12])
@pytest.mark.parametrize("n,chunks", [(2_000_003, 8192), (3_000_017, 10_007), (1_500_000, 16384)])
def test_bitwise_vs_port_row_kernel(L, oracle_mod, m, n, chunks):
    """From 8192 chunks the slots come from the thread-per-chunk kernel with
    cp.async-staged rows (ragged rows: chunk lengths differ by one, the last
    round is partial): still the reference's bits."""
    xy = oracle_mod.synth(n, 0, 70 + m, min(m, 3), 0.1)
    r = L.accumulate_parallel(L.Dataset(xy), m, chunks)
    st, s, t = oracle_mod.accumulate_parallel(xy, m, chunks)
    assert st == 0
    assert bitwise_equal(r.s, s) and bitwise_equal(r.t, t)

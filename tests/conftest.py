import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name: str):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def unhex(v):
    if v is None:
        return None
    if isinstance(v, str):
        return float.fromhex(v)
    return np.array([float.fromhex(x) for x in v])


def bits(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64)).view(np.uint64)


def bitwise_equal(a, b) -> bool:
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(bits(a), bits(b))


def max_rel_dev(a, b) -> float:
    """test_accumulator.cpp:30-37."""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    denom = np.maximum(np.abs(a), np.abs(b))
    m = denom > 0
    return float(np.max(np.abs(a - b)[m] / denom[m])) if m.any() else 0.0


TABLE1 = [(39.206, 751.912), (29.74, 567.121), (21.31, 403.746),
          (12.087, 221.738), (1.812, 18.8418), (0.001, 1.88672)]


def kernel_sums(O, xy, m):
    """Exact (double-double) sums of the terms the fused kernel forms at degree
    m — the reference's rounded terms, or the exact fused-multiply-add
    products (lsqfit_cuda_sum_terms) — as (s_hi, s_lo, s_abs, t_hi, t_lo, t_abs)."""
    from paper_1512_08017_b200 import _capi
    return O.kernel_exact_sums(xy, m, _capi.sum_terms(m) == _capi.TERMS_PRODUCTS)


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.build()
    return oracle

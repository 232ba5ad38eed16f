"""TEST INFRASTRUCTURE ONLY — ctypes wrappers over the CPU oracle.

``oracle.port()`` is the plain-C restatement (``oracle/lsqfit_oracle.c``) of the
reference's normal-equation path; ``oracle.ref()`` is the reference itself,
compiled from /root/reference by ``oracle/Makefile`` into ``oracle/_ref/``.
Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs import this
package: it is the checker, never the measured or shipped path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from functools import lru_cache

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref_lsqfit.so")

OK, EINVAL, EOVERFLOW, ESINGULAR, EDEGREE = 0, 1, 2, 3, 4

_dp = C.POINTER(C.c_double)
_u64 = C.c_uint64


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def build(force: bool = False) -> None:
    """Compile liboracle.so (and _ref when the reference sources are present)."""
    if force or not os.path.exists(PORT_SO) or (
        os.path.exists("/root/reference/proj/src") and not os.path.exists(REF_SO)):
        subprocess.run(["make", "-s", "-C", HERE], check=True)


@lru_cache(None)
def _port():
    if not os.path.exists(PORT_SO):
        build()
    lib = C.CDLL(PORT_SO)
    i, d, u32 = C.c_int, C.c_double, C.c_uint32
    sig = {
        "orc_accumulate": (i, [_dp, _u64, i, _dp, _dp]),
        "orc_accumulate_parallel": (i, [_dp, _u64, i, i, _dp, _dp]),
        "orc_build_normal_system": (None, [_dp, i, _dp]),
        "orc_solve_gaussian": (i, [_dp, _dp, i, _dp]),
        "orc_fit_normal": (i, [_dp, _u64, i, i, _dp]),
        "orc_exact_sums": (i, [_dp, _u64, i, _dp, _dp, _dp, _dp, _dp, _dp]),
        "orc_kahan_pow_sums": (None, [_dp, _u64, i, _dp, _dp]),
        "orc_exact_sums_terms": (i, [_dp, _u64, i] + [_dp] * 12),
        "orc_residual_moments": (None, [_dp, _u64, _dp, i, d, _dp]),
        "orc_fit_batched": (None, [_dp, _u64, u32, i, _dp, C.POINTER(C.c_int32)]),
        "orc_synth": (None, [_dp, _u64, _u64, _u64, i, d]),
        "orc_synth_batched": (None, [_dp, _u64, u32, _u64, i, d]),
        "orc_synth_truth": (None, [_u64, _u64, i, _dp]),
        "orc_generate_synthetic": (i, [_u64, i, d, _u64, _dp]),
        "orc_max_threads": (i, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    return lib


@lru_cache(None)
def _ref():
    if not os.path.exists(REF_SO):
        build()
    if not os.path.exists(REF_SO):
        return None
    lib = C.CDLL(REF_SO)
    i, d, vp = C.c_int, C.c_double, C.c_void_p
    sig = {
        "ref_dataset_new": (vp, [_dp, _u64]),
        "ref_dataset_free": (None, [vp]),
        "ref_accumulate_ds": (i, [vp, i, _dp, _dp]),
        "ref_accumulate_parallel_ds": (i, [vp, i, i, _dp, _dp]),
        "ref_fit_sums_solve_ds": (i, [vp, i, i, _dp, _dp, _dp]),
        "ref_fit_normal_ds": (i, [vp, i, i, _dp, _dp, _dp]),
        "ref_accumulate": (i, [_dp, _u64, i, _dp, _dp]),
        "ref_accumulate_parallel": (i, [_dp, _u64, i, i, _dp, _dp]),
        "ref_solve_gaussian": (i, [_dp, _dp, i, _dp]),
        "ref_solve_from_sums": (i, [_dp, _dp, i, _dp]),
        "ref_fit_normal": (i, [_dp, _u64, i, i, _dp, _dp, _dp]),
        "ref_fit_qr": (i, [_dp, _u64, i, _dp, _dp, _dp]),
        "ref_generate_synthetic": (i, [_u64, i, d, _u64, _dp]),
        "ref_accumulate_oracle": (i, [_dp, _u64, i, _dp, _dp]),
        "ref_fit_batched": (None, [_dp, _u64, C.c_uint32, i, _dp, C.POINTER(C.c_int32)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    return lib


def have_ref() -> bool:
    return _ref() is not None


def _xy(points) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(points, dtype=np.float64)).reshape(-1, 2)
    return a


# ----------------------------------------------------------------------------
# Port (C restatement)
# ----------------------------------------------------------------------------

def accumulate(points, degree: int):
    xy = _xy(points)
    s = np.zeros(2 * max(degree, 0) + 1)
    t = np.zeros(max(degree, 0) + 1)
    st = _port().orc_accumulate(_ptr(xy), len(xy), degree, _ptr(s), _ptr(t))
    return st, s, t


def accumulate_parallel(points, degree: int, chunks: int):
    xy = _xy(points)
    s = np.zeros(2 * max(degree, 0) + 1)
    t = np.zeros(max(degree, 0) + 1)
    st = _port().orc_accumulate_parallel(_ptr(xy), len(xy), degree, chunks, _ptr(s), _ptr(t))
    return st, s, t


def build_normal_system(s: np.ndarray, degree: int) -> np.ndarray:
    s = np.ascontiguousarray(s, dtype=np.float64)
    a = np.zeros((degree + 1) * (degree + 1))
    _port().orc_build_normal_system(_ptr(s), degree, _ptr(a))
    return a.reshape(degree + 1, degree + 1)


def solve_gaussian(a, b):
    a = np.array(a, dtype=np.float64, copy=True, order="C")
    b = np.array(b, dtype=np.float64, copy=True)
    dim = b.shape[0]
    x = np.zeros(dim)
    st = _port().orc_solve_gaussian(_ptr(a), _ptr(b), dim, _ptr(x))
    return st, x


def solve_from_sums(s, t, degree: int):
    return solve_gaussian(build_normal_system(s, degree), t)


def fit_normal(points, degree: int, chunks: int = 1):
    xy = _xy(points)
    c = np.zeros(max(degree, 0) + 1)
    st = _port().orc_fit_normal(_ptr(xy), len(xy), degree, chunks, _ptr(c))
    return st, c


def exact_sums(points, degree: int):
    """Double-double sums of the reference's own terms -> (s_hi, s_lo, s_abs, t_hi, t_lo, t_abs)."""
    xy = _xy(points)
    out = [np.zeros(2 * degree + 1) for _ in range(3)] + [np.zeros(degree + 1) for _ in range(3)]
    _port().orc_exact_sums(_ptr(xy), len(xy), degree, *[_ptr(o) for o in out])
    return tuple(out)


def exact_sums_terms(points, degree: int) -> dict:
    """Exact (double-double) sums of both term families the CUDA kernel may
    form: 'sp' plain powers, 'sx' exact products pw_a*pw_b (a = k//2), 'tr'
    the reference's rounded moments, 'tx' exact moment products; each maps to
    (hi, lo, abs)."""
    xy = _xy(points)
    ns, nt = 2 * degree + 1, degree + 1
    g = {k: tuple(np.zeros(ns if k in ("sp", "sx") else nt) for _ in range(3)) for k in ("sp", "sx", "tr", "tx")}
    st = _port().orc_exact_sums_terms(_ptr(xy), len(xy), degree,
                                      *[_ptr(a) for k in ("sp", "sx", "tr", "tx") for a in g[k]])
    if st != OK:
        raise ValueError("exact_sums_terms: invalid arguments")
    return g


def kernel_term_sums(terms: dict, degree: int, products: bool):
    """(s_hi, s_lo, s_abs, t_hi, t_lo, t_abs) of the terms the fused kernel forms
    at `degree`, from exact_sums_terms() at any degree >= `degree`: the
    reference's terms, or (products) plain powers for k <= m, exact products
    pw_{k//2} * pw_{k-k//2} for k > m, and exact moment products."""
    ns, nt = 2 * degree + 1, degree + 1
    out = []
    for i in range(3):
        s = terms["sp"][i][:ns].copy()
        if products:
            s[degree + 1:] = terms["sx"][i][degree + 1:ns]
        out.append(s)
    for i in range(3):
        out.append((terms["tx"] if products else terms["tr"])[i][:nt].copy())
    return tuple(out)


def residual_moments(points, coeffs, shift: float):
    """(sum r^2, sum (y - shift), sum (y - shift)^2), r = y - Horner(coeffs, x)
    rounded as the reference's evaluate(), each summed exactly."""
    xy = _xy(points)
    c = np.ascontiguousarray(coeffs, dtype=np.float64)
    out = np.zeros(3)
    _port().orc_residual_moments(_ptr(xy), len(xy), _ptr(c), len(c) - 1, float(shift), _ptr(out))
    return float(out[0]), float(out[1]), float(out[2])


def kernel_exact_sums(points, degree: int, products: bool):
    """exact_sums() of the terms the fused CUDA kernel forms at `degree`
    (products: lsqfit_cuda_sum_terms(degree) == LSQFIT_TERMS_PRODUCTS)."""
    if not products:
        return exact_sums(points, degree)
    return kernel_term_sums(exact_sums_terms(points, degree), degree, True)


def kahan_pow_sums(points, degree: int):
    xy = _xy(points)
    s = np.zeros(2 * degree + 1)
    t = np.zeros(degree + 1)
    _port().orc_kahan_pow_sums(_ptr(xy), len(xy), degree, _ptr(s), _ptr(t))
    return s, t


def fit_batched(xy: np.ndarray, n_curves: int, ppc: int, degree: int):
    xy = np.ascontiguousarray(xy, dtype=np.float64)
    coeffs = np.zeros(n_curves * (degree + 1))
    status = np.zeros(n_curves, dtype=np.int32)
    _port().orc_fit_batched(_ptr(xy), n_curves, ppc, degree, _ptr(coeffs),
                            status.ctypes.data_as(C.POINTER(C.c_int32)))
    return coeffs.reshape(n_curves, degree + 1), status


def synth(n: int, offset: int, seed: int, truth_degree: int, sigma: float) -> np.ndarray:
    xy = np.empty((n, 2))
    _port().orc_synth(_ptr(xy), n, offset, seed, truth_degree, sigma)
    return xy


def synth_batched(n_curves: int, ppc: int, seed: int, truth_degree: int, sigma: float) -> np.ndarray:
    xy = np.empty((n_curves * ppc, 2))
    _port().orc_synth_batched(_ptr(xy), n_curves, ppc, seed, truth_degree, sigma)
    return xy


def synth_truth(seed: int, curve: int, truth_degree: int) -> np.ndarray:
    c = np.zeros(truth_degree + 1)
    _port().orc_synth_truth(seed, curve, truth_degree, _ptr(c))
    return c


def generate_synthetic(n: int, degree: int, sigma: float, seed: int) -> np.ndarray:
    xy = np.empty((n, 2))
    st = _port().orc_generate_synthetic(n, degree, sigma, seed, _ptr(xy))
    if st != OK:
        raise ValueError("generate_synthetic: invalid arguments")
    return xy


def max_threads() -> int:
    return int(_port().orc_max_threads())


# ----------------------------------------------------------------------------
# Reference (compiled from /root/reference) — None-safe helpers
# ----------------------------------------------------------------------------

class RefDataset:
    """A reference lsqfit::Dataset built once (untimed)."""

    def __init__(self, xy: np.ndarray):
        lib = _ref()
        if lib is None:
            raise RuntimeError("oracle/_ref not built")
        xy = _xy(xy)
        self._lib = lib
        self.n = len(xy)
        self.h = lib.ref_dataset_new(_ptr(xy), self.n)
        if not self.h:
            raise ValueError("reference Dataset rejected the input")

    def accumulate(self, degree: int):
        s, t = np.zeros(2 * degree + 1), np.zeros(degree + 1)
        st = self._lib.ref_accumulate_ds(self.h, degree, _ptr(s), _ptr(t))
        return st, s, t

    def accumulate_parallel(self, degree: int, chunks: int):
        s, t = np.zeros(2 * degree + 1), np.zeros(degree + 1)
        st = self._lib.ref_accumulate_parallel_ds(self.h, degree, chunks, _ptr(s), _ptr(t))
        return st, s, t

    def fit(self, degree: int, chunks: int):
        s, t, c = np.zeros(2 * degree + 1), np.zeros(degree + 1), np.zeros(degree + 1)
        st = self._lib.ref_fit_sums_solve_ds(self.h, degree, chunks, _ptr(s), _ptr(t), _ptr(c))
        return st, s, t, c

    def fit_normal(self, degree: int, chunks: int):
        """The reference's fit_normal: (status, coeffs, sse, r)."""
        c, sse, r = np.zeros(degree + 1), np.zeros(1), np.zeros(1)
        st = self._lib.ref_fit_normal_ds(self.h, degree, chunks, _ptr(c), _ptr(sse), _ptr(r))
        return st, c, float(sse[0]), float(r[0])

    def close(self):
        if self.h:
            self._lib.ref_dataset_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ref_accumulate(points, degree: int):
    xy = _xy(points)
    s, t = np.zeros(2 * max(degree, 0) + 1), np.zeros(max(degree, 0) + 1)
    st = _ref().ref_accumulate(_ptr(xy), len(xy), degree, _ptr(s), _ptr(t))
    return st, s, t


def ref_accumulate_parallel(points, degree: int, chunks: int):
    xy = _xy(points)
    s, t = np.zeros(2 * max(degree, 0) + 1), np.zeros(max(degree, 0) + 1)
    st = _ref().ref_accumulate_parallel(_ptr(xy), len(xy), degree, chunks, _ptr(s), _ptr(t))
    return st, s, t


def ref_solve_gaussian(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(b.shape[0])
    st = _ref().ref_solve_gaussian(_ptr(a), _ptr(b), b.shape[0], _ptr(x))
    return st, x


def ref_solve_from_sums(s, t, degree: int):
    s = np.ascontiguousarray(s, dtype=np.float64)
    t = np.ascontiguousarray(t, dtype=np.float64)
    x = np.zeros(degree + 1)
    st = _ref().ref_solve_from_sums(_ptr(s), _ptr(t), degree, _ptr(x))
    return st, x


def ref_fit_normal(points, degree: int, chunks: int = 1):
    xy = _xy(points)
    c = np.zeros(max(degree, 0) + 1)
    sse, r = C.c_double(), C.c_double()
    st = _ref().ref_fit_normal(_ptr(xy), len(xy), degree, chunks, _ptr(c), C.byref(sse), C.byref(r))
    return st, c, sse.value, r.value


def ref_fit_qr(points, degree: int):
    """The reference's Householder-QR fit (qr_backend.cpp:126-133)."""
    xy = _xy(points)
    c = np.zeros(max(degree, 0) + 1)
    sse, r = C.c_double(), C.c_double()
    st = _ref().ref_fit_qr(_ptr(xy), len(xy), degree, _ptr(c), C.byref(sse), C.byref(r))
    return st, c, sse.value, r.value


def ref_generate_synthetic(n: int, degree: int, sigma: float, seed: int) -> np.ndarray:
    xy = np.empty((n, 2))
    st = _ref().ref_generate_synthetic(n, degree, sigma, seed, _ptr(xy))
    if st != OK:
        raise ValueError("generate_synthetic failed")
    return xy


def ref_accumulate_oracle(points, degree: int):
    xy = _xy(points)
    s, t = np.zeros(2 * degree + 1), np.zeros(degree + 1)
    _ref().ref_accumulate_oracle(_ptr(xy), len(xy), degree, _ptr(s), _ptr(t))
    return s, t


def ref_fit_batched(xy: np.ndarray, n_curves: int, ppc: int, degree: int):
    """The reference's per-curve path (Dataset -> accumulate -> build_normal_system
    -> solve_gaussian) in an OpenMP loop over curves -> (coeffs, status)."""
    xy = np.ascontiguousarray(xy, dtype=np.float64)
    coeffs = np.zeros(n_curves * (degree + 1))
    status = np.zeros(n_curves, dtype=np.int32)
    _ref().ref_fit_batched(_ptr(xy), n_curves, ppc, degree, _ptr(coeffs),
                           status.ctypes.data_as(C.POINTER(C.c_int32)))
    return coeffs.reshape(n_curves, degree + 1), status

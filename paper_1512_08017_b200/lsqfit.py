"""Python mirror of the reference's ``lsqfit`` fit/solve interface, GPU-backed.

Same names, argument meaning and error behaviour as the reference C++ API
(citations relative to /root/reference/proj):

=====================================  ========================================
reference                              here
=====================================  ========================================
``Dataset`` (dataset.hpp:18-37)        :class:`Dataset` (same validation)
``PowerSums`` (power_sums.hpp:13-18)   :class:`PowerSums`
``accumulate`` (power_sums.hpp:23)     :func:`accumulate`
``accumulate_parallel`` (:31)          :func:`accumulate_parallel`
``NormalSystem`` (normal_backend.hpp)  :class:`NormalSystem`
``build_normal_system`` (:17)          :func:`build_normal_system`
``solve_gaussian`` (:22)               :func:`solve_gaussian`
``fit_normal`` (:27)                   :func:`fit_normal`
``FitReport`` (diagnostics.hpp:21-28)  :class:`FitReport`
errors.hpp:10-68                       :class:`InputError`, :class:`NumericError`,
                                       :class:`OverflowError`, :class:`SingularSystemError`,
                                       :class:`DegreeTooHighError`; ``std::invalid_argument``
                                       maps to :class:`ValueError`
=====================================  ========================================

Every numeric operation runs in the sm_100a library through the C ABI
(``include/lsqfit_cuda.h``): the power sums, the finite check, the solve and
the diagnostics pass. ``chunks`` is validated as the reference does and then
ignored for partitioning: the device reduction order is a fixed function of
(data, degree, GPU), so the result is still a pure function of
(dataset, degree, chunks) and ``accumulate_parallel(d, m, 1)`` is
bit-identical to ``accumulate(d, m)`` (power_sums.hpp:25-31).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _capi

K_MAX_DEGREE = 12  # diagnostics.hpp:13


# ---------------------------------------------------------------------------
# errors.hpp
# ---------------------------------------------------------------------------

class InputError(RuntimeError):
    pass


class NumericError(RuntimeError):
    pass


class OverflowError(NumericError):  # noqa: A001 - mirrors lsqfit::OverflowError
    pass


class SingularSystemError(NumericError):
    pass


class RankDeficientError(NumericError):
    pass


class DegreeTooHighError(NumericError):
    pass


def _raise_for(status: int, what: str) -> None:
    if status == _capi.OK:
        return
    if status == _capi.EOVERFLOW:
        raise OverflowError(f"{what}: non-finite result; the data scale is incompatible with this degree")
    if status == _capi.ESINGULAR:
        raise SingularSystemError(f"{what}: singular normal system (fewer than degree+1 distinct x values, "
                                  "or hopeless conditioning)")
    if status == _capi.EDEGREE:
        raise DegreeTooHighError(f"{what}: degree exceeds the cap of {K_MAX_DEGREE}")
    if status == _capi.EINVAL:
        raise ValueError(f"{what}: invalid argument")
    raise _capi.CudaError(f"{what}: {_capi.STATUS_NAMES.get(status, status)}")


# ---------------------------------------------------------------------------
# Domain types
# ---------------------------------------------------------------------------

class Dataset:
    """Ordered, immutable (x, y) samples; AoS float64 of shape (n, 2).

    Rejects empty input and non-finite coordinates (dataset.hpp:20-26).
    """

    def __init__(self, points):
        arr = np.array(points, dtype=np.float64, copy=True, order="C")
        if arr.size == 0:
            raise ValueError("dataset must contain at least one point")
        arr = arr.reshape(-1, 2)
        if not np.isfinite(arr).all():
            raise ValueError("dataset coordinates must be finite")
        arr.setflags(write=False)
        self._xy = arr

    @classmethod
    def _trusted(cls, arr: np.ndarray) -> "Dataset":
        d = cls.__new__(cls)
        d._xy = arr
        return d

    def size(self) -> int:
        return self._xy.shape[0]

    __len__ = size

    def points(self) -> np.ndarray:
        return self._xy

    def __getitem__(self, i):
        return tuple(self._xy[i])

    def __iter__(self):
        return (tuple(p) for p in self._xy)


@dataclass
class PowerSums:
    degree: int = 0
    s: list = field(default_factory=list)  # 2*degree + 1
    t: list = field(default_factory=list)  # degree + 1
    n: int = 0


@dataclass
class NormalSystem:
    a: np.ndarray
    b: np.ndarray
    degree: int = 0


class Polynomial:
    """a_0 + a_1 x + ... + a_m x^m, ascending (polynomial.hpp:11-27)."""

    def __init__(self, coefficients):
        c = [float(v) for v in coefficients]
        if not c:
            raise ValueError("polynomial needs at least one coefficient")
        if not all(np.isfinite(c)):
            raise ValueError("polynomial coefficients must be finite")
        self._c = c

    def degree(self) -> int:
        return len(self._c) - 1

    def coefficients(self) -> list:
        return list(self._c)


@dataclass
class FitReport:
    polynomial: Polynomial
    backend: str
    residuals: np.ndarray
    sse: float
    r: float
    n_points: int


# ---------------------------------------------------------------------------
# Operations
# ---------------------------------------------------------------------------

def _ctx():
    return _capi.context(0)


def _xy_ptr(dataset: Dataset) -> int:
    return dataset.points().ctypes.data


def _sums_from(r: _capi.Result, degree: int) -> PowerSums:
    return PowerSums(degree=degree, s=list(r.s[: 2 * degree + 1]), t=list(r.t[: degree + 1]), n=int(r.n))


_REFERENCE_ORDER = False


def set_reference_order(enabled: bool) -> None:
    """Reference-order mode: accumulate / accumulate_parallel reproduce the
    reference's bits exactly (same chunk boundaries, sequential per-chunk
    chains and ascending combine, one GPU thread per chunk). Fast when chunks
    is large (>= ~1e4); exact but slow for few chunks (accumulate() itself is
    a single chain). Default off: the compensated fused kernel."""
    global _REFERENCE_ORDER
    _REFERENCE_ORDER = bool(enabled)


def _ordered(dataset: Dataset, degree: int, chunks: int) -> PowerSums:
    st, r = _ctx().fit_ordered_host(_xy_ptr(dataset), dataset.size(), degree, chunks, _capi.SUMS)
    _raise_for(st, "accumulate")
    return _sums_from(r, degree)


def _any_degree(dataset: Dataset, degree: int, chunks: int = 1) -> PowerSums:
    """Degrees above the fused kernels' cap: the generic any-degree kernel
    (the reference's accumulate has no cap, power_sums.hpp:20-31), or in
    reference-order mode its bit-exact column replay."""
    if _REFERENCE_ORDER:
        st, s, t = _ctx().power_sums_ordered_host(_xy_ptr(dataset), dataset.size(), degree, chunks)
    else:
        st, s, t = _ctx().power_sums_host(_xy_ptr(dataset), dataset.size(), degree)
    _raise_for(st, "accumulate")
    return PowerSums(degree=degree, s=list(s), t=list(t), n=dataset.size())


def accumulate(dataset: Dataset, degree: int) -> PowerSums:
    """power_sums.cpp:39-50 on the GPU (one fused streaming launch)."""
    if degree < 0:
        raise ValueError("degree must be nonnegative")
    if degree > _capi.MAX_DEGREE:
        return _any_degree(dataset, degree)
    if _REFERENCE_ORDER:
        return _ordered(dataset, degree, 1)
    st, r = _ctx().fit_host(_xy_ptr(dataset), dataset.size(), degree, _capi.SUMS)
    _raise_for(st, "accumulate")
    return _sums_from(r, degree)


def accumulate_parallel(dataset: Dataset, degree: int, chunks: int) -> PowerSums:
    """power_sums.cpp:52-90: same validation; the device grid is the parallelism
    (or, in reference-order mode, exactly the reference's `chunks` slices)."""
    if degree < 0:
        raise ValueError("degree must be nonnegative")
    if chunks < 1:
        raise ValueError("chunks must be at least 1")
    if degree > _capi.MAX_DEGREE:
        return _any_degree(dataset, degree, chunks)
    if _REFERENCE_ORDER:
        return _ordered(dataset, degree, chunks)
    return accumulate(dataset, degree)


def build_normal_system(sums: PowerSums) -> NormalSystem:
    """normal_backend.cpp:13-20: a(j,k) = s[j+k], b = t (exact copies)."""
    dim = sums.degree + 1
    s = np.asarray(sums.s, dtype=np.float64)
    j = np.arange(dim)
    return NormalSystem(a=s[j[:, None] + j[None, :]].copy(), b=np.array(sums.t, dtype=np.float64),
                        degree=sums.degree)


def solve_gaussian(system: NormalSystem) -> Polynomial:
    """normal_backend.cpp:22-74, computed by one GPU warp (bit-identical ops)."""
    a = np.ascontiguousarray(system.a, dtype=np.float64)
    b = np.ascontiguousarray(system.b, dtype=np.float64)
    dim = a.shape[0] if a.ndim == 2 else 0
    if dim == 0 or a.shape != (dim, dim) or b.shape != (dim,):
        raise ValueError("normal system dimensions are inconsistent")
    if dim > _capi.MAX_SOLVE_DIM:
        raise ValueError(f"system dimension {dim} exceeds the device solver's cap of {_capi.MAX_SOLVE_DIM}")
    x = np.zeros(dim)
    st = _ctx().solve_host(a.ctypes.data, b.ctypes.data, dim, x.ctypes.data)
    _raise_for(st, "solve_gaussian")
    return Polynomial(x)


def fit_normal(dataset: Dataset, degree: int, chunks: int = 1) -> FitReport:
    """normal_backend.cpp:76-85: sums + solve (one launch) + diagnostics pass."""
    if degree < 0:
        raise ValueError("degree must be nonnegative")
    if degree > K_MAX_DEGREE:
        raise DegreeTooHighError(f"degree {degree} exceeds the cap of {K_MAX_DEGREE}")
    if chunks < 1:
        raise ValueError("chunks must be at least 1")
    if _REFERENCE_ORDER:
        # as the C++ drop-in (cpp/lsqfit_b200.cpp fit_normal): the reference's
        # sums bit for bit over its `chunks` slices, its solve bit for bit,
        # then the device report pass
        st, r = _ctx().fit_ordered_host(_xy_ptr(dataset), dataset.size(), degree, chunks, _capi.SOLVE)
        _raise_for(st, "fit_normal")
        _raise_for(r.status, "fit_normal")
        return make_fit_report(dataset, Polynomial(list(r.coeffs[: degree + 1])), "normal")
    n = dataset.size()
    res = np.empty(n)
    r = _capi.Result()
    d = _capi.Diag()
    ctx = _ctx()
    st = ctx._lib.lsqfit_cuda_fit_report_host(ctx.h, C.cast(C.c_void_p(_xy_ptr(dataset)), C.POINTER(C.c_double)),
                                              n, degree, C.byref(r), C.byref(d),
                                              res.ctypes.data_as(C.POINTER(C.c_double)))
    ctx.check(st, "fit_normal")
    _raise_for(r.status, "fit_normal")
    if d.status != _capi.OK:
        raise OverflowError("polynomial evaluation overflowed on the input data")
    poly = Polynomial(list(r.coeffs[: degree + 1]))
    return FitReport(polynomial=poly, backend="normal", residuals=res, sse=float(d.sse), r=float(d.r),
                     n_points=n)


def fit_qr(dataset: Dataset, degree: int) -> FitReport:
    """fit_qr (qr_backend.cpp:126-133) on the GPU: TSQR of the augmented
    Vandermonde rows (orthogonal factorisation, cond(V) not cond(V)^2), then
    the device diagnostics pass. RankDeficientError as the reference's
    householder_qr; degrees above MAX_QR_DEGREE (12) exceed the TSQR kernels (ValueError)."""
    if degree < 0:
        raise ValueError("degree must be nonnegative")
    if degree > K_MAX_DEGREE:
        raise DegreeTooHighError(f"degree {degree} exceeds the cap of {K_MAX_DEGREE}")
    if degree > _capi.MAX_QR_DEGREE:
        raise ValueError(f"degree {degree} exceeds the TSQR kernels' cap of {_capi.MAX_QR_DEGREE}")
    ctx = _ctx()
    n = dataset.size()
    st, q = ctx.qr_fit_host(_xy_ptr(dataset), n, degree)
    if st == _capi.ERANKDEF:
        raise RankDeficientError("rank-deficient system (fewer than degree+1 distinct x values)")
    _raise_for(st, "fit_qr")
    coeffs = list(q.coeffs[: degree + 1])
    res = np.empty(n)
    d = _capi.Diag()
    c_arr = (C.c_double * (degree + 1))(*coeffs)
    st = ctx._lib.lsqfit_cuda_report_host(ctx.h, C.cast(C.c_void_p(_xy_ptr(dataset)), C.POINTER(C.c_double)), n,
                                          c_arr, degree, C.byref(d), res.ctypes.data_as(C.POINTER(C.c_double)))
    ctx.check(st, "fit_qr diagnostics")
    if d.status != _capi.OK:
        raise OverflowError("polynomial evaluation overflowed on the input data")
    return FitReport(polynomial=Polynomial(coeffs), backend="qr", residuals=res, sse=float(d.sse), r=float(d.r),
                     n_points=n)


def _report(dataset: Dataset, coeffs, want_residuals: bool):
    n = dataset.size()
    res = np.empty(n) if want_residuals else None
    d = _capi.Diag()
    degree = len(coeffs) - 1
    c_arr = (C.c_double * (degree + 1))(*[float(v) for v in coeffs])
    ctx = _ctx()
    st = ctx._lib.lsqfit_cuda_report_host(ctx.h, C.cast(C.c_void_p(_xy_ptr(dataset)), C.POINTER(C.c_double)), n,
                                          c_arr, degree, C.byref(d),
                                          res.ctypes.data_as(C.POINTER(C.c_double)) if res is not None else None)
    ctx.check(st, "diagnostics")
    return d, res


def residuals(dataset: Dataset, poly: Polynomial) -> np.ndarray:
    """diagnostics.cpp:14-19: y_i - evaluate(poly, x_i) for every point, on the
    device (Horner rounded exactly as polynomial.cpp:5-11); any degree."""
    return _report(dataset, poly.coefficients(), True)[1]


def sum_squared_error(res) -> float:
    """diagnostics.cpp:21-25 over a caller-owned residual vector (host utility)."""
    sse = 0.0
    for e in np.asarray(res, dtype=np.float64):
        sse += float(e) * float(e)
    return sse


def correlation_coefficient(dataset: Dataset, sse: float) -> float:
    """diagnostics.cpp:27-38: R = sqrt(max(0, 1 - sse/sst)); sst from the device pass."""
    d, _ = _report(dataset, [0.0], False)
    n = dataset.size()
    if d.sst == 0.0:
        return 1.0 if sse <= 1e-12 * n else 0.0
    v = 1.0 - sse / d.sst
    return float(np.sqrt(v if v > 0.0 else 0.0))


def make_fit_report(dataset: Dataset, poly: Polynomial, backend: str = "normal") -> FitReport:
    """diagnostics.cpp:40-48: residuals, SSE and R of `poly` on `dataset` in
    one device pass; OverflowError for a non-finite residual; any degree."""
    d, res = _report(dataset, poly.coefficients(), True)
    if d.status != _capi.OK:
        raise OverflowError("polynomial evaluation overflowed on the input data")
    return FitReport(polynomial=poly, backend=backend, residuals=res, sse=float(d.sse), r=float(d.r),
                     n_points=dataset.size())


# ------------------------------------------------ batched fits (B200 extension)

def fit_batched(points, n_curves: int, points_per_curve: int, degree: int):
    """Many independent fits in one launch (lsqfit::cuda::fit_batched): curve c =
    points[c*ppc, (c+1)*ppc) of a host (n, 2) float64 array. Returns
    (coeffs [n_curves, degree+1], status [n_curves]: 0 ok, 2 overflow, 3 singular)."""
    xy = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
    if degree < 0 or degree > K_MAX_DEGREE:
        raise ValueError(f"degree must be in [0, {K_MAX_DEGREE}]")
    if points_per_curve < 1 or len(xy) < n_curves * points_per_curve:
        raise ValueError("need n_curves * points_per_curve points")
    coeffs = np.zeros((n_curves, degree + 1))
    status = np.zeros(n_curves, dtype=np.int32)
    if n_curves == 0:
        return coeffs, status
    ctx = _ctx()
    dp = C.POINTER(C.c_double)
    st = ctx._lib.lsqfit_cuda_fit_batched_host(ctx.h, xy.ctypes.data_as(dp), n_curves, points_per_curve, degree,
                                               coeffs.ctypes.data_as(dp), status.ctypes.data_as(C.POINTER(C.c_int32)))
    ctx.check(st, "fit_batched")
    _raise_for(st, "fit_batched")
    return coeffs, status


def fit_batched_ragged(points, offsets, degree: int):
    """Curves of different lengths (lsqfit::cuda::fit_batched_ragged): curve c =
    points[offsets[c], offsets[c+1]); empty curves get status 3."""
    xy = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    if degree < 0 or degree > K_MAX_DEGREE:
        raise ValueError(f"degree must be in [0, {K_MAX_DEGREE}]")
    if off.ndim != 1 or off.size < 1 or np.any(off[1:] < off[:-1]) or (off.size and int(off[-1]) > len(xy)):
        raise ValueError("offsets must be n_curves + 1 non-decreasing indices into points")
    n_curves = off.size - 1
    coeffs = np.zeros((n_curves, degree + 1))
    status = np.zeros(n_curves, dtype=np.int32)
    if n_curves == 0:
        return coeffs, status
    ctx = _ctx()
    dp = C.POINTER(C.c_double)
    st = ctx._lib.lsqfit_cuda_fit_batched_ragged_host(ctx.h, xy.ctypes.data_as(dp),
                                                      off.ctypes.data_as(C.POINTER(C.c_uint64)), n_curves, degree,
                                                      coeffs.ctypes.data_as(dp),
                                                      status.ctypes.data_as(C.POINTER(C.c_int32)))
    ctx.check(st, "fit_batched_ragged")
    _raise_for(st, "fit_batched_ragged")
    return coeffs, status


# ------------------------------------------------------- fit facade (fit.hpp)

@dataclass
class FitOutcome:
    """fit.hpp:20-27: one report per backend (normal first for both)."""
    reports: list
    max_coef_discrepancy: float | None = None
    backends_agree: bool = True


def max_coefficient_discrepancy(a: Polynomial, b: Polynomial) -> float:
    """fit.cpp:12-21: max_k |a_k - b_k| (same degree required)."""
    ca, cb = a.coefficients(), b.coefficients()
    if len(ca) != len(cb):
        raise ValueError("polynomials have different degrees")
    return max((abs(x - y) for x, y in zip(ca, cb)), default=0.0)


def coefficients_agree(a: Polynomial, b: Polynomial, rel_tol: float) -> bool:
    """fit.cpp:23-32: |a_k - b_k| <= rel_tol * (1 + max(|a_k|, |b_k|)) for all k."""
    ca, cb = a.coefficients(), b.coefficients()
    if len(ca) != len(cb):
        return False
    return all(abs(x - y) <= rel_tol * (1.0 + max(abs(x), abs(y))) for x, y in zip(ca, cb))


def fit(dataset: Dataset, degree: int, backend: str = "normal", chunks: int = 1) -> FitOutcome:
    """fit.cpp:34-57: dispatch to the normal and/or QR (TSQR) backend."""
    if degree < 0:
        raise ValueError("degree must be nonnegative")
    if chunks < 1:
        raise ValueError("chunks must be at least 1")
    if backend == "normal":
        return FitOutcome(reports=[fit_normal(dataset, degree, chunks)])
    if backend == "qr":
        return FitOutcome(reports=[fit_qr(dataset, degree)])
    if backend == "both":
        rn, rq = fit_normal(dataset, degree, chunks), fit_qr(dataset, degree)
        return FitOutcome(reports=[rn, rq],
                          max_coef_discrepancy=max_coefficient_discrepancy(rn.polynomial, rq.polynomial),
                          backends_agree=coefficients_agree(rn.polynomial, rq.polynomial, 1e-4))
    raise ValueError(f"unknown backend {backend!r} (normal, qr, both)")


def evaluate(poly: Polynomial, x: float) -> float:
    """Horner (polynomial.cpp:5-11) — host utility for callers, not on the hot path."""
    c = poly.coefficients()
    acc = c[-1]
    for v in reversed(c[:-1]):
        acc = acc * x + v
    return acc

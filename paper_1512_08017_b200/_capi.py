"""ctypes binding of the C ABI declared in include/lsqfit_cuda.h.

The shared library ``lib/liblsqfit_cuda.so`` is the product: hand-written
sm_100a kernels behind a plain C interface. This module only marshals
pointers and sizes; there is no computational fallback — if the library or a
CUDA device is missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from functools import lru_cache

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
# LSQFIT_CUDA_LIB: load another in-tree build of the same library (A/B tooling, tools/*.py)
LIB_PATH = os.environ.get("LSQFIT_CUDA_LIB") or os.path.join(PKG_DIR, "lib", "liblsqfit_cuda.so")
DROPIN_PATH = os.path.join(PKG_DIR, "lib", "liblsqfit_b200.so")

MAX_DEGREE = 12
MAX_NV = 3 * MAX_DEGREE + 1
MAX_SOLVE_DIM = 4096

OK, EINVAL, EOVERFLOW, ESINGULAR, EDEGREE, ECUDA, ENOMEM = range(7)
SUMS, SOLVE = 0, 1

STATUS_NAMES = {OK: "OK", EINVAL: "EINVAL", EOVERFLOW: "EOVERFLOW", ESINGULAR: "ESINGULAR",
                EDEGREE: "EDEGREE", ECUDA: "ECUDA", ENOMEM: "ENOMEM"}


class Result(C.Structure):
    """Mirror of ``lsqfit_result`` (include/lsqfit_cuda.h)."""

    _fields_ = [
        ("s", C.c_double * (2 * MAX_DEGREE + 1)),
        ("t", C.c_double * (MAX_DEGREE + 1)),
        ("coeffs", C.c_double * (MAX_DEGREE + 1)),
        ("part_hi", C.c_double * MAX_NV),
        ("part_lo", C.c_double * MAX_NV),
        ("n", C.c_uint64),
        ("degree", C.c_int32),
        ("status", C.c_int32),
    ]


RESULT_BYTES = C.sizeof(Result)


class Diag(C.Structure):
    """Mirror of ``lsqfit_diag`` (include/lsqfit_cuda.h)."""

    _fields_ = [("sse", C.c_double), ("r", C.c_double), ("sum_y", C.c_double), ("sst", C.c_double),
                ("part_hi", C.c_double * 3), ("part_lo", C.c_double * 3), ("shift", C.c_double),
                ("n", C.c_uint64),
                ("status", C.c_int32), ("pad", C.c_int32)]


DIAG_BYTES = C.sizeof(Diag)

MAX_QR_DEGREE = 12
ERANKDEF = 7
STATUS_NAMES[ERANKDEF] = "ERANKDEF"


class QrResult(C.Structure):
    """Mirror of ``lsqfit_qr_result`` (include/lsqfit_cuda.h)."""

    _fields_ = [("r", C.c_double * ((MAX_DEGREE + 2) * (MAX_DEGREE + 2))),
                ("coeffs", C.c_double * (MAX_DEGREE + 1)), ("residual_norm", C.c_double),
                ("n", C.c_uint64), ("degree", C.c_int32), ("status", C.c_int32)]


QR_BYTES = C.sizeof(QrResult)


def build_library(force: bool = False) -> None:
    """Compile the sm_100a library in-tree (nvcc cross-compiles; no GPU needed)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", REPO_DIR, os.path.relpath(LIB_PATH, REPO_DIR)], check=True)


_lock = threading.RLock()


@lru_cache(None)
def lib() -> C.CDLL:
    with _lock:
        if not os.path.exists(LIB_PATH):
            build_library()
        L = C.CDLL(LIB_PATH)
    vp, i, u32, u64, d = C.c_void_p, C.c_int, C.c_uint32, C.c_uint64, C.c_double
    dp = C.POINTER(C.c_double)
    sig = {
        "lsqfit_cuda_create": (i, [C.POINTER(vp), i]),
        "lsqfit_cuda_destroy": (None, [vp]),
        "lsqfit_cuda_strerror": (C.c_char_p, [i]),
        "lsqfit_cuda_last_error": (C.c_char_p, [vp]),
        "lsqfit_cuda_grid_size": (i, [vp, C.POINTER(i)]),
        "lsqfit_cuda_sum_error_levels": (i, [i]),
        "lsqfit_cuda_sum_terms": (i, [i]),
        "lsqfit_cuda_power_sums_host": (i, [vp, dp, u64, i, dp, dp]),
        "lsqfit_cuda_release_buffers": (i, [vp]),
        "lsqfit_cuda_power_sums_ordered_host": (i, [vp, dp, u64, i, u64, dp, dp]),
        "lsqfit_cuda_solve_sums_host": (i, [vp, dp, dp, i, dp]),
        "lsqfit_cuda_group_fit_device": (i, [vp, C.POINTER(vp), C.POINTER(u64), i, C.c_uint, C.POINTER(Result)]),
        "lsqfit_cuda_fit_batched_ragged_device": (i, [vp, vp, vp, u64, u64, i, vp, vp, vp]),
        "lsqfit_cuda_fit_batched_ragged_host": (i, [vp, dp, C.POINTER(u64), u64, i, dp, C.POINTER(C.c_int32)]),
        "lsqfit_cuda_power_sums_device": (i, [vp, vp, u64, i, vp, vp, vp]),
        "lsqfit_cuda_set_stream_chunk": (i, [vp, u64]),
        "lsqfit_cuda_fit_host": (i, [vp, dp, u64, i, C.c_uint, C.POINTER(Result)]),
        "lsqfit_cuda_fit_report_host": (i, [vp, dp, u64, i, C.POINTER(Result), C.POINTER(Diag), dp]),
        "lsqfit_cuda_report_host": (i, [vp, dp, u64, dp, i, C.POINTER(Diag), dp]),
        "lsqfit_cuda_fit_batched_host": (i, [vp, dp, u64, u32, i, dp, C.POINTER(C.c_int32)]),
        "lsqfit_cuda_fit_device": (i, [vp, vp, u64, i, C.c_uint, vp, vp]),
        "lsqfit_cuda_fit_ordered_device": (i, [vp, vp, u64, i, u64, C.c_uint, vp, vp]),
        "lsqfit_cuda_fit_ordered_host": (i, [vp, dp, u64, i, u64, C.c_uint, C.POINTER(Result)]),
        "lsqfit_cuda_qr_fit_device": (i, [vp, vp, u64, i, C.c_uint, vp, vp]),
        "lsqfit_cuda_qr_combine_device": (i, [vp, vp, i, i, C.c_uint, vp, vp]),
        "lsqfit_cuda_qr_fit_host": (i, [vp, dp, u64, i, C.POINTER(QrResult)]),
        "lsqfit_cuda_group_create": (i, [C.POINTER(vp), C.POINTER(i), i]),
        "lsqfit_cuda_group_destroy": (None, [vp]),
        "lsqfit_cuda_group_size": (i, [vp]),
        "lsqfit_cuda_group_fit_host": (i, [vp, dp, u64, i, C.c_uint, C.POINTER(Result)]),
        "lsqfit_cuda_group_fit_report_host": (i, [vp, dp, u64, i, C.POINTER(Result), C.POINTER(Diag), dp]),
        "lsqfit_cuda_diagnostics_device": (i, [vp, vp, u64, i, vp, vp, d, vp, vp, vp]),
        "lsqfit_cuda_combine_device": (i, [vp, vp, i, i, C.c_uint, vp, vp]),
        "lsqfit_cuda_solve_host": (i, [vp, dp, dp, i, dp]),
        "lsqfit_cuda_fit_batched_device": (i, [vp, vp, u64, u32, i, vp, vp, vp]),
        "lsqfit_cuda_synth_device": (i, [vp, vp, u64, u64, u64, i, d, vp]),
        "lsqfit_cuda_synth_batched_device": (i, [vp, vp, u64, u32, u64, i, d, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    return L


def exported_symbols() -> list[str]:
    """Names the header declares (used by the CPU export test)."""
    return ["lsqfit_cuda_create", "lsqfit_cuda_destroy", "lsqfit_cuda_strerror", "lsqfit_cuda_last_error",
            "lsqfit_cuda_grid_size", "lsqfit_cuda_set_stream_chunk", "lsqfit_cuda_fit_host", "lsqfit_cuda_fit_report_host",
            "lsqfit_cuda_fit_device", "lsqfit_cuda_diagnostics_device", "lsqfit_cuda_report_host",
            "lsqfit_cuda_fit_ordered_device", "lsqfit_cuda_fit_ordered_host",
            "lsqfit_cuda_fit_batched_host", "lsqfit_cuda_qr_fit_device", "lsqfit_cuda_qr_combine_device",
            "lsqfit_cuda_qr_fit_host", "lsqfit_cuda_group_create", "lsqfit_cuda_group_destroy",
            "lsqfit_cuda_group_size", "lsqfit_cuda_group_fit_host", "lsqfit_cuda_group_fit_report_host",
            "lsqfit_cuda_combine_device", "lsqfit_cuda_solve_host", "lsqfit_cuda_fit_batched_device",
            "lsqfit_cuda_synth_device", "lsqfit_cuda_synth_batched_device", "lsqfit_cuda_sum_error_levels",
            "lsqfit_cuda_sum_terms",
            "lsqfit_cuda_power_sums_host", "lsqfit_cuda_power_sums_device", "lsqfit_cuda_release_buffers",
            "lsqfit_cuda_power_sums_ordered_host", "lsqfit_cuda_solve_sums_host", "lsqfit_cuda_group_fit_device",
            "lsqfit_cuda_fit_batched_ragged_device", "lsqfit_cuda_fit_batched_ragged_host"]


def sum_error_levels(degree: int) -> int:
    """L of the stated power-sum bound |S - S_exact| <= L*2^-53*sum|T| + ulp(S_exact)
    at ``degree`` (host-only query; -1 outside [0, 12])."""
    return int(lib().lsqfit_cuda_sum_error_levels(degree))


TERMS_REFERENCE, TERMS_PRODUCTS = 0, 1


def sum_terms(degree: int) -> int:
    """Which terms the fused kernel sums at ``degree``: TERMS_REFERENCE (the
    reference's rounded terms, degrees 0..2) or TERMS_PRODUCTS (exact
    fused-multiply-add products, degrees 3..12); -1 outside [0, 12]."""
    return int(lib().lsqfit_cuda_sum_terms(degree))


class CudaError(RuntimeError):
    pass


class Context:
    """One ``lsqfit_cuda_ctx``: a CUDA device plus grow-only scratch."""

    def __init__(self, device: int = 0):
        self._lib = lib()
        h = C.c_void_p()
        st = self._lib.lsqfit_cuda_create(C.byref(h), device)
        if st != OK:
            raise CudaError(f"lsqfit_cuda_create(device={device}) failed: "
                            f"{self._lib.lsqfit_cuda_strerror(st).decode()}")
        self.h = h
        self.device = device

    def close(self) -> None:
        if getattr(self, "h", None):
            self._lib.lsqfit_cuda_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def last_error(self) -> str:
        return self._lib.lsqfit_cuda_last_error(self.h).decode()

    def check(self, st: int, what: str) -> int:
        if st in (ECUDA, ENOMEM):
            raise CudaError(f"{what}: {STATUS_NAMES[st]} ({self.last_error()})")
        return st

    def grid_size(self) -> int:
        g = C.c_int()
        self._lib.lsqfit_cuda_grid_size(self.h, C.byref(g))
        return g.value

    def set_stream_chunk(self, points: int) -> None:
        """Host-path out-of-core granule (points); 0 = default (2^27)."""
        self._lib.lsqfit_cuda_set_stream_chunk(self.h, points)

    # ---- host-resident path -------------------------------------------------
    def fit_host(self, xy_ptr: int, n: int, degree: int, flags: int) -> tuple[int, Result]:
        r = Result()
        st = self._lib.lsqfit_cuda_fit_host(self.h, C.cast(C.c_void_p(xy_ptr), C.POINTER(C.c_double)), n,
                                            degree, flags, C.byref(r))
        return self.check(st, "lsqfit_cuda_fit_host"), r

    def release_buffers(self) -> None:
        """Free the grow-only device / pinned buffers (re-allocated on demand)."""
        self.check(self._lib.lsqfit_cuda_release_buffers(self.h), "lsqfit_cuda_release_buffers")

    def power_sums_host(self, xy_ptr: int, n: int, degree: int):
        """Any-degree power sums of host points -> (status, s[2m+1], t[m+1])."""
        import numpy as np
        s = np.zeros(2 * degree + 1)
        t = np.zeros(degree + 1)
        dptr = C.POINTER(C.c_double)
        st = self._lib.lsqfit_cuda_power_sums_host(self.h, C.cast(C.c_void_p(xy_ptr), dptr), n, degree,
                                                   s.ctypes.data_as(dptr), t.ctypes.data_as(dptr))
        return self.check(st, "lsqfit_cuda_power_sums_host"), s, t

    def power_sums_ordered_host(self, xy_ptr: int, n: int, degree: int, chunks: int):
        """Reference-order (bit-exact) sums at any degree -> (status, s, t)."""
        import numpy as np
        s = np.zeros(2 * degree + 1)
        t = np.zeros(degree + 1)
        dptr = C.POINTER(C.c_double)
        st = self._lib.lsqfit_cuda_power_sums_ordered_host(self.h, C.cast(C.c_void_p(xy_ptr), dptr), n, degree,
                                                           chunks, s.ctypes.data_as(dptr), t.ctypes.data_as(dptr))
        return self.check(st, "lsqfit_cuda_power_sums_ordered_host"), s, t

    def power_sums_device(self, d_xy: int, n: int, degree: int, d_st: int, d_status: int, stream: int = 0) -> int:
        st = self._lib.lsqfit_cuda_power_sums_device(self.h, d_xy, n, degree, d_st, d_status, stream)
        return self.check(st, "lsqfit_cuda_power_sums_device")

    def fit_ordered_host(self, xy_ptr: int, n: int, degree: int, chunks: int, flags: int) -> tuple[int, Result]:
        r = Result()
        st = self._lib.lsqfit_cuda_fit_ordered_host(self.h, C.cast(C.c_void_p(xy_ptr), C.POINTER(C.c_double)), n,
                                                    degree, chunks, flags, C.byref(r))
        return self.check(st, "lsqfit_cuda_fit_ordered_host"), r

    def fit_ordered_device(self, d_xy: int, n: int, degree: int, chunks: int, flags: int, d_result: int,
                           stream: int = 0) -> int:
        st = self._lib.lsqfit_cuda_fit_ordered_device(self.h, d_xy, n, degree, chunks, flags, d_result, stream)
        return self.check(st, "lsqfit_cuda_fit_ordered_device")

    def qr_fit_host(self, xy_ptr: int, n: int, degree: int) -> tuple[int, "QrResult"]:
        r = QrResult()
        st = self._lib.lsqfit_cuda_qr_fit_host(self.h, C.cast(C.c_void_p(xy_ptr), C.POINTER(C.c_double)), n,
                                               degree, C.byref(r))
        return self.check(st, "lsqfit_cuda_qr_fit_host"), r

    def qr_fit_device(self, d_xy: int, n: int, degree: int, flags: int, d_result: int, stream: int = 0) -> int:
        st = self._lib.lsqfit_cuda_qr_fit_device(self.h, d_xy, n, degree, flags, d_result, stream)
        return self.check(st, "lsqfit_cuda_qr_fit_device")

    def qr_combine_device(self, d_parts: int, n_parts: int, degree: int, flags: int, d_result: int,
                          stream: int = 0) -> int:
        st = self._lib.lsqfit_cuda_qr_combine_device(self.h, d_parts, n_parts, degree, flags, d_result, stream)
        return self.check(st, "lsqfit_cuda_qr_combine_device")

    def solve_host(self, a_ptr: int, b_ptr: int, dim: int, x_ptr: int) -> int:
        dp = C.POINTER(C.c_double)
        st = self._lib.lsqfit_cuda_solve_host(self.h, C.cast(C.c_void_p(a_ptr), dp), C.cast(C.c_void_p(b_ptr), dp),
                                              dim, C.cast(C.c_void_p(x_ptr), dp))
        return self.check(st, "lsqfit_cuda_solve_host")

    # ---- device-resident path (pointers are CUDA device addresses) ----------
    def fit_device(self, d_xy: int, n: int, degree: int, flags: int, d_result: int, stream: int = 0) -> int:
        st = self._lib.lsqfit_cuda_fit_device(self.h, d_xy, n, degree, flags, d_result, stream)
        return self.check(st, "lsqfit_cuda_fit_device")

    def diagnostics_device(self, d_xy: int, n: int, degree: int, d_coeffs: int, d_gate: int,
                           d_residuals: int, d_out: int, stream: int = 0, shift: float = float("nan")) -> int:
        st = self._lib.lsqfit_cuda_diagnostics_device(self.h, d_xy, n, degree, d_coeffs, d_gate or None, shift,
                                                      d_residuals or None, d_out, stream)
        return self.check(st, "lsqfit_cuda_diagnostics_device")

    def combine_device(self, d_parts: int, n_parts: int, degree: int, flags: int, d_result: int,
                       stream: int = 0) -> int:
        st = self._lib.lsqfit_cuda_combine_device(self.h, d_parts, n_parts, degree, flags, d_result, stream)
        return self.check(st, "lsqfit_cuda_combine_device")

    def fit_batched_device(self, d_xy: int, n_curves: int, ppc: int, degree: int, d_coeffs: int,
                           d_status: int, stream: int = 0) -> int:
        st = self._lib.lsqfit_cuda_fit_batched_device(self.h, d_xy, n_curves, ppc, degree, d_coeffs, d_status,
                                                      stream)
        return self.check(st, "lsqfit_cuda_fit_batched_device")

    def synth_device(self, d_xy: int, n: int, offset: int, seed: int, truth_degree: int, sigma: float,
                     stream: int = 0) -> int:
        st = self._lib.lsqfit_cuda_synth_device(self.h, d_xy, n, offset, seed, truth_degree, sigma, stream)
        return self.check(st, "lsqfit_cuda_synth_device")

    def synth_batched_device(self, d_xy: int, n_curves: int, ppc: int, seed: int, truth_degree: int,
                             sigma: float, stream: int = 0) -> int:
        st = self._lib.lsqfit_cuda_synth_batched_device(self.h, d_xy, n_curves, ppc, seed, truth_degree, sigma,
                                                        stream)
        return self.check(st, "lsqfit_cuda_synth_batched_device")


class Group:
    """``lsqfit_cuda_group``: one host dataset sharded over several devices."""

    def __init__(self, devices):
        self._lib = lib()
        arr = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        st = self._lib.lsqfit_cuda_group_create(C.byref(h), arr, len(devices))
        if st != OK:
            raise CudaError(f"lsqfit_cuda_group_create({list(devices)}) failed: {STATUS_NAMES.get(st, st)}")
        self.h = h
        self.devices = list(devices)

    def close(self) -> None:
        if getattr(self, "h", None):
            self._lib.lsqfit_cuda_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def fit_host(self, xy_ptr: int, n: int, degree: int, flags: int) -> tuple[int, Result]:
        r = Result()
        st = self._lib.lsqfit_cuda_group_fit_host(self.h, C.cast(C.c_void_p(xy_ptr), C.POINTER(C.c_double)), n,
                                                  degree, flags, C.byref(r))
        if st in (ECUDA, ENOMEM):
            raise CudaError(f"lsqfit_cuda_group_fit_host: {STATUS_NAMES[st]}")
        return st, r

    def fit_device(self, shard_ptrs, shard_counts, degree: int, flags: int) -> tuple[int, Result]:
        """Device-resident shards (shard d on the group's device d): fused sums per
        device, records peer-copied to device 0, ordered combine (+ solve)."""
        G = len(self.devices)
        ptrs = (C.c_void_p * G)(*shard_ptrs)
        counts = (C.c_uint64 * G)(*shard_counts)
        r = Result()
        st = self._lib.lsqfit_cuda_group_fit_device(self.h, ptrs, counts, degree, flags, C.byref(r))
        if st in (ECUDA, ENOMEM):
            raise CudaError(f"lsqfit_cuda_group_fit_device: {STATUS_NAMES[st]}")
        return st, r


_contexts: dict[int, Context] = {}


def context(device: int = 0) -> Context:
    """Process-wide context per device (created on first use)."""
    with _lock:
        ctx = _contexts.get(device)
        if ctx is None:
            ctx = _contexts[device] = Context(device)
        return ctx

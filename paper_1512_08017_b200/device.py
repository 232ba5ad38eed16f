"""Device-resident helpers over the C ABI, with PyTorch as the allocator and
stream provider (plumbing only: every kernel is ours, in lib/liblsqfit_cuda.so).

Tensors holding points are float64 of shape (n, 2) (AoS, the memory image of
``std::vector<lsqfit::Point>``); results are the raw ``lsqfit_result`` /
``lsqfit_diag`` records in uint8 tensors.
"""
from __future__ import annotations

import torch

from . import _capi


def _stream(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _dev_index(t: torch.Tensor) -> int:
    return t.device.index if t.device.index is not None else torch.cuda.current_device()


def ctx_for(t: torch.Tensor) -> _capi.Context:
    return _capi.context(_dev_index(t))


def empty_result(device, count: int = 1) -> torch.Tensor:
    return torch.zeros(count * _capi.RESULT_BYTES, dtype=torch.uint8, device=device)


def empty_diag(device) -> torch.Tensor:
    return torch.zeros(_capi.DIAG_BYTES, dtype=torch.uint8, device=device)


def read_result(t: torch.Tensor, index: int = 0) -> _capi.Result:
    host = t.detach().to("cpu").numpy()
    off = index * _capi.RESULT_BYTES
    return _capi.Result.from_buffer_copy(host[off: off + _capi.RESULT_BYTES].tobytes())


def read_diag(t: torch.Tensor) -> _capi.Diag:
    return _capi.Diag.from_buffer_copy(t.detach().to("cpu").numpy().tobytes())


def result_field_ptr(t: torch.Tensor, name: str, index: int = 0) -> int:
    return t.data_ptr() + index * _capi.RESULT_BYTES + getattr(_capi.Result, name).offset


def synth(n: int, offset: int, seed: int, truth_degree: int, sigma: float, device="cuda") -> torch.Tensor:
    xy = torch.empty((n, 2), dtype=torch.float64, device=device)
    if n:
        ctx_for(xy).synth_device(xy.data_ptr(), n, offset, seed, truth_degree, sigma, _stream(xy.device))
    return xy


def synth_batched(n_curves: int, ppc: int, seed: int, truth_degree: int, sigma: float,
                  device="cuda") -> torch.Tensor:
    xy = torch.empty((n_curves * ppc, 2), dtype=torch.float64, device=device)
    ctx_for(xy).synth_batched_device(xy.data_ptr(), n_curves, ppc, seed, truth_degree, sigma,
                                     _stream(xy.device))
    return xy


def _check_points(xy: torch.Tensor) -> None:
    if not xy.is_cuda or xy.dtype != torch.float64 or not xy.is_contiguous():
        raise ValueError("points must be a contiguous float64 CUDA tensor of shape (n, 2)")
    if xy.numel() % 2:
        raise ValueError("points must have shape (n, 2)")


def fit(xy: torch.Tensor, degree: int, flags: int = _capi.SOLVE, out: torch.Tensor | None = None) -> torch.Tensor:
    """Launch the fused power-sums (+ solve) kernel on the current stream."""
    _check_points(xy)
    out = empty_result(xy.device) if out is None else out
    st = ctx_for(xy).fit_device(xy.data_ptr(), xy.numel() // 2, degree, flags, out.data_ptr(),
                                _stream(xy.device))
    if st != _capi.OK:
        raise ValueError(f"lsqfit_cuda_fit_device: {_capi.STATUS_NAMES.get(st, st)}")
    return out


def fit_ordered(xy: torch.Tensor, degree: int, chunks: int, flags: int = _capi.SOLVE,
                out: torch.Tensor | None = None) -> torch.Tensor:
    """Reference-order sums (bit-identical to accumulate_parallel(d, m, chunks))."""
    _check_points(xy)
    out = empty_result(xy.device) if out is None else out
    st = ctx_for(xy).fit_ordered_device(xy.data_ptr(), xy.numel() // 2, degree, chunks, flags, out.data_ptr(),
                                        _stream(xy.device))
    if st != _capi.OK:
        raise ValueError(f"lsqfit_cuda_fit_ordered_device: {_capi.STATUS_NAMES.get(st, st)}")
    return out


def combine(parts: torch.Tensor, n_parts: int, degree: int, flags: int = _capi.SOLVE,
            out: torch.Tensor | None = None) -> torch.Tensor:
    out = empty_result(parts.device) if out is None else out
    st = ctx_for(parts).combine_device(parts.data_ptr(), n_parts, degree, flags, out.data_ptr(),
                                       _stream(parts.device))
    if st != _capi.OK:
        raise ValueError(f"lsqfit_cuda_combine_device: {_capi.STATUS_NAMES.get(st, st)}")
    return out


def diagnostics(xy: torch.Tensor, degree: int, fit_result: torch.Tensor, residuals: torch.Tensor | None = None,
                out: torch.Tensor | None = None, shift: float = float("nan")) -> torch.Tensor:
    """FitReport pass (residuals, SSE, SST, R) of device-resident points against
    ``fit_result``'s coefficients. ``shift`` is the centring constant of the SST
    moments (NaN: this array's first y); records that are to be combined must
    share it."""
    _check_points(xy)
    out = empty_diag(xy.device) if out is None else out
    st = ctx_for(xy).diagnostics_device(xy.data_ptr(), xy.numel() // 2, degree,
                                        result_field_ptr(fit_result, "coeffs"),
                                        result_field_ptr(fit_result, "status"),
                                        residuals.data_ptr() if residuals is not None else 0,
                                        out.data_ptr(), _stream(xy.device), shift)
    if st != _capi.OK:
        raise ValueError(f"lsqfit_cuda_diagnostics_device: {_capi.STATUS_NAMES.get(st, st)}")
    return out


def fit_batched_ragged(xy: torch.Tensor, offsets: torch.Tensor, degree: int,
                       coeffs: torch.Tensor | None = None, status: torch.Tensor | None = None):
    """Ragged batch: curve c = points [offsets[c], offsets[c+1]) of ``xy``
    (``offsets``: int64 CUDA tensor of n_curves + 1 non-decreasing values)."""
    _check_points(xy)
    if offsets.dtype != torch.int64 or not offsets.is_cuda or offsets.dim() != 1 or offsets.numel() < 1:
        raise ValueError("offsets must be a 1-D int64 CUDA tensor of n_curves + 1 values")
    n_curves = offsets.numel() - 1
    total = int(offsets[-1].item() - offsets[0].item()) if n_curves else 0
    coeffs = torch.empty((n_curves, degree + 1), dtype=torch.float64, device=xy.device) if coeffs is None else coeffs
    status = torch.empty(n_curves, dtype=torch.int32, device=xy.device) if status is None else status
    ctx = ctx_for(xy)
    st = ctx.check(ctx._lib.lsqfit_cuda_fit_batched_ragged_device(ctx.h, xy.data_ptr(), offsets.data_ptr(), n_curves,
                                                                  total, degree, coeffs.data_ptr(), status.data_ptr(),
                                                                  _stream(xy.device)),
                   "lsqfit_cuda_fit_batched_ragged_device")
    if st != _capi.OK:
        raise ValueError(f"lsqfit_cuda_fit_batched_ragged_device: {_capi.STATUS_NAMES.get(st, st)}")
    return coeffs, status


def empty_qr_result(device, count: int = 1) -> torch.Tensor:
    return torch.zeros(count * _capi.QR_BYTES, dtype=torch.uint8, device=device)


def read_qr_result(t: torch.Tensor, index: int = 0) -> _capi.QrResult:
    host = t.detach().to("cpu").numpy()
    off = index * _capi.QR_BYTES
    return _capi.QrResult.from_buffer_copy(host[off: off + _capi.QR_BYTES].tobytes())


def qr_fit(xy: torch.Tensor, degree: int, flags: int = _capi.SOLVE, out: torch.Tensor | None = None) -> torch.Tensor:
    """TSQR cross-check fit of device-resident points (current stream)."""
    _check_points(xy)
    out = empty_qr_result(xy.device) if out is None else out
    st = ctx_for(xy).qr_fit_device(xy.data_ptr(), xy.numel() // 2, degree, flags, out.data_ptr(),
                                   _stream(xy.device))
    if st != _capi.OK:
        raise ValueError(f"lsqfit_cuda_qr_fit_device: {_capi.STATUS_NAMES.get(st, st)}")
    return out


def qr_combine(parts: torch.Tensor, n_parts: int, degree: int, flags: int = _capi.SOLVE,
               out: torch.Tensor | None = None) -> torch.Tensor:
    out = empty_qr_result(parts.device) if out is None else out
    st = ctx_for(parts).qr_combine_device(parts.data_ptr(), n_parts, degree, flags, out.data_ptr(),
                                          _stream(parts.device))
    if st != _capi.OK:
        raise ValueError(f"lsqfit_cuda_qr_combine_device: {_capi.STATUS_NAMES.get(st, st)}")
    return out


def fit_batched(xy: torch.Tensor, n_curves: int, ppc: int, degree: int,
                coeffs: torch.Tensor | None = None, status: torch.Tensor | None = None):
    _check_points(xy)
    if xy.numel() // 2 < n_curves * ppc:
        raise ValueError("points tensor is smaller than n_curves * points_per_curve")
    coeffs = torch.empty((n_curves, degree + 1), dtype=torch.float64, device=xy.device) if coeffs is None else coeffs
    status = torch.empty(n_curves, dtype=torch.int32, device=xy.device) if status is None else status
    st = ctx_for(xy).fit_batched_device(xy.data_ptr(), n_curves, ppc, degree, coeffs.data_ptr(),
                                        status.data_ptr(), _stream(xy.device))
    if st != _capi.OK:
        raise ValueError(f"lsqfit_cuda_fit_batched_device: {_capi.STATUS_NAMES.get(st, st)}")
    return coeffs, status

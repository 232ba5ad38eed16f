// lsqfit/cuda.hpp — B200 extensions of the lsqfit C++ API that have no
// reference counterpart: device selection and the batched many-curve fit.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "lsqfit/dataset.hpp"
#include "lsqfit/diagnostics.hpp"

namespace lsqfit::cuda {

// CUDA device used by subsequent lsqfit calls in this process (default: 0, or
// the LSQFIT_CUDA_DEVICE environment variable).
void set_device(int device);

// Shard every subsequent host-dataset fit (accumulate*, fit_normal) over
// these devices: each GPU streams its contiguous slice over its own PCIe
// link, partial records combine in device order. One entry = set_device.
void set_devices(const std::vector<int>& devices);

// Reference-order mode (default off): accumulate / accumulate_parallel /
// fit_normal reproduce the reference's power sums — and hence, through the
// bit-identical device solve, its coefficients — exactly: one GPU thread per
// reference chunk replays accumulate_into, then the ascending combine. Fast
// for many chunks (~1e4+); exact but slow for few (accumulate is one chain).
void set_reference_order(bool enabled);

/// Free the default context's grow-only device and pinned buffers (a large
/// fit keeps its device copy for reuse); they are re-allocated on demand.
void release_buffers();

// Many independent fits in one launch: curve c owns
// points[c * points_per_curve, (c + 1) * points_per_curve). Per curve the
// semantics are accumulate -> build_normal_system -> solve_gaussian;
// status[c] is 0 (ok), 2 (overflow) or 3 (singular) — no exception per curve.
struct BatchedFit {
    int degree = 0;
    std::vector<double> coeffs;   // n_curves * (degree + 1), curve-major
    std::vector<std::int32_t> status;
};
BatchedFit fit_batched(const std::vector<Point>& points, std::size_t n_curves, std::uint32_t points_per_curve,
                       int degree);
/// Curves of different lengths: curve c = points[offsets[c], offsets[c+1])
/// (offsets.size() = n_curves + 1, non-decreasing; empty curves -> status 3).
BatchedFit fit_batched_ragged(const std::vector<Point>& points, const std::vector<std::uint64_t>& offsets,
                              int degree);

// The QR cross-check fit (the role of the reference's fit_qr,
// qr_backend.cpp:126-133) computed on the GPU by TSQR (Givens factors merged
// in a fixed tree): backend HouseholderQR in the report, RankDeficientError /
// OverflowError / DegreeTooHighError like the reference; any degree <= 12.
FitReport fit_qr_tsqr(const Dataset& dataset, int degree);

}  // namespace lsqfit::cuda

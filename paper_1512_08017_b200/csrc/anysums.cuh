// anysums.cuh — power sums for any degree (no template cap).
//
// The reference's accumulate / accumulate_parallel accept every degree >= 0
// (power_sums.cpp:39-90); the fused kernels are instantiated up to
// LSQFIT_MAX_DEGREE (the cap of fit_normal, diagnostics.hpp:13). Beyond it
// this generic path keeps the drop-in complete: one column of sums per
// blockIdx.y (s[k], k = 1..2m, then t[j], j = 0..m), each point's term formed
// with the reference's exact operation chain (power *= x repeated, then
// power * y; power_sums.cpp:20-24 — O(k) multiplies per term, which is what
// the reference's single loop also spends), per-thread compensated
// (Fast2Sum) accumulation, a fixed-order block reduction into one
// double-double partial per (chunk, block, column), and a final kernel that
// folds the partials in a fixed order and applies require_finite
// (power_sums.cpp:28-35). Deterministic for a given (n, degree, grid).
#pragma once

#include "common.cuh"

namespace lsq {

constexpr int kAnyThreads = 256;

// Term of column c for point (x, y): c < 2m -> x^(c+1); else y * x^(c-2m).
__device__ __forceinline__ double any_term(int m, int c, double x, double y) {
    const int k = c < 2 * m ? c + 1 : c - 2 * m;  // power of x
    double p = 1.0;
    if (k >= 1) {
        p = x;  // power = 1.0 * x == x exactly
        for (int i = 1; i < k; ++i) p = __dmul_rn(p, x);
    }
    if (c < 2 * m) return p;
    return k == 0 ? y : __dmul_rn(p, y);  // t[0]: 1.0 * y == y
}

// grid (B, 3m+1): block b of column c sums points [n*b/B, n*(b+1)/B) of this
// chunk into parts[(c * B + b)] as (hi, lo).
__global__ void __launch_bounds__(kAnyThreads) anysums_partial_kernel(const double2* __restrict__ xy, uint64_t n,
                                                                     int m, double2* __restrict__ parts) {
    const int c = blockIdx.y;
    const uint64_t B = gridDim.x, b = blockIdx.x;
    const uint64_t lo_i = n * b / B, hi_i = n * (b + 1) / B;
    double hi = 0.0, lo = 0.0;
    for (uint64_t i = lo_i + threadIdx.x; i < hi_i; i += kAnyThreads) {
        const double2 p = __ldg(xy + i);
        fold_sorted(hi, lo, any_term(m, c, p.x, p.y));
    }
    __shared__ double s_hi[kAnyThreads / 32], s_lo[kAnyThreads / 32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    warp_reduce_dd_down(hi, lo);
    if (lane == 0) {
        s_hi[warp] = hi;
        s_lo[warp] = lo;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double h = s_hi[0], l = s_lo[0];
        for (int w = 1; w < kAnyThreads / 32; ++w) dd_add(h, l, s_hi[w], s_lo[w]);
        parts[size_t(c) * B + b] = make_double2(h, l);
    }
}

// One thread per column: fold the `count` partials of every column in order
// (chunk-major), then s[0] = n and require_finite. out: s[0..2m], t[0..m],
// then the status word (as a double).
__global__ void anysums_final_kernel(const double2* __restrict__ parts, int chunks, uint64_t B, int m, uint64_t n,
                                     double* __restrict__ out, int* __restrict__ status) {
    const int nc = 3 * m + 1;
    __shared__ int s_bad;
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    for (int c = threadIdx.x; c < nc; c += blockDim.x) {
        double h = 0.0, l = 0.0;
        for (int k = 0; k < chunks; ++k)
            for (uint64_t b = 0; b < B; ++b) {
                const double2 v = parts[(size_t(k) * nc + c) * B + b];
                dd_add(h, l, v.x, v.y);
            }
        const double val = __dadd_rn(h, l);
        if (!isfinite(val)) atomicOr(&s_bad, 1);
        if (c < 2 * m) out[c + 1] = val;             // s[c+1]
        else out[(2 * m + 1) + (c - 2 * m)] = val;   // t[c-2m]
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        out[0] = static_cast<double>(n);  // s[0] counts points exactly
        *status = s_bad ? LSQFIT_EOVERFLOW : LSQFIT_OK;
    }
}

}  // namespace lsq

namespace lsq {

// Reference order at any degree (bit-identical to accumulate_parallel(d, m,
// chunks), power_sums.cpp:52-90): thread (chunk q, column c) replays column
// c's chain over chunk q in point order — s[k] += x^k with x^k formed by the
// reference's repeated multiplication, t[j] += x^j * y — one plain rounded
// add per point, exactly the reference's sequence for that accumulator.
// s[0] counts the chunk's points (exact). slots[q * (3m+2) + v], v over
// s[0..2m] then t[0..m] (the reference's partial layout).
__global__ void __launch_bounds__(128) ordered_any_kernel(const double2* __restrict__ xy, uint64_t n,
                                                          uint64_t chunks, int m, double* __restrict__ slots) {
    const int nc = 3 * m + 1;  // non-trivial columns
    const uint64_t total = chunks * uint64_t(nc);
    for (uint64_t id = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; id < total;
         id += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t q = id / nc;
        const int c = static_cast<int>(id % nc);
        const uint64_t lo = n * q / chunks, hi = n * (q + 1) / chunks;  // power_sums.cpp:69-70
        double acc = 0.0;
        for (uint64_t i = lo; i < hi; ++i) {
            const double2 p = __ldg(xy + i);
            acc = __dadd_rn(acc, any_term(m, c, p.x, p.y));
        }
        double* slot = slots + q * uint64_t(nc + 1);
        if (c < 2 * m) slot[c + 1] = acc;              // s[c+1]
        else slot[(2 * m + 1) + (c - 2 * m)] = acc;    // t[c-2m]
        if (c == 0) slot[0] = static_cast<double>(hi - lo);
    }
}

// The ascending element-wise combine (power_sums.cpp:80-87): sums = slot 0,
// then + slot 1, + slot 2 ...; require_finite. out: s[0..2m], t[0..m].
__global__ void ordered_any_combine_kernel(const double* __restrict__ slots, uint64_t chunks, int m,
                                           double* __restrict__ out, int* __restrict__ status) {
    const int stride = 3 * m + 2;
    __shared__ int s_bad;
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    for (int v = threadIdx.x; v < stride; v += blockDim.x) {
        double acc = slots[v];
        for (uint64_t q = 1; q < chunks; ++q) acc = __dadd_rn(acc, slots[q * stride + v]);
        out[v] = acc;
        if (!isfinite(acc)) atomicOr(&s_bad, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) *status = s_bad ? LSQFIT_EOVERFLOW : LSQFIT_OK;
}

}  // namespace lsq

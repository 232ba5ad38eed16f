// ordered.cuh — reference-order power sums: bit-identical to the reference's
// accumulate_parallel(dataset, degree, chunks) (proj/src/power_sums.cpp:52-90).
//
// The reference's result is a pure function of (data, degree, chunks): chunk
// c = [n*c/C, n*(c+1)/C) is summed sequentially with accumulate_into's exact
// operation sequence (power = 1; s[k] += power; t[k] += power*y; power *= x;
// power_sums.cpp:13-26), and the C partial vectors are added element-wise in
// ascending chunk order (:80-87). Every chunk is independent, so on the GPU
// each thread replays one chunk's sequential chain (explicitly rounded
// binary64, no FMA contraction — the x86-64 SSE2 arithmetic of the reference
// build), and one thread per sum replays the ascending combine. With tens of
// thousands of chunks this is parallel enough to stream near HBM speed while
// reproducing the reference's bits exactly; with few chunks it is exact but
// slow (a chunk is a dependency chain). chunks == 1 is accumulate() itself.
#pragma once

#include "common.cuh"
#include "power_sums.cuh"

namespace lsq {

constexpr int kOrderedThreads = 128;

// One thread per chunk: accumulate_into over the chunk, written as the
// reference's per-chunk slot (s[0..2M], t[0..M]).
template <int M>
__global__ void __launch_bounds__(kOrderedThreads) ordered_chunks_kernel(const double2* __restrict__ xy, uint64_t n,
                                                                        uint64_t chunks, double* __restrict__ slots) {
    constexpr int NSL = 2 * M + 1, NTL = M + 1, STRIDE = NSL + NTL;
    for (uint64_t c = uint64_t(blockIdx.x) * kOrderedThreads + threadIdx.x; c < chunks;
         c += uint64_t(gridDim.x) * kOrderedThreads) {
        const uint64_t lo = n * c / chunks, hi = n * (c + 1) / chunks;  // power_sums.cpp:69-70
        double s[NSL], t[NTL];
#pragma unroll
        for (int k = 0; k < NSL; ++k) s[k] = 0.0;
#pragma unroll
        for (int j = 0; j < NTL; ++j) t[j] = 0.0;
        // The chain is sequential per thread, so memory parallelism comes from
        // loading a batch of points ahead of processing them in order.
        constexpr int B = 16;
        uint64_t i = lo;
        for (; i + B <= hi; i += B) {
            double2 p[B];
#pragma unroll
            for (int q = 0; q < B; ++q) p[q] = __ldg(xy + i + q);
#pragma unroll
            for (int q = 0; q < B; ++q) {
                double power = 1.0;
#pragma unroll
                for (int k = 0; k < NSL; ++k) {
                    s[k] = __dadd_rn(s[k], power);
                    if (k <= M) t[k] = __dadd_rn(t[k], __dmul_rn(power, p[q].y));
                    power = __dmul_rn(power, p[q].x);
                }
            }
        }
        for (; i < hi; ++i) {
            const double2 p = __ldg(xy + i);
            double power = 1.0;
#pragma unroll
            for (int k = 0; k < NSL; ++k) {
                s[k] = __dadd_rn(s[k], power);
                if (k <= M) t[k] = __dadd_rn(t[k], __dmul_rn(power, p.y));
                power = __dmul_rn(power, p.x);
            }
        }
        double* slot = slots + c * STRIDE;
#pragma unroll
        for (int k = 0; k < NSL; ++k) slot[k] = s[k];
#pragma unroll
        for (int j = 0; j < NTL; ++j) slot[NSL + j] = t[j];
    }
}

// The ascending element-wise combine (power_sums.cpp:80-87), one thread per
// sum (the order is the reference's: slot 0, then + slot 1, + slot 2, ...),
// fed from blocks of slots staged through shared memory by the whole CTA;
// then require_finite and (SOLVE) the one-warp solve. One CTA.
constexpr int kOrderedCombineThreads = 256;
constexpr int kOrderedRows = 64;

template <int M>
__global__ void __launch_bounds__(kOrderedCombineThreads) ordered_combine_kernel(const double* __restrict__ slots,
                                                                                uint64_t chunks, uint64_t n,
                                                                                unsigned flags, lsqfit_result* out) {
    constexpr int NSL = 2 * M + 1, NTL = M + 1, STRIDE = NSL + NTL, DIM = M + 1;
    __shared__ double s_rows[kOrderedRows * STRIDE];
    __shared__ double s_sum[STRIDE];
    __shared__ double s_scratch[DIM * DIM + 2 * DIM + 8];
    __shared__ int s_bad;
    const int tid = threadIdx.x;
    if (tid == 0) s_bad = 0;
    double acc = 0.0;
    for (uint64_t c0 = 0; c0 < chunks; c0 += kOrderedRows) {
        const int rows = static_cast<int>((chunks - c0 < kOrderedRows) ? (chunks - c0) : kOrderedRows);
        for (int i = tid; i < rows * STRIDE; i += kOrderedCombineThreads) s_rows[i] = __ldg(slots + c0 * STRIDE + i);
        __syncthreads();
        if (tid < STRIDE) {
            int r = 0;
            if (c0 == 0) acc = s_rows[tid], r = 1;  // sums = partials[0]
#pragma unroll 16
            for (; r < rows; ++r) acc = __dadd_rn(acc, s_rows[r * STRIDE + tid]);
        }
        __syncthreads();
    }
    if (tid < STRIDE) {
        s_sum[tid] = acc;
        if (!isfinite(acc)) atomicOr(&s_bad, 1);  // require_finite, power_sums.cpp:28-35
    }
    __syncthreads();
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    for (int k = lane; k < NSL; k += 32) out->s[k] = s_sum[k];
    for (int j = lane; j < NTL; j += 32) out->t[j] = s_sum[NSL + j];
    for (int v = lane; v < 3 * M + 1; v += 32) {  // the same sums as (hi, lo = 0) records
        out->part_hi[v] = v < 2 * M ? s_sum[v + 1] : s_sum[NSL + v - 2 * M];
        out->part_lo[v] = 0.0;
    }
    if (lane == 0) {
        out->n = n;
        out->degree = M;
    }
    int status = s_bad ? LSQFIT_EOVERFLOW : LSQFIT_OK;
    if (status == LSQFIT_OK && (flags & LSQFIT_SOLVE)) {
        double* A = s_scratch;
        double* b = A + DIM * DIM;
        double* x = b + DIM;
        warp_build_normal_system(s_sum, s_sum + NSL, M, A, b);
        status = warp_solve_gaussian(A, b, x, DIM);
        if (status == LSQFIT_OK)
            for (int k = lane; k < DIM; k += 32) out->coeffs[k] = x[k];
    }
    if (lane == 0) out->status = status;
}

}  // namespace lsq

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

// One WARP per chunk (long chunks; k_ordered.cu picks it from ~3k points per
// chunk, where it measured faster than a thread per chunk): the chain
// only fixes the order of the additions into each accumulator, not where the
// terms are formed. Lanes form the terms of 32 consecutive points in parallel
// (coalesced loads; the reference's operation sequence power = 1; t[0] term
// 1*y = y; power = x; s[k] term = power; t[k] term = power*y; power *= x),
// stage them in shared memory (odd row stride: conflict-free), and lane v then
// adds column v's 32 terms in point order — the reference's sequential chain,
// bit for bit, now one dependent add per point per column instead of the whole
// per-point operation sequence. s[0] is the exact point count (the reference
// adds 1.0 once per point: exact below 2^53).
// Warps per CTA (a 32-row term buffer per warp).
template <int M>
struct OrderedWarpCfg {
    static constexpr int NV = 3 * M + 1;  // columns: s[1..2M] -> 0..2M-1, t[0..M] -> 2M..3M
    static constexpr int R = NV | 1;      // odd row stride: conflict-free
#ifndef LSQ_ORDERED_GROUP
#define LSQ_ORDERED_GROUP 128  // A/B: 32 -> 64 -> 128 points per group, C = 1..128: 1.5x faster (fewer barriers per add)
#endif
    static constexpr int GROUP = LSQ_ORDERED_GROUP;  // points per staged group (32 or 64)
    static constexpr int FIT = (48 * 1024) / (GROUP * R * 8);  // warps whose staging fits 48 KB
    static constexpr int WARPS = FIT >= 4 ? 4 : (FIT >= 2 ? 2 : 1);
    static constexpr int THREADS = WARPS * 32;
};

template <int M>
__global__ void __launch_bounds__(OrderedWarpCfg<M>::THREADS) ordered_warp_kernel(const double2* __restrict__ xy,
                                                                                 uint64_t n, uint64_t chunks,
                                                                                 double* __restrict__ slots) {
    using C = OrderedWarpCfg<M>;
    constexpr int NSL = 2 * M + 1, NTL = M + 1, STRIDE = NSL + NTL;
    constexpr int NV = C::NV, R = C::R, WARPS = C::WARPS, GROUP = C::GROUP, SUB = GROUP / 32;
    __shared__ double terms[WARPS][GROUP * R];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* T = terms[warp];
    // PF batches of 32 points in flight per lane (register ring, static indices);
    // SUB consecutive batches form one staged group
    constexpr int PF = 8;
    static_assert(PF % SUB == 0, "groups tile the ring");
    for (uint64_t c = uint64_t(blockIdx.x) * WARPS + warp; c < chunks; c += uint64_t(gridDim.x) * WARPS) {
        const uint64_t lo = n * c / chunks, hi = n * (c + 1) / chunks;  // power_sums.cpp:69-70
        double acc0 = 0.0, acc1 = 0.0;  // this lane's columns: lane, lane + 32
        double2 p[PF];
#pragma unroll
        for (int i = 0; i < PF; ++i) {
            const uint64_t gi = lo + uint64_t(i) * 32 + lane;
            p[i] = (gi < hi) ? __ldg(xy + gi) : make_double2(0.0, 0.0);
        }
        for (uint64_t g0 = lo; g0 < hi; g0 += uint64_t(PF) * 32) {
#pragma unroll
            for (int i = 0; i < PF; i += SUB) {
                const uint64_t g = g0 + uint64_t(i) * 32;
                if (g >= hi) break;  // warp-uniform
                const int cnt = (hi - g < uint64_t(GROUP)) ? static_cast<int>(hi - g) : GROUP;
#pragma unroll
                for (int sb = 0; sb < SUB; ++sb) {
                    double* row = T + (sb * 32 + lane) * R;
                    const double2 pt = p[i + sb];
                    row[2 * M] = pt.y;  // t[0] += power * y with power == 1.0: exactly y
                    double pw = pt.x;   // power = 1.0 * x == x exactly
#pragma unroll
                    for (int k = 1; k <= 2 * M; ++k) {
                        row[k - 1] = pw;                                   // s[k] += power
                        if (k <= M) row[2 * M + k] = __dmul_rn(pw, pt.y);  // t[k] += power * y
                        if (k < 2 * M) pw = __dmul_rn(pw, pt.x);           // power *= x
                    }
                    // refill this slot with the batch PF ahead (in flight during the adds)
                    const uint64_t gn = g + uint64_t(sb) * 32 + uint64_t(PF) * 32 + lane;
                    p[i + sb] = (gn < hi) ? __ldg(xy + gn) : make_double2(0.0, 0.0);
                }
                __syncwarp();
                if (cnt == GROUP) {
                    if (lane < NV) {
#pragma unroll
                        for (int q = 0; q < GROUP; ++q) acc0 = __dadd_rn(acc0, T[q * R + lane]);
                    }
                    if (lane + 32 < NV) {
#pragma unroll
                        for (int q = 0; q < GROUP; ++q) acc1 = __dadd_rn(acc1, T[q * R + lane + 32]);
                    }
                } else {
                    if (lane < NV)
                        for (int q = 0; q < cnt; ++q) acc0 = __dadd_rn(acc0, T[q * R + lane]);
                    if (lane + 32 < NV)
                        for (int q = 0; q < cnt; ++q) acc1 = __dadd_rn(acc1, T[q * R + lane + 32]);
                }
                __syncwarp();
            }
        }
        double* slot = slots + c * STRIDE;
        if (lane == 0) slot[0] = static_cast<double>(hi - lo);
        if (lane < NV) slot[lane < 2 * M ? lane + 1 : NSL + (lane - 2 * M)] = acc0;
        if (lane + 32 < NV) slot[NSL + (lane + 32 - 2 * M)] = acc1;
    }
}

// One THREAD per chunk, rows staged by cp.async (many chunks): a warp owns
// 32 consecutive chunks, one per lane. Each round stages the next K = 16
// points of every one of its chunks into a shared-memory tile — two 256-byte
// rows per warp copy instruction, 16 bytes per lane, cp.async (no register
// staging) — into a STAGES-deep ring per warp, so several rounds are in
// flight while lane j replays accumulate_into over its row (the reference's
// exact per-point operation sequence, power_sums.cpp:18-25, explicitly
// rounded, in point order). Row stride K + 1 points: conflict-free reads.
constexpr int kRowK = 16;
constexpr int kRowStride = kRowK + 1;
#ifndef LSQ_ROW_STAGES
#define LSQ_ROW_STAGES 3  // A/B: 3 >= 4 (more CTAs resident; 32k chunks m = 8, 12: 21-26% faster)
#endif
constexpr int kRowStages = LSQ_ROW_STAGES;
constexpr int kRowWarps = 2;
constexpr size_t kRowTileBytes = size_t(32) * kRowStride * 16;  // one round of one warp
constexpr size_t kRowSmemBytes = kRowTileBytes * kRowStages * kRowWarps;

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(smem_dst)), "l"(gmem_src),
                 "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int M>
__global__ void __launch_bounds__(kRowWarps * 32) ordered_rows_kernel(const double2* __restrict__ xy, uint64_t n,
                                                                     uint64_t chunks, double* __restrict__ slots) {
    constexpr int NSL = 2 * M + 1, NTL = M + 1, STRIDE = NSL + NTL;
    extern __shared__ __align__(16) unsigned char rows_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double2* ring = reinterpret_cast<double2*>(rows_smem) + size_t(warp) * kRowStages * 32 * kRowStride;
    const int half = lane >> 4, col = lane & 15;  // copy role: row (2q + half), point col
    for (uint64_t cb = (uint64_t(blockIdx.x) * kRowWarps + warp) * 32; cb < chunks;
         cb += uint64_t(gridDim.x) * kRowWarps * 32) {
        const uint64_t c = cb + lane;
        const uint64_t lo = c < chunks ? n * c / chunks : n;  // power_sums.cpp:69-70
        const uint64_t hi = c < chunks ? n * (c + 1) / chunks : n;
        const uint64_t len = hi - lo;
        uint64_t maxlen = len;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            const uint64_t o = __shfl_xor_sync(0xffffffffu, maxlen, off);
            maxlen = o > maxlen ? o : maxlen;
        }
        // the copy role's two rows per instruction pair: rows 2q + half
        uint64_t lo_r[16], hi_r[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            lo_r[q] = __shfl_sync(0xffffffffu, lo, 2 * q + half);
            hi_r[q] = __shfl_sync(0xffffffffu, hi, 2 * q + half);
        }
        const uint64_t rounds = (maxlen + kRowK - 1) / kRowK;
        auto issue = [&](uint64_t r) {
            double2* T = ring + (r % kRowStages) * 32 * kRowStride;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const uint64_t gi = lo_r[q] + r * kRowK + col;
                const bool valid = gi < hi_r[q];
                cp_async16(T + (2 * q + half) * kRowStride + col, xy + (valid ? gi : 0), valid);
            }
        };
        // prologue: STAGES - 1 rounds in flight (always commit, possibly empty)
#pragma unroll
        for (int r = 0; r < kRowStages - 1; ++r) {
            if (uint64_t(r) < rounds) issue(r);
            cp_async_commit();
        }
        double s[NSL], t[NTL];
#pragma unroll
        for (int k = 0; k < NSL; ++k) s[k] = 0.0;
#pragma unroll
        for (int j = 0; j < NTL; ++j) t[j] = 0.0;
        auto point = [&](const double2 pt) {
            // accumulate_into: power = 1; s[k] += power; t[k] += power * y; power *= x
            t[0] = __dadd_rn(t[0], pt.y);  // power == 1.0: the term is y exactly
            double pw = pt.x;              // 1.0 * x == x exactly
#pragma unroll
            for (int k = 1; k < NSL; ++k) {
                s[k] = __dadd_rn(s[k], pw);
                if (k <= M) t[k] = __dadd_rn(t[k], __dmul_rn(pw, pt.y));
                if (k + 1 < NSL) pw = __dmul_rn(pw, pt.x);
            }
        };
        for (uint64_t r = 0; r < rounds; ++r) {
            if (r + kRowStages - 1 < rounds) issue(r + kRowStages - 1);
            cp_async_commit();
            cp_async_wait<kRowStages - 1>();  // round r has landed (this lane's copies)
            __syncwarp();                     // ... and every lane's
            const double2* row = ring + (r % kRowStages) * 32 * kRowStride + lane * kRowStride;
            const uint64_t done = r * kRowK;
            const int cnt = len > done ? static_cast<int>(len - done < uint64_t(kRowK) ? len - done : kRowK) : 0;
            if (cnt == kRowK) {
#pragma unroll
                for (int q = 0; q < kRowK; ++q) point(row[q]);
            } else {
                for (int q = 0; q < cnt; ++q) point(row[q]);
            }
            __syncwarp();  // the stage is free for the copies issued next round
        }
        cp_async_wait<0>();
        __syncwarp();
        if (c < chunks) {
            double* slot = slots + c * STRIDE;
            slot[0] = static_cast<double>(len);  // s[0] += 1.0 per point: the exact count
#pragma unroll
            for (int k = 1; k < NSL; ++k) slot[k] = s[k];
#pragma unroll
            for (int j = 0; j < NTL; ++j) slot[NSL + j] = t[j];
        }
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
    // rows per block: as many as two ~20 KB buffers hold (fewer block barriers on the chain)
    constexpr int ROWS = ((2560 / STRIDE) / 16) * 16 > kOrderedRows ? ((2560 / STRIDE) / 16) * 16 : kOrderedRows;
    constexpr int BLOCK = ROWS * STRIDE;                                             // doubles per row block
    constexpr int PER = (BLOCK + kOrderedCombineThreads - 1) / kOrderedCombineThreads;  // per thread
    __shared__ double s_rows[2][BLOCK];  // double-buffered: block b+1 loads while block b is added
    __shared__ double s_sum[STRIDE];
    __shared__ double s_scratch[DIM * DIM + 2 * DIM + 8];
    __shared__ int s_bad;
    const int tid = threadIdx.x;
    if (tid == 0) s_bad = 0;
    auto rows_at = [&](uint64_t c0) { return static_cast<int>((chunks - c0 < ROWS) ? (chunks - c0) : ROWS); };
    {
        const int rows = rows_at(0);
        for (int i = tid; i < rows * STRIDE; i += kOrderedCombineThreads) s_rows[0][i] = __ldg(slots + i);
    }
    __syncthreads();
    double acc = 0.0;
    int buf = 0;
    for (uint64_t c0 = 0; c0 < chunks; c0 += ROWS) {
        const int rows = rows_at(c0);
        const uint64_t c1 = c0 + ROWS;
        const int next = c1 < chunks ? rows_at(c1) : 0;
        double pre[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int i = tid + j * kOrderedCombineThreads;
            pre[j] = (i < next * STRIDE) ? __ldg(slots + c1 * STRIDE + i) : 0.0;
        }
        if (tid < STRIDE) {
            const double* rw = s_rows[buf];
            int r = 0;
            if (c0 == 0) acc = rw[tid], r = 1;  // sums = partials[0]
#pragma unroll 16
            for (; r < rows; ++r) acc = __dadd_rn(acc, rw[r * STRIDE + tid]);
        }
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int i = tid + j * kOrderedCombineThreads;
            if (i < next * STRIDE) s_rows[buf ^ 1][i] = pre[j];
        }
        __syncthreads();
        buf ^= 1;
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
        status = warp_solve<DIM>(A, b, x);
        if (status == LSQFIT_OK)
            for (int k = lane; k < DIM; k += 32) out->coeffs[k] = x[k];
    }
    if (lane == 0) out->status = status;
}

}  // namespace lsq

// k_batched.cu — instantiates the one-warp-per-curve batched fit (batched.cuh).
#include "batched.cuh"
#include "internal.hpp"

namespace lsq_impl {

// Thread-per-curve up to this many points per curve: the measured crossover
// against the warp-per-curve kernel (2^30 points, tools/batched_sweep.py).
#ifdef LSQ_BATCH_SMALL_PPC
constexpr uint32_t small_ppc_max(int) { return LSQ_BATCH_SMALL_PPC; }
#else
constexpr uint32_t small_ppc_max(int m) { return m <= 1 ? 384u : m == 2 ? 512u : m == 3 ? 1024u : 2048u; }
#endif
#ifdef LSQ_BATCH_SMALL_PPC_HI
constexpr uint32_t small_ppc_max_hi(int) { return LSQ_BATCH_SMALL_PPC_HI; }
#else
constexpr uint32_t small_ppc_max_hi(int) { return 1024u; }
#endif
#ifndef LSQ_BATCH_SMALL_MAX_DEGREE
#define LSQ_BATCH_SMALL_MAX_DEGREE 6  // m = 4..6 solve through an L1-resident stack frame: still 4-23x the warp kernel
#endif


cudaError_t batched_configure(int m, int sm_count, int* ctas) {
    return dispatch_degree<0, LSQFIT_MAX_DEGREE>(m, [&](auto M) {
        constexpr int D = decltype(M)::value;
        if constexpr (D > LSQ_BATCH_SMALL_MAX_DEGREE) {  // shared-memory solve of the short-curve kernel
            constexpr int smem = static_cast<int>(lsq::small_solve_smem<D>());
            cudaError_t e = cudaFuncSetAttribute(lsq::batched_small_kernel<D, true, true>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(lsq::batched_small_kernel<D, false, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e != cudaSuccess) return e;
        }
        int per_sm = 0;
        const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, lsq::batched_fit_kernel<D, true>, lsq::kBatchThreads, 0);
        if (e != cudaSuccess) return e;
        *ctas = sm_count * (per_sm > 0 ? per_sm : 1);
        return cudaSuccess;
    });
}

cudaError_t batched_launch(lsqfit_cuda_ctx* ctx, int m, const double* d_xy, uint64_t n_curves, uint32_t ppc,
                           double* d_coeffs, int32_t* d_status, cudaStream_t st) {
    const cudaError_t ce = ensure_batched(ctx, m);
    if (ce != cudaSuccess) return ce;
    return dispatch_degree<0, LSQFIT_MAX_DEGREE>(m, [&](auto M) {
        constexpr int D = decltype(M)::value;
        if constexpr (D > LSQ_BATCH_SMALL_MAX_DEGREE) {
            if (ppc <= small_ppc_max_hi(D)) {
                // one thread per curve, the system in shared memory
                constexpr int T = lsq::small_threads<true>();
                uint64_t blocks = (n_curves + T - 1) / T;
                const uint64_t cap = uint64_t(ctx->sm_count) * 16;
                if (blocks > cap) blocks = cap;
                const double2* xy2 = reinterpret_cast<const double2*>(d_xy);
                constexpr size_t smem = lsq::small_solve_smem<D>();
                if (ppc >= 16)
                    lsq::batched_small_kernel<D, true, true><<<static_cast<unsigned>(blocks), T, smem, st>>>(
                        xy2, n_curves, ppc, d_coeffs, d_status);
                else
                    lsq::batched_small_kernel<D, false, true><<<static_cast<unsigned>(blocks), T, smem, st>>>(
                        xy2, n_curves, ppc, d_coeffs, d_status);
                return cudaGetLastError();
            }
        }
        if constexpr (D <= LSQ_BATCH_SMALL_MAX_DEGREE) {
            if (ppc <= small_ppc_max(D)) {
                // one thread per curve; grid-stride beyond 16 resident blocks per SM
                uint64_t blocks = (n_curves + lsq::kSmallThreads - 1) / lsq::kSmallThreads;
                const uint64_t cap = uint64_t(ctx->sm_count) * 16;
                if (blocks > cap) blocks = cap;
                const double2* xy2 = reinterpret_cast<const double2*>(d_xy);
                if (ppc >= 16)
                    lsq::batched_small_kernel<D, true><<<static_cast<unsigned>(blocks), lsq::kSmallThreads, 0, st>>>(
                        xy2, n_curves, ppc, d_coeffs, d_status);
                else
                    lsq::batched_small_kernel<D, false><<<static_cast<unsigned>(blocks), lsq::kSmallThreads, 0, st>>>(
                        xy2, n_curves, ppc, d_coeffs, d_status);
                return cudaGetLastError();
            }
        }
        uint64_t blocks = (n_curves + lsq::kBatchWarps - 1) / lsq::kBatchWarps;  // one warp per curve
        const uint64_t cap = static_cast<uint64_t>(ctx->batch_ctas[D]);
        if (blocks > cap) blocks = cap;
        if (blocks < 1) blocks = 1;
        // 256-bit loads need every curve base 32-byte aligned
        const bool v256 = (ppc % 2 == 0) && (reinterpret_cast<uintptr_t>(d_xy) % 32 == 0);
        if (v256)
            lsq::batched_fit_kernel<D, true><<<static_cast<unsigned>(blocks), lsq::kBatchThreads, 0, st>>>(
                d_xy, n_curves, ppc, d_coeffs, d_status, nullptr, ctx->d_batch_work);
        else
            lsq::batched_fit_kernel<D, false><<<static_cast<unsigned>(blocks), lsq::kBatchThreads, 0, st>>>(
                d_xy, n_curves, ppc, d_coeffs, d_status, nullptr, ctx->d_batch_work);
        return cudaGetLastError();
    });
}

// Ragged batch: curve c = points [offsets[c], offsets[c+1]) (device array of
// n_curves + 1). total_points only picks the kernel (mean curve length vs the
// crossovers above); results do not depend on it.
cudaError_t batched_ragged_launch(lsqfit_cuda_ctx* ctx, int m, const double* d_xy, const uint64_t* d_offsets,
                                  uint64_t n_curves, uint64_t total_points, double* d_coeffs, int32_t* d_status,
                                  cudaStream_t st) {
    const uint64_t mean = n_curves ? total_points / n_curves : 0;
    const double2* xy2 = reinterpret_cast<const double2*>(d_xy);
    const cudaError_t ce = ensure_batched(ctx, m);
    if (ce != cudaSuccess) return ce;
    return dispatch_degree<0, LSQFIT_MAX_DEGREE>(m, [&](auto M) {
        constexpr int D = decltype(M)::value;
        constexpr bool SMEM = D > LSQ_BATCH_SMALL_MAX_DEGREE;
        const uint64_t limit = SMEM ? small_ppc_max_hi(D) : small_ppc_max(D);
        const uint64_t cap = uint64_t(ctx->sm_count) * 16;
        if (mean <= limit) {  // thread per curve, direct loads
            constexpr int T = lsq::small_threads<SMEM>();
            uint64_t blocks = (n_curves + T - 1) / T;
            if (blocks > cap) blocks = cap;
            lsq::batched_small_kernel<D, false, SMEM>
                <<<static_cast<unsigned>(blocks ? blocks : 1), T, SMEM ? lsq::small_solve_smem<D>() : 0, st>>>(
                    xy2, n_curves, 0, d_coeffs, d_status, d_offsets);
        } else {  // warp per curve, 128-bit loads (curve bases only 16-byte aligned)
            uint64_t blocks = (n_curves + lsq::kBatchWarps - 1) / lsq::kBatchWarps;
            const uint64_t wcap = static_cast<uint64_t>(ctx->batch_ctas[D]);
            if (blocks > wcap) blocks = wcap;
            lsq::batched_fit_kernel<D, false, true>
                <<<static_cast<unsigned>(blocks ? blocks : 1), lsq::kBatchThreads, 0, st>>>(
                    d_xy, n_curves, 0, d_coeffs, d_status, d_offsets, ctx->d_batch_work);
        }
        return cudaGetLastError();
    });
}

}  // namespace lsq_impl

// k_ordered.cu — instantiates the reference-order kernels (ordered.cuh).
#include "internal.hpp"
#include "ordered.cuh"

#ifndef LSQ_ORDERED_WARP_MIN_POINTS
#define LSQ_ORDERED_WARP_MIN_POINTS 3072  // A/B: warp per chunk faster from ~3k points per chunk, a thread per chunk below
#endif

#ifndef LSQ_ORDERED_ROWS_MIN_CHUNKS
#define LSQ_ORDERED_ROWS_MIN_CHUNKS 8192  // thread per chunk with a cp.async row ring from this many chunks (A/B: 1.2-3.1x faster at 8k-32k chunks)
#endif

namespace lsq_impl {

static int g_rows_min_chunks = 0;  // dev A/B override (lsqfit_debug_set_ordered_rows_min)

cudaError_t ordered_launch(lsqfit_cuda_ctx* ctx, int m, const double* d_xy, uint64_t n, uint64_t chunks,
                           unsigned flags, lsqfit_result* out, cudaStream_t st) {
    return dispatch_degree<0, LSQFIT_MAX_DEGREE>(m, [&](auto M) {
        constexpr int D = decltype(M)::value;
        constexpr size_t stride = 3 * D + 2;
        cudaError_t e = grow(&ctx->d_oslots, &ctx->oslots_bytes, size_t(chunks) * stride * sizeof(double));
        if (e != cudaSuccess) return e;
        const uint64_t cap = uint64_t(ctx->sm_count) * 16;
        const uint64_t rows_min = g_rows_min_chunks ? uint64_t(g_rows_min_chunks) : uint64_t(LSQ_ORDERED_ROWS_MIN_CHUNKS);
        if (chunks >= rows_min) {
            // a thread per chunk, rows staged through a cp.async ring per warp
            // per call: the attribute is per device (contexts may differ)
            e = cudaFuncSetAttribute(lsq::ordered_rows_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(lsq::kRowSmemBytes));
            if (e != cudaSuccess) return e;
            // at most one resident wave (warps loop over chunk groups)
            int per_sm = 0;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lsq::ordered_rows_kernel<D>,
                                                              lsq::kRowWarps * 32, lsq::kRowSmemBytes);
            if (e != cudaSuccess) return e;
            uint64_t blocks = (chunks + 32 * lsq::kRowWarps - 1) / (32 * lsq::kRowWarps);
            const uint64_t rcap = uint64_t(ctx->sm_count) * uint64_t(per_sm > 0 ? per_sm : 1);
            if (blocks > rcap) blocks = rcap;
            lsq::ordered_rows_kernel<D><<<static_cast<unsigned>(blocks), lsq::kRowWarps * 32, lsq::kRowSmemBytes, st>>>(
                reinterpret_cast<const double2*>(d_xy), n, chunks, ctx->d_oslots);
        } else if (n / chunks >= uint64_t(LSQ_ORDERED_WARP_MIN_POINTS)) {
            // a warp per chunk: terms in parallel, the ordered adds one per point per column
            using WC = lsq::OrderedWarpCfg<D>;
            uint64_t blocks = (chunks + WC::WARPS - 1) / WC::WARPS;
            if (blocks > cap) blocks = cap;
            lsq::ordered_warp_kernel<D><<<static_cast<unsigned>(blocks), WC::THREADS, 0, st>>>(
                reinterpret_cast<const double2*>(d_xy), n, chunks, ctx->d_oslots);
        } else {
            uint64_t blocks = (chunks + lsq::kOrderedThreads - 1) / lsq::kOrderedThreads;
            if (blocks > cap) blocks = cap;
            lsq::ordered_chunks_kernel<D><<<static_cast<unsigned>(blocks), lsq::kOrderedThreads, 0, st>>>(
                reinterpret_cast<const double2*>(d_xy), n, chunks, ctx->d_oslots);
        }
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        lsq::ordered_combine_kernel<D><<<1, lsq::kOrderedCombineThreads, 0, st>>>(ctx->d_oslots, chunks, n, flags,
                                                                                  out);
        return cudaGetLastError();
    });
}

}  // namespace lsq_impl

extern "C" int lsqfit_debug_set_ordered_rows_min(int chunks) {
    if (chunks < 0) return LSQFIT_EINVAL;
    lsq_impl::g_rows_min_chunks = chunks;
    return LSQFIT_OK;
}

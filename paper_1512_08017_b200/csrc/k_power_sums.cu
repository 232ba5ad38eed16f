// k_power_sums.cu — the only translation unit instantiating the power-sum
// kernels (power_sums.cuh): occupancy/smem configuration and launches.
#include "internal.hpp"
#include "power_sums.cuh"

namespace lsq_impl {

static_assert(lsq::kDynMaxChunks == kPsDynMaxChunks,
              "dynamic-tail scratch sizing out of sync with power_sums.cuh");
static_assert(3 * LSQ_DYN_MAX + 1 <= kPsDynMaxNV, "dynamic-tail records wider than the scratch");

cudaError_t ps_configure(int m, int sm_count, int* ctas) {
    return dispatch_degree<0, LSQFIT_MAX_DEGREE>(m, [&](auto M) {
        constexpr int D = decltype(M)::value;
        using C = lsq::PsCfg<D>;
        cudaError_t e = cudaFuncSetAttribute(lsq::power_sums_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(C::SMEM_BYTES));
        if (e != cudaSuccess) return e;
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lsq::power_sums_kernel<D>, C::THREADS,
                                                          C::SMEM_BYTES);
        if (e != cudaSuccess) return e;
        if (per_sm < 1) return cudaErrorInvalidConfiguration;
        *ctas = sm_count * per_sm;
        return cudaSuccess;
    });
}

int ps_error_levels(int m) {
    if (m < 0 || m > LSQFIT_MAX_DEGREE) return -1;
    int levels = -1;
    dispatch_degree<0, LSQFIT_MAX_DEGREE>(m, [&](auto M) {
        levels = lsq::PsCfg<decltype(M)::value>::ERR_LEVELS;
        return cudaSuccess;
    });
    return levels;
}

cudaError_t ps_launch(lsqfit_cuda_ctx* ctx, int m, const double* d_xy, uint64_t n, unsigned flags,
                      lsqfit_result* out, cudaStream_t st) {
    return dispatch_degree<0, LSQFIT_MAX_DEGREE>(m, [&](auto M) {
        constexpr int D = decltype(M)::value;
        using C = lsq::PsCfg<D>;
        // no more CTAs than tiles (small n: less launch and grid-reduction
        // work); the partition stays a fixed function of (n, degree)
        const uint64_t tiles = (n + C::TILE - 1) / C::TILE;
        const unsigned grid = static_cast<unsigned>(tiles < uint64_t(ctx->ps_ctas[D]) ? (tiles ? tiles : 1)
                                                                                      : uint64_t(ctx->ps_ctas[D]));
        lsq::PsArgs a{reinterpret_cast<const double2*>(d_xy), n, ctx->d_slots, ctx->d_ticket, out, flags,
                      tiles, 0u, 0u, 0u, ctx->d_dyn_chunks, ctx->d_dyn_counters};
        // Dynamic tail (PsCfg::DYN): a fixed function of (n, degree, grid),
        // so the result is reproducible (lsq::dyn_plan).
        if (C::DYN && tiles >= uint64_t(LSQ_DYN_MIN_TILES_PER_CTA(D)) * grid) {
            const lsq::DynPlan p = lsq::dyn_plan(tiles, grid, LSQ_DYN_DEN, LSQ_DYN_CHUNK, lsq::kDynMaxChunks);
            a.static_tiles = p.static_tiles;
            a.chunk_s0 = p.s0;
            a.chunk_min = p.chunk_min;
            a.n_chunks = p.n_chunks;
        }
        lsq::power_sums_kernel<D><<<grid, C::THREADS, C::SMEM_BYTES, st>>>(a);
        return cudaGetLastError();
    });
}

cudaError_t ps_combine(int m, const lsqfit_result* parts, int count, unsigned flags, lsqfit_result* out,
                       cudaStream_t st) {
    return dispatch_degree<0, LSQFIT_MAX_DEGREE>(m, [&](auto M) {
        constexpr int D = decltype(M)::value;
        lsq::combine_kernel<D><<<1, lsq::kConsumers, 0, st>>>(parts, count, flags, out);
        return cudaGetLastError();
    });
}

}  // namespace lsq_impl

#ifdef LSQ_PS_TRACE
extern "C" int lsqfit_debug_ps_trace(unsigned long long* host, int rows) {
    return static_cast<int>(cudaMemcpyFromSymbol(host, lsq::g_ps_trace, size_t(rows) * 4 * sizeof(unsigned long long)));
}
#endif

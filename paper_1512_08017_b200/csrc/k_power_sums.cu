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

int ps_sum_terms(int m) {
    if (m < 0 || m > LSQFIT_MAX_DEGREE) return -1;
    int terms = -1;
    dispatch_degree<0, LSQFIT_MAX_DEGREE>(m, [&](auto M) {
        terms = lsq::PsCfg<decltype(M)::value>::PRODUCTS ? LSQFIT_TERMS_PRODUCTS : LSQFIT_TERMS_REFERENCE;
        return cudaSuccess;
    });
    return terms;
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

// Dev-only tuning overrides of the dynamic-tail plan (tools/ab_dyn.py):
// 0 keeps the compiled default. Not part of the C ABI.
static int g_dyn_den = 0, g_dyn_chunk = 0, g_dyn_min_tiles = 0;
static int g_ps_pdl = 1;  // programmatic dependent launch (dev A/B: lsqfit_debug_set_ps_pdl)

cudaError_t ps_launch(lsqfit_cuda_ctx* ctx, int m, const double* d_xy, uint64_t n, unsigned flags,
                      lsqfit_result* out, cudaStream_t st) {
    return dispatch_degree<0, LSQFIT_MAX_DEGREE>(m, [&](auto M) {
        constexpr int D = decltype(M)::value;
        using C = lsq::PsCfg<D>;
        const cudaError_t ce = ensure_ps(ctx, D);
        if (ce != cudaSuccess) return ce;
        // no more CTAs than tiles (small n: less launch and grid-reduction
        // work); the partition stays a fixed function of (n, degree)
        const uint64_t tiles = (n + C::TILE - 1) / C::TILE;
        const unsigned grid = static_cast<unsigned>(tiles < uint64_t(ctx->ps_ctas[D]) ? (tiles ? tiles : 1)
                                                                                      : uint64_t(ctx->ps_ctas[D]));
        lsq::PsArgs a{reinterpret_cast<const double2*>(d_xy), n, ctx->d_slots, ctx->d_ticket, out, flags,
                      tiles, 0u, 0u, 0u, ctx->d_dyn_chunks, ctx->d_dyn_counters};
        // Dynamic tail (PsCfg::DYN): a fixed function of (n, degree, grid),
        // so the result is reproducible (lsq::dyn_plan).
        // Mid-size launches (< 1024 tiles per CTA, n < ~5e8) take a smaller
        // tail in coarser chunks: A/B at n = 1e8, m = 3: 4.6% faster (m = 2:
        // 0.7%); at n >= 1e9 the long plan is as fast or faster
        // (profiles/r02_ab_dyn_pdl.txt).
        const bool mid = tiles < uint64_t(LSQ_DYN_MID_TILES_PER_CTA) * grid;
        const uint64_t min_tiles = g_dyn_min_tiles ? uint64_t(g_dyn_min_tiles)
                                   : mid           ? uint64_t(LSQ_DYN_MID_MIN_TILES)
                                                   : uint64_t(LSQ_DYN_MIN_TILES_PER_CTA(D));
        const uint64_t den = g_dyn_den ? g_dyn_den : mid ? LSQ_DYN_MID_DEN : LSQ_DYN_DEN;
        const uint64_t chunk = g_dyn_chunk ? g_dyn_chunk : mid ? LSQ_DYN_MID_CHUNK : LSQ_DYN_CHUNK;
        if (C::DYN && tiles >= min_tiles * grid) {
            const lsq::DynPlan p = lsq::dyn_plan(tiles, grid, den, chunk, lsq::kDynMaxChunks);
            a.static_tiles = p.static_tiles;
            a.chunk_s0 = p.s0;
            a.chunk_min = p.chunk_min;
            a.n_chunks = p.n_chunks;
        }
        // Programmatic dependent launch: back-to-back fits overlap this
        // launch's scheduling and prologue with the previous kernel's tail
        // (the kernel waits for it before touching global memory).
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(C::THREADS);
        cfg.dynamicSmemBytes = C::SMEM_BYTES;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = g_ps_pdl;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, lsq::power_sums_kernel<D>, a);
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

extern "C" int lsqfit_debug_set_ps_tuning(int den, int chunk, int min_tiles_per_cta) {
    if (den < 0 || chunk < 0 || min_tiles_per_cta < 0) return LSQFIT_EINVAL;
    lsq_impl::g_dyn_den = den;
    lsq_impl::g_dyn_chunk = chunk;
    lsq_impl::g_dyn_min_tiles = min_tiles_per_cta;
    return LSQFIT_OK;
}

extern "C" int lsqfit_debug_set_ps_pdl(int enabled) {
    lsq_impl::g_ps_pdl = enabled ? 1 : 0;
    return LSQFIT_OK;
}

#ifdef LSQ_PS_TRACE
extern "C" int lsqfit_debug_ps_trace(unsigned long long* host, int rows) {
    return static_cast<int>(cudaMemcpyFromSymbol(host, lsq::g_ps_trace, size_t(rows) * 8 * sizeof(unsigned long long)));
}
#endif

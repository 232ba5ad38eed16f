// k_qr.cu — instantiates the TSQR cross-check kernels (qr.cuh).
#include "internal.hpp"
#include "qr.cuh"

namespace lsq_impl {

cudaError_t qr_configure(int m, int sm_count, int* ctas) {
    return dispatch_degree<0, LSQFIT_MAX_QR_DEGREE>(m, [&](auto M) {
        constexpr int D = decltype(M)::value;
        using Q = lsq::QrCfg<D>;
        static_assert(Q::NT <= kQrSlotDoubles, "TSQR slot too small");
        cudaError_t e = cudaFuncSetAttribute(lsq::qr_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(Q::SMEM));
        if (e != cudaSuccess) return e;
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lsq::qr_kernel<D>, Q::THREADS, Q::SMEM);
        if (e != cudaSuccess) return e;
        *ctas = sm_count * (per_sm > 0 ? per_sm : 1);
        return cudaSuccess;
    });
}

cudaError_t qr_launch(lsqfit_cuda_ctx* ctx, int m, const double* d_xy, uint64_t n, unsigned flags,
                      lsqfit_qr_result* out, cudaStream_t st) {
    const cudaError_t ce = ensure_qr(ctx, m);
    if (ce != cudaSuccess) return ce;
    return dispatch_degree<0, LSQFIT_MAX_QR_DEGREE>(m, [&](auto M) {
        constexpr int D = decltype(M)::value;
        using Q = lsq::QrCfg<D>;
        lsq::QrArgs a{reinterpret_cast<const double2*>(d_xy), n, ctx->d_qslots, ctx->d_qbad, ctx->d_qticket, out,
                      flags};
        lsq::qr_kernel<D><<<ctx->qr_ctas[D], Q::THREADS, Q::SMEM, st>>>(a);
        return cudaGetLastError();
    });
}

cudaError_t qr_combine(int m, const lsqfit_qr_result* parts, int count, unsigned flags, lsqfit_qr_result* out,
                       cudaStream_t st) {
    return dispatch_degree<0, LSQFIT_MAX_QR_DEGREE>(m, [&](auto M) {
        constexpr int D = decltype(M)::value;
        lsq::qr_combine_kernel<D><<<1, 32, 0, st>>>(parts, count, flags, out);
        return cudaGetLastError();
    });
}

}  // namespace lsq_impl

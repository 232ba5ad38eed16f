// k_diagnostics.cu — instantiates the FitReport pass (diagnostics.cuh).
#include "diagnostics.cuh"
#include "internal.hpp"

namespace lsq_impl {

cudaError_t diag_launch(lsqfit_cuda_ctx* ctx, int m, const double* d_xy, uint64_t n, const double* d_coeffs,
                        const int32_t* d_gate, double shift, double* d_residuals, lsqfit_diag* out,
                        cudaStream_t st) {
    if (m > LSQFIT_MAX_DEGREE) {  // any polynomial degree: runtime Horner, coefficients in dynamic smem
        const size_t smem = size_t(m + 1) * sizeof(double);
        if (smem > 48 * 1024) {
            const cudaError_t e = cudaFuncSetAttribute(lsq::diagnostics_kernel<lsq::kAnyDegree>,
                                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       static_cast<int>(smem));
            if (e != cudaSuccess) return e;
        }
        uint64_t blocks = (n + lsq::kDiagThreads * lsq::kDiagBatch - 1) / (lsq::kDiagThreads * lsq::kDiagBatch);
        if (blocks > uint64_t(ctx->diag_ctas)) blocks = ctx->diag_ctas;
        if (blocks < 1) blocks = 1;
        lsq::diagnostics_kernel<lsq::kAnyDegree><<<static_cast<unsigned>(blocks), lsq::kDiagThreads, smem, st>>>(
            reinterpret_cast<const double2*>(d_xy), n, d_coeffs, d_gate, shift, d_residuals, ctx->d_dslots,
            ctx->d_dticket, out, m);
        return cudaGetLastError();
    }
    return dispatch_degree<0, LSQFIT_MAX_DEGREE>(m, [&](auto M) {
        constexpr int D = decltype(M)::value;
        uint64_t blocks = (n + lsq::kDiagThreads * lsq::kDiagBatch - 1) / (lsq::kDiagThreads * lsq::kDiagBatch);
        if (blocks > uint64_t(ctx->diag_ctas)) blocks = ctx->diag_ctas;
        if (blocks < 1) blocks = 1;
        lsq::diagnostics_kernel<D><<<static_cast<unsigned>(blocks), lsq::kDiagThreads, 0, st>>>(
            reinterpret_cast<const double2*>(d_xy), n, d_coeffs, d_gate, shift, d_residuals, ctx->d_dslots,
            ctx->d_dticket, out);
        return cudaGetLastError();
    });
}

cudaError_t diag_combine(const lsqfit_diag* parts, int count, lsqfit_diag* out, cudaStream_t st) {
    lsq::diag_combine_kernel<<<1, 32, 0, st>>>(parts, count, out);
    return cudaGetLastError();
}

}  // namespace lsq_impl

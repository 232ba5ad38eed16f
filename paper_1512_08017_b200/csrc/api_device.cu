// api_device.cu — device-resident entry points (asynchronous on a caller stream).
#include "internal.hpp"

using namespace lsq_impl;

namespace {
bool aligned16(const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; }
cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }
}  // namespace

extern "C" {

int lsqfit_cuda_fit_device(lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n, int degree, unsigned flags,
                           lsqfit_result* d_result, void* stream) {
    if (!ctx || !d_result || (n > 0 && !d_xy) || !aligned16(d_xy)) return LSQFIT_EINVAL;
    if (check_degree(degree) != LSQFIT_OK) return LSQFIT_EINVAL;
    LSQ_ON_DEVICE(ctx);
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, claim_scratch(ctx, as_stream(stream)));
    LSQ_TRY(ctx, ps_launch(ctx, degree, d_xy, n, flags, d_result, as_stream(stream)));
    return LSQFIT_OK;
}

int lsqfit_cuda_power_sums_device(lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n, int degree, double* d_st,
                                  int32_t* d_status, void* stream) {
    if (!ctx || !d_st || !d_status || n == 0 || !d_xy || !aligned16(d_xy)) return LSQFIT_EINVAL;
    if (degree < 0 || degree > kMaxAnyDegree) return LSQFIT_EINVAL;
    LSQ_ON_DEVICE(ctx);
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, claim_scratch(ctx, as_stream(stream)));
    const uint64_t B = anysums_blocks(ctx, n, degree);
    LSQ_TRY(ctx, grow(&ctx->d_aparts, &ctx->aparts_bytes, size_t(3 * degree + 1) * B * sizeof(double2)));
    LSQ_TRY(ctx, anysums_partial(ctx, d_xy, n, degree, B, ctx->d_aparts, as_stream(stream)));
    LSQ_TRY(ctx, anysums_final(ctx->d_aparts, 1, B, degree, n, d_st, d_status, as_stream(stream)));
    return LSQFIT_OK;
}

int lsqfit_cuda_fit_ordered_device(lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n, int degree, uint64_t chunks,
                                   unsigned flags, lsqfit_result* d_result, void* stream) {
    if (!ctx || !d_result || (n > 0 && !d_xy) || !aligned16(d_xy) || chunks < 1) return LSQFIT_EINVAL;
    if (check_degree(degree) != LSQFIT_OK) return LSQFIT_EINVAL;
    LSQ_ON_DEVICE(ctx);
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, claim_scratch(ctx, as_stream(stream)));
    LSQ_TRY(ctx, ordered_launch(ctx, degree, d_xy, n, chunks, flags, d_result, as_stream(stream)));
    return LSQFIT_OK;
}

int lsqfit_cuda_combine_device(lsqfit_cuda_ctx* ctx, const lsqfit_result* d_parts, int n_parts, int degree,
                               unsigned flags, lsqfit_result* d_result, void* stream) {
    if (!ctx || !d_parts || !d_result || n_parts < 1) return LSQFIT_EINVAL;
    if (check_degree(degree) != LSQFIT_OK) return LSQFIT_EINVAL;
    LSQ_ON_DEVICE(ctx);
    LSQ_TRY(ctx, ps_combine(degree, d_parts, n_parts, flags, d_result, as_stream(stream)));
    return LSQFIT_OK;
}

int lsqfit_cuda_diagnostics_device(lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n, int degree,
                                   const double* d_coeffs, const int32_t* d_gate, double shift,
                                   double* d_residuals, lsqfit_diag* d_out, void* stream) {
    if (!ctx || !d_coeffs || !d_out || n == 0 || !d_xy || !aligned16(d_xy)) return LSQFIT_EINVAL;
    if (degree < 0 || degree > kMaxAnyDegree) return LSQFIT_EINVAL;  // any polynomial degree
    LSQ_ON_DEVICE(ctx);
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, claim_scratch(ctx, as_stream(stream)));
    LSQ_TRY(ctx,
            diag_launch(ctx, degree, d_xy, n, d_coeffs, d_gate, shift, d_residuals, d_out, as_stream(stream)));
    return LSQFIT_OK;
}

int lsqfit_cuda_fit_batched_device(lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n_curves,
                                   uint32_t points_per_curve, int degree, double* d_coeffs, int32_t* d_status,
                                   void* stream) {
    if (!ctx || !d_coeffs || !d_status || (n_curves > 0 && !d_xy) || points_per_curve == 0 || !aligned16(d_xy))
        return LSQFIT_EINVAL;
    if (check_degree(degree) != LSQFIT_OK) return LSQFIT_EINVAL;
    if (n_curves == 0) return LSQFIT_OK;
    LSQ_ON_DEVICE(ctx);
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, claim_scratch(ctx, as_stream(stream)));  // the warp kernel's curve-claim counters
    LSQ_TRY(ctx, batched_launch(ctx, degree, d_xy, n_curves, points_per_curve, d_coeffs, d_status, as_stream(stream)));
    return LSQFIT_OK;
}

int lsqfit_cuda_fit_batched_ragged_device(lsqfit_cuda_ctx* ctx, const double* d_xy, const uint64_t* d_offsets,
                                          uint64_t n_curves, uint64_t total_points, int degree, double* d_coeffs,
                                          int32_t* d_status, void* stream) {
    if (!ctx || !d_offsets || !d_coeffs || !d_status || (n_curves > 0 && !d_xy) || !aligned16(d_xy))
        return LSQFIT_EINVAL;
    if (check_degree(degree) != LSQFIT_OK) return LSQFIT_EINVAL;
    if (n_curves == 0) return LSQFIT_OK;
    LSQ_ON_DEVICE(ctx);
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, claim_scratch(ctx, as_stream(stream)));
    LSQ_TRY(ctx, batched_ragged_launch(ctx, degree, d_xy, d_offsets, n_curves, total_points, d_coeffs, d_status,
                                       as_stream(stream)));
    return LSQFIT_OK;
}

int lsqfit_cuda_qr_fit_device(lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n, int degree, unsigned flags,
                              lsqfit_qr_result* d_result, void* stream) {
    if (!ctx || !d_result || (n > 0 && !d_xy) || !aligned16(d_xy)) return LSQFIT_EINVAL;
    if (degree < 0 || degree > LSQFIT_MAX_QR_DEGREE) return LSQFIT_EINVAL;
    LSQ_ON_DEVICE(ctx);
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, claim_scratch(ctx, as_stream(stream)));
    LSQ_TRY(ctx, qr_launch(ctx, degree, d_xy, n, flags, d_result, as_stream(stream)));
    return LSQFIT_OK;
}

int lsqfit_cuda_qr_combine_device(lsqfit_cuda_ctx* ctx, const lsqfit_qr_result* d_parts, int n_parts, int degree,
                                  unsigned flags, lsqfit_qr_result* d_result, void* stream) {
    if (!ctx || !d_parts || !d_result || n_parts < 1) return LSQFIT_EINVAL;
    if (degree < 0 || degree > LSQFIT_MAX_QR_DEGREE) return LSQFIT_EINVAL;
    LSQ_ON_DEVICE(ctx);
    LSQ_TRY(ctx, qr_combine(degree, d_parts, n_parts, flags, d_result, as_stream(stream)));
    return LSQFIT_OK;
}

int lsqfit_cuda_synth_device(lsqfit_cuda_ctx* ctx, double* d_xy, uint64_t n, uint64_t offset, uint64_t seed,
                             int truth_degree, double sigma, void* stream) {
    if (!ctx || (n > 0 && !d_xy) || truth_degree < 0 || truth_degree > LSQFIT_MAX_DEGREE) return LSQFIT_EINVAL;
    if (n == 0) return LSQFIT_OK;
    LSQ_ON_DEVICE(ctx);
    LSQ_TRY(ctx, synth_launch(ctx->sm_count, d_xy, n, offset, seed, truth_degree, sigma, as_stream(stream)));
    return LSQFIT_OK;
}

int lsqfit_cuda_synth_batched_device(lsqfit_cuda_ctx* ctx, double* d_xy, uint64_t n_curves,
                                     uint32_t points_per_curve, uint64_t seed, int truth_degree, double sigma,
                                     void* stream) {
    if (!ctx || (n_curves > 0 && !d_xy) || truth_degree < 0 || truth_degree > LSQFIT_MAX_DEGREE) return LSQFIT_EINVAL;
    if (n_curves == 0 || points_per_curve == 0) return LSQFIT_OK;
    LSQ_ON_DEVICE(ctx);
    LSQ_TRY(ctx, synth_batched_launch(ctx->sm_count, d_xy, n_curves, points_per_curve, seed, truth_degree, sigma,
                                      as_stream(stream)));
    return LSQFIT_OK;
}

}  // extern "C"

// api_host.cu — host-resident entry points: the drop-in path behind
// accumulate / fit_normal / make_fit_report / solve_gaussian / the QR and
// batched fits. Synchronous; serialised per context by ctx->mu.
#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.hpp"

namespace lsq_impl {

bool can_keep_resident(lsqfit_cuda_ctx* ctx, uint64_t n) {
    const char* off = std::getenv("LSQFIT_CUDA_NO_RESIDENT");  // force re-streaming (tests)
    if (off && off[0] == '1' && n_chunks(ctx, n) > 1) return false;
    const size_t need = size_t(n) * 16;
    if (need <= ctx->buf_bytes) return true;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return need + (size_t(4) << 30) <= free_b + ctx->buf_bytes;
}

cudaError_t enqueue_fit(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, int degree, unsigned flags,
                        bool resident) {
    const uint64_t K = n_chunks(ctx, n);
    if (K > 1) {
        const cudaError_t e = grow(&ctx->d_recs, &ctx->recs_bytes, size_t(K) * sizeof(lsqfit_result));
        if (e != cudaSuccess) return e;
    }
    auto chunk = [&](uint64_t k, const double* d, uint64_t cnt) {
        return K == 1 ? ps_launch(ctx, degree, d, cnt, flags, ctx->d_result, ctx->stream)
                      : ps_launch(ctx, degree, d, cnt, LSQFIT_SUMS, ctx->d_recs + k, ctx->stream);
    };
    const cudaError_t e = resident ? stream_points_resident(ctx, xy, n, chunk) : stream_points(ctx, xy, n, chunk);
    if (e != cudaSuccess || K == 1) return e;
    return ps_combine(degree, ctx->d_recs, static_cast<int>(K), flags, ctx->d_result, ctx->stream);
}

cudaError_t enqueue_report(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, int degree, const double* d_coeffs,
                           const int32_t* d_gate, double shift, double* residuals, const double* d_resident) {
    const uint64_t K = n_chunks(ctx, n);
    const uint64_t C = K == 1 ? n : ctx->chunk_points;
    cudaError_t e;
    if (residuals &&
        (e = grow(&ctx->d_res, &ctx->res_bytes, size_t(C) * sizeof(double) * (K == 1 ? 1 : 2))) != cudaSuccess)
        return e;
    if (K > 1 && (e = grow(&ctx->d_drecs, &ctx->drecs_bytes, size_t(K) * sizeof(lsqfit_diag))) != cudaSuccess)
        return e;
    auto chunk = [&](uint64_t k, const double* d, uint64_t cnt) {
        double* d_res = residuals ? ctx->d_res + (K == 1 ? 0 : (k & 1) * C) : nullptr;
        lsqfit_diag* out = K == 1 ? ctx->d_diag : ctx->d_drecs + k;
        cudaError_t e2 = diag_launch(ctx, degree, d, cnt, d_coeffs, d_gate, shift, d_res, out, ctx->stream);
        if (e2 == cudaSuccess && residuals)
            e2 = ctx->stager.d2h(residuals + k * C, d_res, size_t(cnt) * sizeof(double), ctx->stream);
        return e2;
    };
    e = d_resident ? for_resident_chunks(ctx, d_resident, n, chunk) : stream_points(ctx, xy, n, chunk);
    if (e != cudaSuccess || K == 1) return e;
    return diag_combine(ctx->d_drecs, static_cast<int>(K), ctx->d_diag, ctx->stream);
}

}  // namespace lsq_impl

using namespace lsq_impl;

extern "C" {

int lsqfit_cuda_fit_host(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, int degree, unsigned flags,
                         lsqfit_result* result) {
    if (!ctx || !result || !xy || n == 0) return LSQFIT_EINVAL;
    if (check_degree(degree) != LSQFIT_OK) return LSQFIT_EINVAL;
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, cudaSetDevice(ctx->device));
    LSQ_TRY(ctx, claim_scratch(ctx, ctx->stream));
    LSQ_TRY(ctx, enqueue_fit(ctx, xy, n, degree, flags));
    LSQ_TRY(ctx, cudaMemcpyAsync(ctx->h_result, ctx->d_result, sizeof(lsqfit_result), cudaMemcpyDeviceToHost,
                                 ctx->stream));
    LSQ_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    std::memcpy(result, ctx->h_result, sizeof(lsqfit_result));
    return result->status;
}

int lsqfit_cuda_fit_ordered_host(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, int degree, uint64_t chunks,
                                 unsigned flags, lsqfit_result* result) {
    if (!ctx || !result || !xy || n == 0 || chunks < 1) return LSQFIT_EINVAL;
    if (check_degree(degree) != LSQFIT_OK) return LSQFIT_EINVAL;
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, cudaSetDevice(ctx->device));
    LSQ_TRY(ctx, claim_scratch(ctx, ctx->stream));
    LSQ_TRY(ctx, grow(&ctx->d_buf, &ctx->buf_bytes, size_t(n) * 16));
    LSQ_TRY(ctx, ctx->stager.h2d(ctx->d_buf, xy, size_t(n) * 16, ctx->stream));
    LSQ_TRY(ctx, ordered_launch(ctx, degree, ctx->d_buf, n, chunks, flags, ctx->d_result, ctx->stream));
    LSQ_TRY(ctx, cudaMemcpyAsync(ctx->h_result, ctx->d_result, sizeof(lsqfit_result), cudaMemcpyDeviceToHost,
                                 ctx->stream));
    LSQ_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    std::memcpy(result, ctx->h_result, sizeof(lsqfit_result));
    return result->status;
}

int lsqfit_cuda_fit_report_host(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, int degree,
                                lsqfit_result* result, lsqfit_diag* diag, double* residuals) {
    if (!ctx || !result || !diag || !xy || n == 0) return LSQFIT_EINVAL;
    if (check_degree(degree) != LSQFIT_OK) return LSQFIT_EINVAL;
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, cudaSetDevice(ctx->device));
    LSQ_TRY(ctx, claim_scratch(ctx, ctx->stream));
    // The points cross PCIe once when they fit in HBM (the report pass then
    // re-reads them there), else they are re-streamed for the second pass.
    const bool resident = can_keep_resident(ctx, n);
    LSQ_TRY(ctx, enqueue_fit(ctx, xy, n, degree, LSQFIT_SOLVE, resident));
    // second pass: residuals, SSE, R — skipped on the device if the fit failed
    // (gate = the fit's status)
    LSQ_TRY(ctx, enqueue_report(ctx, xy, n, degree, ctx->d_result->coeffs, &ctx->d_result->status, xy[1], residuals,
                                resident ? ctx->d_buf : nullptr));
    LSQ_TRY(ctx, cudaMemcpyAsync(ctx->h_result, ctx->d_result, sizeof(lsqfit_result), cudaMemcpyDeviceToHost,
                                 ctx->stream));
    LSQ_TRY(ctx, cudaMemcpyAsync(ctx->h_diag, ctx->d_diag, sizeof(lsqfit_diag), cudaMemcpyDeviceToHost, ctx->stream));
    LSQ_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    std::memcpy(result, ctx->h_result, sizeof(lsqfit_result));
    std::memcpy(diag, ctx->h_diag, sizeof(lsqfit_diag));
    if (result->status != LSQFIT_OK) return result->status;
    return diag->status;
}

int lsqfit_cuda_report_host(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, const double* coeffs, int degree,
                            lsqfit_diag* diag, double* residuals) {
    if (!ctx || !xy || !coeffs || !diag || n == 0) return LSQFIT_EINVAL;
    if (degree < 0 || degree > kMaxAnyDegree) return LSQFIT_EINVAL;  // any polynomial, as the reference
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, cudaSetDevice(ctx->device));
    LSQ_TRY(ctx, claim_scratch(ctx, ctx->stream));
    double* d_coeffs = ctx->d_result->coeffs;  // ctx-owned scratch (held under ctx->mu)
    if (degree > LSQFIT_MAX_DEGREE) {
        LSQ_TRY(ctx, grow(&ctx->d_aout, &ctx->aout_bytes, sizeof(double) * (size_t(3 * degree + 2) + 1)));
        d_coeffs = ctx->d_aout;
    }
    LSQ_TRY(ctx, cudaMemcpyAsync(d_coeffs, coeffs, sizeof(double) * (degree + 1), cudaMemcpyHostToDevice,
                                 ctx->stream));
    LSQ_TRY(ctx, enqueue_report(ctx, xy, n, degree, d_coeffs, nullptr, xy[1], residuals));
    LSQ_TRY(ctx, cudaMemcpyAsync(ctx->h_diag, ctx->d_diag, sizeof(lsqfit_diag), cudaMemcpyDeviceToHost, ctx->stream));
    LSQ_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    std::memcpy(diag, ctx->h_diag, sizeof(lsqfit_diag));
    return diag->status;
}

int lsqfit_cuda_power_sums_host(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, int degree, double* s,
                                double* t) {
    if (!ctx || !xy || !s || !t || n == 0 || degree < 0 || degree > kMaxAnyDegree) return LSQFIT_EINVAL;
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, cudaSetDevice(ctx->device));
    LSQ_TRY(ctx, claim_scratch(ctx, ctx->stream));
    if (degree <= LSQFIT_MAX_DEGREE) {  // the fused kernel
        LSQ_TRY(ctx, enqueue_fit(ctx, xy, n, degree, LSQFIT_SUMS));
        LSQ_TRY(ctx, cudaMemcpyAsync(ctx->h_result, ctx->d_result, sizeof(lsqfit_result), cudaMemcpyDeviceToHost,
                                     ctx->stream));
        LSQ_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        std::memcpy(s, ctx->h_result->s, sizeof(double) * (2 * degree + 1));
        std::memcpy(t, ctx->h_result->t, sizeof(double) * (degree + 1));
        return ctx->h_result->status;
    }
    const int m = degree;
    const uint64_t K = n_chunks(ctx, n);
    const uint64_t C = K == 1 ? n : ctx->chunk_points;
    const uint64_t B = anysums_blocks(ctx, C, m);
    const size_t nc = size_t(3 * m + 1);
    LSQ_TRY(ctx, grow(&ctx->d_aparts, &ctx->aparts_bytes, size_t(K) * nc * B * sizeof(double2)));
    const size_t out_doubles = size_t(3 * m + 2);
    LSQ_TRY(ctx, grow(&ctx->d_aout, &ctx->aout_bytes, out_doubles * sizeof(double) + sizeof(double)));
    int* d_status = reinterpret_cast<int*>(ctx->d_aout + out_doubles);
    LSQ_TRY(ctx, stream_points(ctx, xy, n, [&](uint64_t k, const double* d, uint64_t cnt) {
                return anysums_partial(ctx, d, cnt, m, B, ctx->d_aparts + k * nc * B, ctx->stream);
            }));
    LSQ_TRY(ctx, anysums_final(ctx->d_aparts, static_cast<int>(K), B, m, n, ctx->d_aout, d_status, ctx->stream));
    int status = LSQFIT_OK;
    LSQ_TRY(ctx, cudaMemcpyAsync(s, ctx->d_aout, sizeof(double) * (2 * m + 1), cudaMemcpyDeviceToHost, ctx->stream));
    LSQ_TRY(ctx, cudaMemcpyAsync(t, ctx->d_aout + (2 * m + 1), sizeof(double) * (m + 1), cudaMemcpyDeviceToHost,
                                 ctx->stream));
    LSQ_TRY(ctx, cudaMemcpyAsync(&status, d_status, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    LSQ_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return status;
}

int lsqfit_cuda_power_sums_ordered_host(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, int degree,
                                        uint64_t chunks, double* s, double* t) {
    if (!ctx || !xy || !s || !t || n == 0 || chunks < 1 || degree < 0 || degree > kMaxAnyDegree)
        return LSQFIT_EINVAL;
    if (degree <= LSQFIT_MAX_DEGREE) {  // the specialised reference-order kernels
        lsqfit_result r{};
        const int st = lsqfit_cuda_fit_ordered_host(ctx, xy, n, degree, chunks, LSQFIT_SUMS, &r);
        if (st != LSQFIT_OK && st != LSQFIT_EOVERFLOW) return st;
        std::memcpy(s, r.s, sizeof(double) * (2 * degree + 1));
        std::memcpy(t, r.t, sizeof(double) * (degree + 1));
        return r.status;
    }
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, cudaSetDevice(ctx->device));
    LSQ_TRY(ctx, claim_scratch(ctx, ctx->stream));
    const int m = degree;
    const size_t stride = size_t(3 * m + 2);
    LSQ_TRY(ctx, grow(&ctx->d_buf, &ctx->buf_bytes, size_t(n) * 16));
    LSQ_TRY(ctx, grow(&ctx->d_oslots, &ctx->oslots_bytes, size_t(chunks) * stride * sizeof(double)));
    LSQ_TRY(ctx, grow(&ctx->d_aout, &ctx->aout_bytes, stride * sizeof(double) + sizeof(double)));
    int* d_status = reinterpret_cast<int*>(ctx->d_aout + stride);
    LSQ_TRY(ctx, ctx->stager.h2d(ctx->d_buf, xy, size_t(n) * 16, ctx->stream));
    LSQ_TRY(ctx, ordered_any(ctx, ctx->d_buf, n, m, chunks, ctx->d_oslots, ctx->d_aout, d_status, ctx->stream));
    int status = LSQFIT_OK;
    LSQ_TRY(ctx, cudaMemcpyAsync(s, ctx->d_aout, sizeof(double) * (2 * m + 1), cudaMemcpyDeviceToHost, ctx->stream));
    LSQ_TRY(ctx, cudaMemcpyAsync(t, ctx->d_aout + (2 * m + 1), sizeof(double) * (m + 1), cudaMemcpyDeviceToHost,
                                 ctx->stream));
    LSQ_TRY(ctx, cudaMemcpyAsync(&status, d_status, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    LSQ_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return status;
}

int lsqfit_cuda_fit_batched_host(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n_curves,
                                 uint32_t points_per_curve, int degree, double* coeffs, int32_t* status) {
    if (!ctx || !xy || !coeffs || !status || points_per_curve == 0) return LSQFIT_EINVAL;
    if (check_degree(degree) != LSQFIT_OK) return LSQFIT_EINVAL;
    if (n_curves == 0) return LSQFIT_OK;
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, cudaSetDevice(ctx->device));
    LSQ_TRY(ctx, claim_scratch(ctx, ctx->stream));
    const size_t in_bytes = size_t(n_curves) * points_per_curve * 16;
    const size_t c_bytes = size_t(n_curves) * (degree + 1) * sizeof(double);
    const size_t c_pad = (c_bytes + 15) & ~size_t(15);
    const size_t s_bytes = size_t(n_curves) * sizeof(int32_t);
    LSQ_TRY(ctx, grow(&ctx->d_buf, &ctx->buf_bytes, in_bytes));
    LSQ_TRY(ctx, grow(&ctx->d_res, &ctx->res_bytes, c_pad + s_bytes));
    double* d_coeffs = ctx->d_res;
    int32_t* d_status = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(ctx->d_res) + c_pad);
    LSQ_TRY(ctx, ctx->stager.h2d(ctx->d_buf, xy, in_bytes, ctx->stream));
    LSQ_TRY(ctx, batched_launch(ctx, degree, ctx->d_buf, n_curves, points_per_curve, d_coeffs, d_status, ctx->stream));
    LSQ_TRY(ctx, ctx->stager.d2h(coeffs, d_coeffs, c_bytes, ctx->stream));
    LSQ_TRY(ctx, ctx->stager.d2h(status, d_status, s_bytes, ctx->stream));
    LSQ_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return LSQFIT_OK;
}

int lsqfit_cuda_fit_batched_ragged_host(lsqfit_cuda_ctx* ctx, const double* xy, const uint64_t* offsets,
                                        uint64_t n_curves, int degree, double* coeffs, int32_t* status) {
    if (!ctx || !offsets || !coeffs || !status) return LSQFIT_EINVAL;
    if (check_degree(degree) != LSQFIT_OK) return LSQFIT_EINVAL;
    if (n_curves == 0) return LSQFIT_OK;
    const uint64_t first = offsets[0], last = offsets[n_curves];
    for (uint64_t c = 0; c < n_curves; ++c)
        if (offsets[c + 1] < offsets[c]) return LSQFIT_EINVAL;  // non-decreasing
    if (last > first && !xy) return LSQFIT_EINVAL;
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, cudaSetDevice(ctx->device));
    LSQ_TRY(ctx, claim_scratch(ctx, ctx->stream));
    const uint64_t total = last - first;
    const size_t in_bytes = size_t(total) * 16;
    const size_t off_bytes = size_t(n_curves + 1) * sizeof(uint64_t);
    const size_t c_bytes = size_t(n_curves) * (degree + 1) * sizeof(double);
    const size_t c_pad = (c_bytes + 15) & ~size_t(15);
    const size_t s_bytes = size_t(n_curves) * sizeof(int32_t);
    const size_t in_pad = (in_bytes + 15) & ~size_t(15);
    LSQ_TRY(ctx, grow(&ctx->d_buf, &ctx->buf_bytes, in_pad + off_bytes + 16));
    LSQ_TRY(ctx, grow(&ctx->d_res, &ctx->res_bytes, c_pad + s_bytes));
    double* d_xy = ctx->d_buf;
    uint64_t* d_off = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(ctx->d_buf) + in_pad);
    double* d_coeffs = ctx->d_res;
    int32_t* d_status = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(ctx->d_res) + c_pad);
    if (in_bytes) LSQ_TRY(ctx, ctx->stager.h2d(d_xy, xy + 2 * first, in_bytes, ctx->stream));
    // offsets rebased to the copied range
    std::vector<uint64_t> rebased;
    try {
        rebased.resize(n_curves + 1);
    } catch (...) {
        return LSQFIT_ENOMEM;
    }
    for (uint64_t c = 0; c <= n_curves; ++c) rebased[c] = offsets[c] - first;
    LSQ_TRY(ctx, cudaMemcpyAsync(d_off, rebased.data(), off_bytes, cudaMemcpyHostToDevice, ctx->stream));
    LSQ_TRY(ctx, batched_ragged_launch(ctx, degree, d_xy, d_off, n_curves, total, d_coeffs, d_status, ctx->stream));
    LSQ_TRY(ctx, ctx->stager.d2h(coeffs, d_coeffs, c_bytes, ctx->stream));
    LSQ_TRY(ctx, ctx->stager.d2h(status, d_status, s_bytes, ctx->stream));
    LSQ_TRY(ctx, cudaStreamSynchronize(ctx->stream));  // (also keeps `rebased` alive for the H2D)
    return LSQFIT_OK;
}

int lsqfit_cuda_qr_fit_host(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, int degree, lsqfit_qr_result* result) {
    if (!ctx || !result || !xy || n == 0) return LSQFIT_EINVAL;
    if (degree < 0 || degree > LSQFIT_MAX_QR_DEGREE) return LSQFIT_EINVAL;
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, cudaSetDevice(ctx->device));
    LSQ_TRY(ctx, claim_scratch(ctx, ctx->stream));
    const uint64_t K = n_chunks(ctx, n);
    if (K == 1) {
        LSQ_TRY(ctx, stream_points(ctx, xy, n, [&](uint64_t, const double* d, uint64_t cnt) {
                    return qr_launch(ctx, degree, d, cnt, LSQFIT_SOLVE, ctx->d_qresult, ctx->stream);
                }));
    } else {
        LSQ_TRY(ctx, grow(&ctx->d_qrecs, &ctx->qrecs_bytes, size_t(K) * sizeof(lsqfit_qr_result)));
        LSQ_TRY(ctx, stream_points(ctx, xy, n, [&](uint64_t k, const double* d, uint64_t cnt) {
                    return qr_launch(ctx, degree, d, cnt, LSQFIT_SUMS, ctx->d_qrecs + k, ctx->stream);
                }));
        LSQ_TRY(ctx, qr_combine(degree, ctx->d_qrecs, static_cast<int>(K), LSQFIT_SOLVE, ctx->d_qresult, ctx->stream));
    }
    LSQ_TRY(ctx, cudaMemcpyAsync(ctx->h_qresult, ctx->d_qresult, sizeof(lsqfit_qr_result), cudaMemcpyDeviceToHost,
                                 ctx->stream));
    LSQ_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    std::memcpy(result, ctx->h_qresult, sizeof(lsqfit_qr_result));
    return result->status;
}

int lsqfit_cuda_solve_sums_host(lsqfit_cuda_ctx* ctx, const double* s, const double* t, int degree, double* coeffs) {
    if (!ctx || !s || !t || !coeffs || degree < 0 || degree + 1 > LSQFIT_MAX_SOLVE_DIM) return LSQFIT_EINVAL;
    const int dim = degree + 1;
    std::vector<double> a;
    try {  // no exception may cross the C ABI
        a.resize(size_t(dim) * dim);
    } catch (...) {
        return LSQFIT_ENOMEM;
    }
    for (int j = 0; j < dim; ++j)  // build_normal_system: a(j,k) = s[j+k], b = t
        for (int k = 0; k < dim; ++k) a[size_t(j) * dim + k] = s[j + k];
    return lsqfit_cuda_solve_host(ctx, a.data(), t, dim, coeffs);
}

int lsqfit_cuda_solve_host(lsqfit_cuda_ctx* ctx, const double* a, const double* b, int dim, double* x) {
    if (!ctx || !a || !b || !x) return LSQFIT_EINVAL;
    if (dim < 1 || dim > LSQFIT_MAX_SOLVE_DIM) return LSQFIT_EINVAL;
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, cudaSetDevice(ctx->device));
    LSQ_TRY(ctx, claim_scratch(ctx, ctx->stream));
    const size_t na = size_t(dim) * dim;
    LSQ_TRY(ctx, grow(&ctx->d_buf, &ctx->buf_bytes, (na + 2 * size_t(dim)) * sizeof(double) + sizeof(int)));
    double* da = ctx->d_buf;
    double* db = da + na;
    double* dx = db + dim;
    int* dst = reinterpret_cast<int*>(dx + dim);
    LSQ_TRY(ctx, cudaMemcpyAsync(da, a, na * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    LSQ_TRY(ctx, cudaMemcpyAsync(db, b, dim * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    LSQ_TRY(ctx, solve_launch(da, db, dim, dx, dst, ctx->stream));
    int status = 0;
    LSQ_TRY(ctx, cudaMemcpyAsync(x, dx, dim * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    LSQ_TRY(ctx, cudaMemcpyAsync(&status, dst, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    LSQ_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return status;
}

}  // extern "C"

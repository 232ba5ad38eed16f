// capi.cu — the C ABI (include/lsqfit_cuda.h): contexts, launch tables and the
// host-resident / device-resident entry points. No exception crosses it.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

#include "batched.cuh"
#include "diagnostics.cuh"
#include "lsqfit_cuda.h"
#include "power_sums.cuh"
#include "solve.cuh"
#include "synth.cuh"
#include "qr.cuh"
#include "host_staging.hpp"

struct lsqfit_cuda_ctx {
    int device = 0;
    int sm_count = 0;
    int ps_ctas[LSQFIT_MAX_DEGREE + 1] = {};  // persistent grid per degree
    int batch_ctas[LSQFIT_MAX_DEGREE + 1] = {};
    cudaStream_t stream = nullptr;             // host-path stream
    double2* d_slots = nullptr;                // [max grid][LSQFIT_MAX_NV] dd partials
    unsigned* d_ticket = nullptr;
    int qr_ctas[LSQFIT_MAX_QR_DEGREE + 1] = {};  // TSQR grid per degree
    double* d_qslots = nullptr;                  // [max grid][55] packed factors
    int* d_qbad = nullptr;
    unsigned* d_qticket = nullptr;
    lsqfit_qr_result* d_qresult = nullptr;
    lsqfit_qr_result* h_qresult = nullptr;       // pinned
    lsqfit_qr_result* d_qrecs = nullptr;         // streamed chunk records
    size_t qrecs_bytes = 0;
    lsqfit_result* d_result = nullptr;         // host-path result
    lsqfit_result* h_result = nullptr;         // pinned
    double2* d_dslots = nullptr;               // diagnostics per-CTA partials
    unsigned* d_dticket = nullptr;
    int diag_ctas = 0;
    lsqfit_diag* d_diag = nullptr;
    lsqfit_diag* h_diag = nullptr;             // pinned
    double* d_res = nullptr;                   // residual staging (grow-only)
    size_t res_bytes = 0;
    double* d_buf = nullptr;                   // host-path staging (grow-only)
    size_t buf_bytes = 0;
    // out-of-core streaming of host inputs
    uint64_t chunk_points = 0;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_copied[2] = {nullptr, nullptr};
    cudaEvent_t ev_consumed[2] = {nullptr, nullptr};
    double* d_sbuf[2] = {nullptr, nullptr};
    size_t sbuf_bytes[2] = {0, 0};
    lsqfit_result* d_recs = nullptr;
    size_t recs_bytes = 0;
    lsqfit_diag* d_drecs = nullptr;
    size_t drecs_bytes = 0;
    lsq_host::Stager stager;                   // pageable host <-> device copies
    std::mutex mu;
    char last_error[256] = {0};
};

namespace {

using lsq::PsCfg;

constexpr uint64_t kDefaultStreamChunk = uint64_t(1) << 27;  // points (2 GiB per buffer)

int record(lsqfit_cuda_ctx* ctx, cudaError_t e) {
    if (e == cudaSuccess) return LSQFIT_OK;
    if (ctx) std::snprintf(ctx->last_error, sizeof ctx->last_error, "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? LSQFIT_ENOMEM : LSQFIT_ECUDA;
}

#define LSQ_TRY(ctx, expr)                          \
    do {                                            \
        const cudaError_t _e = (expr);              \
        if (_e != cudaSuccess) return record(ctx, _e); \
    } while (0)

// Launch table over the compile-time degree.
template <int M>
cudaError_t configure_ps(int sm_count, int* ctas) {
    using C = PsCfg<M>;
    cudaError_t e = cudaFuncSetAttribute(lsq::power_sums_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(C::SMEM_BYTES));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lsq::power_sums_kernel<M>, lsq::kPsThreads,
                                                      C::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    *ctas = sm_count * per_sm;
    int b_per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b_per_sm, lsq::batched_fit_kernel<M, true>,
                                                      lsq::kBatchThreads, 0);
    if (e != cudaSuccess) return e;
    ctas[LSQFIT_MAX_DEGREE + 1] = sm_count * (b_per_sm > 0 ? b_per_sm : 1);
    return cudaSuccess;
}

template <int M>
cudaError_t launch_ps(lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n, unsigned flags, lsqfit_result* d_out,
                      cudaStream_t st) {
    lsq::PsArgs a{reinterpret_cast<const double2*>(d_xy), n, ctx->d_slots, ctx->d_ticket, d_out, flags};
    lsq::power_sums_kernel<M><<<ctx->ps_ctas[M], lsq::kPsThreads, PsCfg<M>::SMEM_BYTES, st>>>(a);
    return cudaGetLastError();
}

template <int M>
cudaError_t launch_combine(const lsqfit_result* parts, int n_parts, unsigned flags, lsqfit_result* d_out,
                           cudaStream_t st) {
    lsq::combine_kernel<M><<<1, lsq::kConsumers, 0, st>>>(parts, n_parts, flags, d_out);
    return cudaGetLastError();
}

template <int M>
cudaError_t launch_batched(lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n_curves, uint32_t ppc,
                           double* coeffs, int32_t* status, cudaStream_t st) {
    const uint64_t warps_needed = (n_curves + 0);
    uint64_t blocks = (warps_needed + lsq::kBatchWarps - 1) / lsq::kBatchWarps;
    const uint64_t cap = static_cast<uint64_t>(ctx->batch_ctas[M]);
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    const bool v256 = (ppc % 2 == 0) && (reinterpret_cast<uintptr_t>(d_xy) % 32 == 0);
    if (v256)
        lsq::batched_fit_kernel<M, true><<<static_cast<unsigned>(blocks), lsq::kBatchThreads, 0, st>>>(
            d_xy, n_curves, ppc, coeffs, status);
    else
        lsq::batched_fit_kernel<M, false><<<static_cast<unsigned>(blocks), lsq::kBatchThreads, 0, st>>>(
            d_xy, n_curves, ppc, coeffs, status);
    return cudaGetLastError();
}


#define LSQ_DISPATCH(fn, degree, ...)                 \
    [&]() -> cudaError_t {                            \
        switch (degree) {                             \
            case 0: return fn<0>(__VA_ARGS__);        \
            case 1: return fn<1>(__VA_ARGS__);        \
            case 2: return fn<2>(__VA_ARGS__);        \
            case 3: return fn<3>(__VA_ARGS__);        \
            case 4: return fn<4>(__VA_ARGS__);        \
            case 5: return fn<5>(__VA_ARGS__);        \
            case 6: return fn<6>(__VA_ARGS__);        \
            case 7: return fn<7>(__VA_ARGS__);        \
            case 8: return fn<8>(__VA_ARGS__);        \
            case 9: return fn<9>(__VA_ARGS__);        \
            case 10: return fn<10>(__VA_ARGS__);      \
            case 11: return fn<11>(__VA_ARGS__);      \
            case 12: return fn<12>(__VA_ARGS__);      \
            default: return cudaErrorInvalidValue;    \
        }                                             \
    }()

template <int M>
cudaError_t launch_diag(lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n, const double* coeffs,
                        const int32_t* gate, double* residuals, lsqfit_diag* out, cudaStream_t st) {
    uint64_t blocks = (n + lsq::kDiagThreads * 4 - 1) / (lsq::kDiagThreads * 4);
    if (blocks > uint64_t(ctx->diag_ctas)) blocks = ctx->diag_ctas;
    if (blocks < 1) blocks = 1;
    lsq::diagnostics_kernel<M><<<static_cast<unsigned>(blocks), lsq::kDiagThreads, 0, st>>>(
        reinterpret_cast<const double2*>(d_xy), n, coeffs, gate, residuals, ctx->d_dslots, ctx->d_dticket, out);
    return cudaGetLastError();
}

#define LSQ_DISPATCH_QR(fn, degree, ...)              \
    [&]() -> cudaError_t {                            \
        switch (degree) {                             \
            case 0: return fn<0>(__VA_ARGS__);        \
            case 1: return fn<1>(__VA_ARGS__);        \
            case 2: return fn<2>(__VA_ARGS__);        \
            case 3: return fn<3>(__VA_ARGS__);        \
            case 4: return fn<4>(__VA_ARGS__);        \
            case 5: return fn<5>(__VA_ARGS__);        \
            case 6: return fn<6>(__VA_ARGS__);        \
            case 7: return fn<7>(__VA_ARGS__);        \
            case 8: return fn<8>(__VA_ARGS__);        \
            default: return cudaErrorInvalidValue;    \
        }                                             \
    }()

template <int M>
cudaError_t configure_qr(int sm_count, int* ctas) {
    using Q = lsq::QrCfg<M>;
    cudaError_t e = cudaFuncSetAttribute(lsq::qr_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(Q::SMEM));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lsq::qr_kernel<M>, Q::THREADS, Q::SMEM);
    if (e != cudaSuccess) return e;
    *ctas = sm_count * (per_sm > 0 ? per_sm : 1);
    return cudaSuccess;
}

template <int M>
cudaError_t launch_qr(lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n, unsigned flags, lsqfit_qr_result* out,
                      cudaStream_t st) {
    using Q = lsq::QrCfg<M>;
    lsq::QrArgs a{reinterpret_cast<const double2*>(d_xy), n, ctx->d_qslots, ctx->d_qbad, ctx->d_qticket, out, flags};
    lsq::qr_kernel<M><<<ctx->qr_ctas[M], Q::THREADS, Q::SMEM, st>>>(a);
    return cudaGetLastError();
}

template <int M>
cudaError_t launch_qr_combine(const lsqfit_qr_result* parts, int count, unsigned flags, lsqfit_qr_result* out,
                              cudaStream_t st) {
    lsq::qr_combine_kernel<M><<<1, 32, 0, st>>>(parts, count, flags, out);
    return cudaGetLastError();
}

cudaError_t grow(double** buf, size_t* cap, size_t bytes) {
    if (bytes <= *cap) return cudaSuccess;
    cudaFree(*buf);
    *buf = nullptr;
    *cap = 0;
    const cudaError_t e = cudaMalloc(buf, bytes);
    if (e == cudaSuccess) *cap = bytes;
    return e;
}

__global__ void solve_kernel(const double* a, const double* b, int dim, double* x, int* status) {
    extern __shared__ double sm[];
    double* A = sm;
    double* B = A + dim * dim;
    double* X = B + dim;
    for (int i = threadIdx.x; i < dim * dim; i += 32) A[i] = a[i];
    for (int i = threadIdx.x; i < dim; i += 32) B[i] = b[i];
    __syncwarp();
    const int st = lsq::warp_solve_gaussian(A, B, X, dim);
    for (int i = threadIdx.x; i < dim; i += 32) x[i] = X[i];
    if (threadIdx.x == 0) *status = st;
}

int check_degree(int degree) {
    if (degree < 0) return LSQFIT_EINVAL;
    if (degree > LSQFIT_MAX_DEGREE) return LSQFIT_EINVAL;
    return LSQFIT_OK;
}

// ---------------------------------------------------------------------------
// Host-resident inputs: one H2D + one launch when the points fit in one
// streaming chunk; otherwise out of core — chunks double-buffered through two
// device buffers, H2D on a copy stream overlapped with the per-chunk kernels
// on ctx->stream, partial records combined in chunk order.
// ---------------------------------------------------------------------------

cudaError_t grow_raw(void** buf, size_t* cap, size_t bytes) {
    return grow(reinterpret_cast<double**>(buf), cap, bytes);
}

uint64_t n_chunks(const lsqfit_cuda_ctx* ctx, uint64_t n) { return (n + ctx->chunk_points - 1) / ctx->chunk_points; }

// Run fn(k, d_points, count) on ctx->stream for every chunk k of the host array.
template <class F>
cudaError_t stream_points(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, F&& fn) {
    const uint64_t C = ctx->chunk_points;
    const uint64_t K = n_chunks(ctx, n);
    if (K == 1) {
        cudaError_t e = grow(&ctx->d_buf, &ctx->buf_bytes, size_t(n) * 16);
        if (e != cudaSuccess) return e;
        e = ctx->stager.h2d(ctx->d_buf, xy, size_t(n) * 16, ctx->stream);
        if (e != cudaSuccess) return e;
        return fn(uint64_t(0), static_cast<const double*>(ctx->d_buf), n);
    }
    for (int b = 0; b < 2; ++b) {
        const cudaError_t e = grow(&ctx->d_sbuf[b], &ctx->sbuf_bytes[b], size_t(C) * 16);
        if (e != cudaSuccess) return e;
    }
    for (uint64_t k = 0; k < K; ++k) {
        const int b = int(k & 1);
        const uint64_t lo = k * C;
        const uint64_t cnt = (n - lo < C) ? (n - lo) : C;
        cudaError_t e;
        if (k >= 2 && (e = cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_consumed[b], 0)) != cudaSuccess) return e;
        if ((e = ctx->stager.h2d(ctx->d_sbuf[b], xy + 2 * lo, size_t(cnt) * 16, ctx->copy_stream)) != cudaSuccess)
            return e;
        if ((e = cudaEventRecord(ctx->ev_copied[b], ctx->copy_stream)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(ctx->stream, ctx->ev_copied[b], 0)) != cudaSuccess) return e;
        if ((e = fn(k, static_cast<const double*>(ctx->d_sbuf[b]), cnt)) != cudaSuccess) return e;
        if ((e = cudaEventRecord(ctx->ev_consumed[b], ctx->stream)) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// Sums (+ solve per flags) of host points into ctx->d_result.
cudaError_t enqueue_fit(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, int degree, unsigned flags) {
    const uint64_t K = n_chunks(ctx, n);
    if (K == 1)
        return stream_points(ctx, xy, n, [&](uint64_t, const double* d, uint64_t cnt) {
            return LSQ_DISPATCH(launch_ps, degree, ctx, d, cnt, flags, ctx->d_result, ctx->stream);
        });
    cudaError_t e = grow_raw(reinterpret_cast<void**>(&ctx->d_recs), &ctx->recs_bytes, size_t(K) * sizeof(lsqfit_result));
    if (e != cudaSuccess) return e;
    e = stream_points(ctx, xy, n, [&](uint64_t k, const double* d, uint64_t cnt) {
        return LSQ_DISPATCH(launch_ps, degree, ctx, d, cnt, LSQFIT_SUMS, ctx->d_recs + k, ctx->stream);
    });
    if (e != cudaSuccess) return e;
    return LSQ_DISPATCH(launch_combine, degree, ctx->d_recs, static_cast<int>(K), flags, ctx->d_result, ctx->stream);
}

// Diagnostics pass of host points against device coefficients into ctx->d_diag;
// residuals (host, n doubles) copied back chunk by chunk when requested.
cudaError_t enqueue_report(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, int degree, const double* d_coeffs,
                           const int32_t* d_gate, double* residuals) {
    const uint64_t K = n_chunks(ctx, n);
    const uint64_t C = K == 1 ? n : ctx->chunk_points;
    cudaError_t e;
    if (residuals && (e = grow(&ctx->d_res, &ctx->res_bytes, size_t(C) * sizeof(double) * (K == 1 ? 1 : 2))) !=
                         cudaSuccess)
        return e;
    if (K > 1 && (e = grow_raw(reinterpret_cast<void**>(&ctx->d_drecs), &ctx->drecs_bytes,
                               size_t(K) * sizeof(lsqfit_diag))) != cudaSuccess)
        return e;
    e = stream_points(ctx, xy, n, [&](uint64_t k, const double* d, uint64_t cnt) {
        double* d_res = residuals ? ctx->d_res + (K == 1 ? 0 : (k & 1) * C) : nullptr;
        lsqfit_diag* out = K == 1 ? ctx->d_diag : ctx->d_drecs + k;
        cudaError_t e2 = LSQ_DISPATCH(launch_diag, degree, ctx, d, cnt, d_coeffs, d_gate, d_res, out, ctx->stream);
        if (e2 == cudaSuccess && residuals)
            e2 = ctx->stager.d2h(residuals + k * C, d_res, size_t(cnt) * sizeof(double), ctx->stream);
        return e2;
    });
    if (e != cudaSuccess || K == 1) return e;
    lsq::diag_combine_kernel<<<1, 32, 0, ctx->stream>>>(ctx->d_drecs, static_cast<int>(K), ctx->d_diag);
    return cudaGetLastError();
}

}  // namespace

extern "C" {

const char* lsqfit_cuda_strerror(int status) {
    switch (status) {
        case LSQFIT_OK: return "ok";
        case LSQFIT_EINVAL: return "invalid argument";
        case LSQFIT_EOVERFLOW: return "non-finite power sums or coefficients (overflow)";
        case LSQFIT_ESINGULAR: return "singular normal system";
        case LSQFIT_EDEGREE: return "degree exceeds the supported cap";
        case LSQFIT_ECUDA: return "CUDA runtime error";
        case LSQFIT_ENOMEM: return "device memory allocation failed";
        case LSQFIT_ERANKDEF: return "rank-deficient system (fewer than degree+1 distinct x values)";
        default: return "unknown status";
    }
}

const char* lsqfit_cuda_last_error(lsqfit_cuda_ctx* ctx) { return ctx ? ctx->last_error : ""; }

int lsqfit_cuda_create(lsqfit_cuda_ctx** out, int device) {
    if (!out) return LSQFIT_EINVAL;
    *out = nullptr;
    lsqfit_cuda_ctx* ctx = new (std::nothrow) lsqfit_cuda_ctx();
    if (!ctx) return LSQFIT_ENOMEM;
    auto fail = [&](cudaError_t e) {
        const int st = record(ctx, e);
        std::fprintf(stderr, "lsqfit_cuda_create: %s\n", ctx->last_error);
        lsqfit_cuda_destroy(ctx);
        return st;
    };
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return fail(e);
    ctx->device = device;
    e = cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return fail(e);
    int cfg[LSQFIT_MAX_DEGREE + 2];
    int max_ctas = 0;
    for (int m = 0; m <= LSQFIT_MAX_DEGREE; ++m) {
        e = LSQ_DISPATCH(configure_ps, m, ctx->sm_count, cfg);
        if (e != cudaSuccess) return fail(e);
        ctx->ps_ctas[m] = cfg[0];
        ctx->batch_ctas[m] = cfg[LSQFIT_MAX_DEGREE + 1];
        if (cfg[0] > max_ctas) max_ctas = cfg[0];
    }
    if ((e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking)) != cudaSuccess) return fail(e);
    if ((e = cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking)) != cudaSuccess) return fail(e);
    for (int b = 0; b < 2; ++b) {
        if ((e = cudaEventCreateWithFlags(&ctx->ev_copied[b], cudaEventDisableTiming)) != cudaSuccess) return fail(e);
        if ((e = cudaEventCreateWithFlags(&ctx->ev_consumed[b], cudaEventDisableTiming)) != cudaSuccess) return fail(e);
    }
    ctx->chunk_points = kDefaultStreamChunk;
    if ((e = cudaMalloc(&ctx->d_slots, sizeof(double2) * size_t(max_ctas) * LSQFIT_MAX_NV)) != cudaSuccess)
        return fail(e);
    if ((e = cudaMalloc(&ctx->d_ticket, sizeof(unsigned))) != cudaSuccess) return fail(e);
    if ((e = cudaMemset(ctx->d_ticket, 0, sizeof(unsigned))) != cudaSuccess) return fail(e);
    if ((e = cudaMalloc(&ctx->d_result, sizeof(lsqfit_result))) != cudaSuccess) return fail(e);
    if ((e = cudaMallocHost(&ctx->h_result, sizeof(lsqfit_result))) != cudaSuccess) return fail(e);
    ctx->diag_ctas = ctx->sm_count * 8;
    if ((e = cudaMalloc(&ctx->d_dslots, sizeof(double2) * size_t(ctx->diag_ctas) * 4)) != cudaSuccess) return fail(e);
    if ((e = cudaMalloc(&ctx->d_dticket, sizeof(unsigned))) != cudaSuccess) return fail(e);
    if ((e = cudaMemset(ctx->d_dticket, 0, sizeof(unsigned))) != cudaSuccess) return fail(e);
    if ((e = cudaMalloc(&ctx->d_diag, sizeof(lsqfit_diag))) != cudaSuccess) return fail(e);
    if ((e = cudaMallocHost(&ctx->h_diag, sizeof(lsqfit_diag))) != cudaSuccess) return fail(e);
    int max_q = 0;
    for (int m = 0; m <= LSQFIT_MAX_QR_DEGREE; ++m) {
        e = LSQ_DISPATCH_QR(configure_qr, m, ctx->sm_count, &ctx->qr_ctas[m]);
        if (e != cudaSuccess) return fail(e);
        if (ctx->qr_ctas[m] > max_q) max_q = ctx->qr_ctas[m];
    }
    if ((e = cudaMalloc(&ctx->d_qslots, sizeof(double) * size_t(max_q) * 55)) != cudaSuccess) return fail(e);
    if ((e = cudaMalloc(&ctx->d_qbad, sizeof(int) * size_t(max_q))) != cudaSuccess) return fail(e);
    if ((e = cudaMalloc(&ctx->d_qticket, sizeof(unsigned))) != cudaSuccess) return fail(e);
    if ((e = cudaMemset(ctx->d_qticket, 0, sizeof(unsigned))) != cudaSuccess) return fail(e);
    if ((e = cudaMalloc(&ctx->d_qresult, sizeof(lsqfit_qr_result))) != cudaSuccess) return fail(e);
    if ((e = cudaMallocHost(&ctx->h_qresult, sizeof(lsqfit_qr_result))) != cudaSuccess) return fail(e);
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return fail(e);
    *out = ctx;
    return LSQFIT_OK;
}

void lsqfit_cuda_destroy(lsqfit_cuda_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    cudaFree(ctx->d_slots);
    cudaFree(ctx->d_ticket);
    cudaFree(ctx->d_qslots);
    cudaFree(ctx->d_qbad);
    cudaFree(ctx->d_qticket);
    cudaFree(ctx->d_qresult);
    cudaFree(ctx->d_qrecs);
    if (ctx->h_qresult) cudaFreeHost(ctx->h_qresult);
    cudaFree(ctx->d_result);
    cudaFree(ctx->d_buf);
    cudaFree(ctx->d_dslots);
    cudaFree(ctx->d_dticket);
    cudaFree(ctx->d_diag);
    cudaFree(ctx->d_res);
    if (ctx->h_diag) cudaFreeHost(ctx->h_diag);
    if (ctx->h_result) cudaFreeHost(ctx->h_result);
    if (ctx->copy_stream) cudaStreamSynchronize(ctx->copy_stream);
    for (int b = 0; b < 2; ++b) {
        cudaFree(ctx->d_sbuf[b]);
        if (ctx->ev_copied[b]) cudaEventDestroy(ctx->ev_copied[b]);
        if (ctx->ev_consumed[b]) cudaEventDestroy(ctx->ev_consumed[b]);
    }
    cudaFree(ctx->d_recs);
    cudaFree(ctx->d_drecs);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

int lsqfit_cuda_grid_size(lsqfit_cuda_ctx* ctx, int* ctas) {
    if (!ctx || !ctas) return LSQFIT_EINVAL;
    *ctas = ctx->ps_ctas[3];
    return LSQFIT_OK;
}

int lsqfit_cuda_fit_device(lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n, int degree, unsigned flags,
                           lsqfit_result* d_result, void* stream) {
    if (!ctx || !d_result || (n > 0 && !d_xy)) return LSQFIT_EINVAL;
    if (check_degree(degree) != LSQFIT_OK) return LSQFIT_EINVAL;
    if (reinterpret_cast<uintptr_t>(d_xy) % 16 != 0) return LSQFIT_EINVAL;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    LSQ_TRY(ctx, LSQ_DISPATCH(launch_ps, degree, ctx, d_xy, n, flags, d_result, st));
    return LSQFIT_OK;
}

int lsqfit_cuda_combine_device(lsqfit_cuda_ctx* ctx, const lsqfit_result* d_parts, int n_parts, int degree,
                               unsigned flags, lsqfit_result* d_result, void* stream) {
    if (!ctx || !d_parts || !d_result || n_parts < 1) return LSQFIT_EINVAL;
    if (check_degree(degree) != LSQFIT_OK) return LSQFIT_EINVAL;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    LSQ_TRY(ctx, LSQ_DISPATCH(launch_combine, degree, d_parts, n_parts, flags, d_result, st));
    return LSQFIT_OK;
}

int lsqfit_cuda_set_stream_chunk(lsqfit_cuda_ctx* ctx, uint64_t points) {
    if (!ctx) return LSQFIT_EINVAL;
    std::lock_guard<std::mutex> lock(ctx->mu);
    ctx->chunk_points = points ? points : kDefaultStreamChunk;
    return LSQFIT_OK;
}

int lsqfit_cuda_fit_host(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, int degree, unsigned flags,
                         lsqfit_result* result) {
    if (!ctx || !result || !xy || n == 0) return LSQFIT_EINVAL;
    if (check_degree(degree) != LSQFIT_OK) return LSQFIT_EINVAL;
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, cudaSetDevice(ctx->device));
    LSQ_TRY(ctx, enqueue_fit(ctx, xy, n, degree, flags));
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
    LSQ_TRY(ctx, enqueue_fit(ctx, xy, n, degree, LSQFIT_SOLVE));
    // second pass over the (re-streamed) points: residuals, SSE, R
    LSQ_TRY(ctx, enqueue_report(ctx, xy, n, degree, ctx->d_result->coeffs, &ctx->d_result->status, residuals));
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
    if (check_degree(degree) != LSQFIT_OK) return LSQFIT_EINVAL;
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, cudaSetDevice(ctx->device));
    double* d_coeffs = ctx->d_result->coeffs;  // ctx-owned scratch (held under ctx->mu)
    LSQ_TRY(ctx, cudaMemcpyAsync(d_coeffs, coeffs, sizeof(double) * (degree + 1), cudaMemcpyHostToDevice,
                                 ctx->stream));
    LSQ_TRY(ctx, enqueue_report(ctx, xy, n, degree, d_coeffs, nullptr, residuals));
    LSQ_TRY(ctx, cudaMemcpyAsync(ctx->h_diag, ctx->d_diag, sizeof(lsqfit_diag), cudaMemcpyDeviceToHost, ctx->stream));
    LSQ_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    std::memcpy(diag, ctx->h_diag, sizeof(lsqfit_diag));
    return diag->status;
}

int lsqfit_cuda_fit_batched_host(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n_curves,
                                 uint32_t points_per_curve, int degree, double* coeffs, int32_t* status) {
    if (!ctx || !xy || !coeffs || !status || points_per_curve == 0) return LSQFIT_EINVAL;
    if (check_degree(degree) != LSQFIT_OK) return LSQFIT_EINVAL;
    if (n_curves == 0) return LSQFIT_OK;
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, cudaSetDevice(ctx->device));
    const size_t in_bytes = size_t(n_curves) * points_per_curve * 16;
    const size_t c_bytes = size_t(n_curves) * (degree + 1) * sizeof(double);
    const size_t s_bytes = size_t(n_curves) * sizeof(int32_t);
    LSQ_TRY(ctx, grow(&ctx->d_buf, &ctx->buf_bytes, in_bytes));
    LSQ_TRY(ctx, grow(&ctx->d_res, &ctx->res_bytes, c_bytes + s_bytes + 16));
    double* d_coeffs = ctx->d_res;
    int32_t* d_status = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(ctx->d_res) + ((c_bytes + 15) & ~size_t(15)));
    LSQ_TRY(ctx, ctx->stager.h2d(ctx->d_buf, xy, in_bytes, ctx->stream));
    LSQ_TRY(ctx, LSQ_DISPATCH(launch_batched, degree, ctx, ctx->d_buf, n_curves, points_per_curve, d_coeffs, d_status,
                              ctx->stream));
    LSQ_TRY(ctx, cudaMemcpyAsync(coeffs, d_coeffs, c_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    LSQ_TRY(ctx, cudaMemcpyAsync(status, d_status, s_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    LSQ_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return LSQFIT_OK;
}

int lsqfit_cuda_diagnostics_device(lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n, int degree,
                                   const double* d_coeffs, const int32_t* d_gate, double* d_residuals,
                                   lsqfit_diag* d_out, void* stream) {
    if (!ctx || !d_coeffs || !d_out || n == 0 || !d_xy) return LSQFIT_EINVAL;
    if (check_degree(degree) != LSQFIT_OK) return LSQFIT_EINVAL;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    LSQ_TRY(ctx, LSQ_DISPATCH(launch_diag, degree, ctx, d_xy, n, d_coeffs, d_gate, d_residuals, d_out, st));
    return LSQFIT_OK;
}

int lsqfit_cuda_qr_fit_device(lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n, int degree, unsigned flags,
                              lsqfit_qr_result* d_result, void* stream) {
    if (!ctx || !d_result || (n > 0 && !d_xy)) return LSQFIT_EINVAL;
    if (degree < 0 || degree > LSQFIT_MAX_QR_DEGREE) return LSQFIT_EINVAL;
    if (reinterpret_cast<uintptr_t>(d_xy) % 16 != 0) return LSQFIT_EINVAL;
    LSQ_TRY(ctx, LSQ_DISPATCH_QR(launch_qr, degree, ctx, d_xy, n, flags, d_result, static_cast<cudaStream_t>(stream)));
    return LSQFIT_OK;
}

int lsqfit_cuda_qr_combine_device(lsqfit_cuda_ctx* ctx, const lsqfit_qr_result* d_parts, int n_parts, int degree,
                                  unsigned flags, lsqfit_qr_result* d_result, void* stream) {
    if (!ctx || !d_parts || !d_result || n_parts < 1) return LSQFIT_EINVAL;
    if (degree < 0 || degree > LSQFIT_MAX_QR_DEGREE) return LSQFIT_EINVAL;
    LSQ_TRY(ctx, LSQ_DISPATCH_QR(launch_qr_combine, degree, d_parts, n_parts, flags, d_result,
                                 static_cast<cudaStream_t>(stream)));
    return LSQFIT_OK;
}

int lsqfit_cuda_qr_fit_host(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, int degree, lsqfit_qr_result* result) {
    if (!ctx || !result || !xy || n == 0) return LSQFIT_EINVAL;
    if (degree < 0 || degree > LSQFIT_MAX_QR_DEGREE) return LSQFIT_EINVAL;
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, cudaSetDevice(ctx->device));
    const uint64_t K = n_chunks(ctx, n);
    if (K == 1) {
        LSQ_TRY(ctx, stream_points(ctx, xy, n, [&](uint64_t, const double* d, uint64_t cnt) {
                    return LSQ_DISPATCH_QR(launch_qr, degree, ctx, d, cnt, LSQFIT_SOLVE, ctx->d_qresult, ctx->stream);
                }));
    } else {
        LSQ_TRY(ctx, grow_raw(reinterpret_cast<void**>(&ctx->d_qrecs), &ctx->qrecs_bytes,
                              size_t(K) * sizeof(lsqfit_qr_result)));
        LSQ_TRY(ctx, stream_points(ctx, xy, n, [&](uint64_t k, const double* d, uint64_t cnt) {
                    return LSQ_DISPATCH_QR(launch_qr, degree, ctx, d, cnt, LSQFIT_SUMS, ctx->d_qrecs + k, ctx->stream);
                }));
        LSQ_TRY(ctx, LSQ_DISPATCH_QR(launch_qr_combine, degree, ctx->d_qrecs, static_cast<int>(K), LSQFIT_SOLVE,
                                     ctx->d_qresult, ctx->stream));
    }
    LSQ_TRY(ctx, cudaMemcpyAsync(ctx->h_qresult, ctx->d_qresult, sizeof(lsqfit_qr_result), cudaMemcpyDeviceToHost,
                                 ctx->stream));
    LSQ_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    std::memcpy(result, ctx->h_qresult, sizeof(lsqfit_qr_result));
    return result->status;
}

int lsqfit_cuda_solve_host(lsqfit_cuda_ctx* ctx, const double* a, const double* b, int dim, double* x) {
    if (!ctx || !a || !b || !x) return LSQFIT_EINVAL;
    if (dim < 1 || dim > LSQFIT_MAX_SOLVE_DIM) return LSQFIT_EINVAL;
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, cudaSetDevice(ctx->device));
    const size_t na = size_t(dim) * dim;
    const size_t bytes = (na + 2 * size_t(dim)) * sizeof(double) + sizeof(int);
    LSQ_TRY(ctx, grow(&ctx->d_buf, &ctx->buf_bytes, bytes));
    double* da = ctx->d_buf;
    double* db = da + na;
    double* dx = db + dim;
    int* dst = reinterpret_cast<int*>(dx + dim);
    LSQ_TRY(ctx, cudaMemcpyAsync(da, a, na * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    LSQ_TRY(ctx, cudaMemcpyAsync(db, b, dim * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    const size_t smem = (na + 2 * size_t(dim)) * sizeof(double);
    if (smem > 48 * 1024)
        LSQ_TRY(ctx, cudaFuncSetAttribute(solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(smem)));
    solve_kernel<<<1, 32, smem, ctx->stream>>>(da, db, dim, dx, dst);
    LSQ_TRY(ctx, cudaGetLastError());
    int status = 0;
    LSQ_TRY(ctx, cudaMemcpyAsync(x, dx, dim * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    LSQ_TRY(ctx, cudaMemcpyAsync(&status, dst, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    LSQ_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return status;
}

int lsqfit_cuda_fit_batched_device(lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n_curves,
                                   uint32_t points_per_curve, int degree, double* d_coeffs, int32_t* d_status,
                                   void* stream) {
    if (!ctx || !d_coeffs || !d_status || (n_curves > 0 && !d_xy) || points_per_curve == 0) return LSQFIT_EINVAL;
    if (check_degree(degree) != LSQFIT_OK) return LSQFIT_EINVAL;
    if (reinterpret_cast<uintptr_t>(d_xy) % 16 != 0) return LSQFIT_EINVAL;
    if (n_curves == 0) return LSQFIT_OK;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    LSQ_TRY(ctx, LSQ_DISPATCH(launch_batched, degree, ctx, d_xy, n_curves, points_per_curve, d_coeffs, d_status, st));
    return LSQFIT_OK;
}

int lsqfit_cuda_synth_device(lsqfit_cuda_ctx* ctx, double* d_xy, uint64_t n, uint64_t offset, uint64_t seed,
                             int truth_degree, double sigma, void* stream) {
    if (!ctx || (n > 0 && !d_xy) || truth_degree < 0 || truth_degree > LSQFIT_MAX_DEGREE) return LSQFIT_EINVAL;
    if (n == 0) return LSQFIT_OK;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint64_t blocks = (n + 255) / 256;
    const uint64_t cap = uint64_t(ctx->sm_count) * 16;
    if (blocks > cap) blocks = cap;
    lsq::synth_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(reinterpret_cast<double2*>(d_xy), n, offset,
                                                                      seed, truth_degree, sigma);
    LSQ_TRY(ctx, cudaGetLastError());
    return LSQFIT_OK;
}

int lsqfit_cuda_synth_batched_device(lsqfit_cuda_ctx* ctx, double* d_xy, uint64_t n_curves,
                                     uint32_t points_per_curve, uint64_t seed, int truth_degree, double sigma,
                                     void* stream) {
    if (!ctx || (n_curves > 0 && !d_xy) || truth_degree < 0 || truth_degree > LSQFIT_MAX_DEGREE) return LSQFIT_EINVAL;
    if (n_curves == 0 || points_per_curve == 0) return LSQFIT_OK;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint64_t blocks = (n_curves * 32 + 255) / 256;
    const uint64_t cap = uint64_t(ctx->sm_count) * 16;
    if (blocks > cap) blocks = cap;
    lsq::synth_batched_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(
        reinterpret_cast<double2*>(d_xy), n_curves, points_per_curve, seed, truth_degree, sigma);
    LSQ_TRY(ctx, cudaGetLastError());
    return LSQFIT_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Device groups: one host dataset sharded over G GPUs of this process. Each
// GPU streams its contiguous shard [n*g/G, n*(g+1)/G) over its own PCIe link
// into its own context; the G partial records (1 KB each) come back to the
// host and are combined, in ascending device order, on the first device.
// ---------------------------------------------------------------------------

struct lsqfit_cuda_group {
    std::vector<lsqfit_cuda_ctx*> ctx;
    lsqfit_result* h_parts = nullptr;  // pinned [G]
    lsqfit_diag* h_dparts = nullptr;   // pinned [G]
    lsqfit_result* d_parts = nullptr;  // on ctx[0]
    lsqfit_diag* d_dparts = nullptr;   // on ctx[0]
    std::mutex mu;
};

namespace {

template <class F>
int group_run(lsqfit_cuda_group* g, F&& per_device) {
    const int G = static_cast<int>(g->ctx.size());
    std::vector<int> st(G, LSQFIT_OK);
    std::vector<std::thread> th;
    for (int d = 1; d < G; ++d) th.emplace_back([&, d] { st[d] = per_device(d); });
    st[0] = per_device(0);
    for (auto& t : th) t.join();
    for (int d = 0; d < G; ++d)
        if (st[d] != LSQFIT_OK) return st[d];
    return LSQFIT_OK;
}

// Sums of shard d into g->h_parts[d] (an empty record for an empty shard).
int group_shard_sums(lsqfit_cuda_group* g, int d, const double* xy, uint64_t n, int degree) {
    const int G = static_cast<int>(g->ctx.size());
    lsqfit_cuda_ctx* c = g->ctx[d];
    const uint64_t lo = n * uint64_t(d) / G, hi = n * uint64_t(d + 1) / G;
    if (hi == lo) {
        std::memset(&g->h_parts[d], 0, sizeof(lsqfit_result));
        g->h_parts[d].degree = degree;
        return LSQFIT_OK;
    }
    std::lock_guard<std::mutex> lock(c->mu);
    LSQ_TRY(c, cudaSetDevice(c->device));
    LSQ_TRY(c, enqueue_fit(c, xy + 2 * lo, hi - lo, degree, LSQFIT_SUMS));
    LSQ_TRY(c, cudaMemcpyAsync(&g->h_parts[d], c->d_result, sizeof(lsqfit_result), cudaMemcpyDeviceToHost, c->stream));
    LSQ_TRY(c, cudaStreamSynchronize(c->stream));
    return LSQFIT_OK;
}

// Combine the host records on device 0 into ctx[0]->d_result.
int group_combine(lsqfit_cuda_group* g, int degree, unsigned flags) {
    lsqfit_cuda_ctx* c = g->ctx[0];
    const int G = static_cast<int>(g->ctx.size());
    LSQ_TRY(c, cudaSetDevice(c->device));
    LSQ_TRY(c, cudaMemcpyAsync(g->d_parts, g->h_parts, sizeof(lsqfit_result) * G, cudaMemcpyHostToDevice, c->stream));
    LSQ_TRY(c, LSQ_DISPATCH(launch_combine, degree, g->d_parts, G, flags, c->d_result, c->stream));
    return LSQFIT_OK;
}

}  // namespace

extern "C" {

int lsqfit_cuda_group_create(lsqfit_cuda_group** out, const int* devices, int count) {
    if (!out || !devices || count < 1 || count > 64) return LSQFIT_EINVAL;
    *out = nullptr;
    lsqfit_cuda_group* g = new (std::nothrow) lsqfit_cuda_group();
    if (!g) return LSQFIT_ENOMEM;
    for (int d = 0; d < count; ++d) {
        lsqfit_cuda_ctx* c = nullptr;
        const int st = lsqfit_cuda_create(&c, devices[d]);
        if (st != LSQFIT_OK) {
            lsqfit_cuda_group_destroy(g);
            return st;
        }
        g->ctx.push_back(c);
    }
    lsqfit_cuda_ctx* c0 = g->ctx[0];
    cudaSetDevice(c0->device);
    if (cudaMallocHost(&g->h_parts, sizeof(lsqfit_result) * count) != cudaSuccess ||
        cudaMallocHost(&g->h_dparts, sizeof(lsqfit_diag) * count) != cudaSuccess ||
        cudaMalloc(&g->d_parts, sizeof(lsqfit_result) * count) != cudaSuccess ||
        cudaMalloc(&g->d_dparts, sizeof(lsqfit_diag) * count) != cudaSuccess) {
        lsqfit_cuda_group_destroy(g);
        return LSQFIT_ENOMEM;
    }
    *out = g;
    return LSQFIT_OK;
}

void lsqfit_cuda_group_destroy(lsqfit_cuda_group* g) {
    if (!g) return;
    if (!g->ctx.empty()) {
        cudaSetDevice(g->ctx[0]->device);
        cudaFree(g->d_parts);
        cudaFree(g->d_dparts);
    }
    if (g->h_parts) cudaFreeHost(g->h_parts);
    if (g->h_dparts) cudaFreeHost(g->h_dparts);
    for (lsqfit_cuda_ctx* c : g->ctx) lsqfit_cuda_destroy(c);
    delete g;
}

int lsqfit_cuda_group_size(lsqfit_cuda_group* g) { return g ? static_cast<int>(g->ctx.size()) : 0; }

int lsqfit_cuda_group_fit_host(lsqfit_cuda_group* g, const double* xy, uint64_t n, int degree, unsigned flags,
                               lsqfit_result* result) {
    if (!g || !xy || !result || n == 0) return LSQFIT_EINVAL;
    if (check_degree(degree) != LSQFIT_OK) return LSQFIT_EINVAL;
    std::lock_guard<std::mutex> glock(g->mu);
    int st = group_run(g, [&](int d) { return group_shard_sums(g, d, xy, n, degree); });
    if (st != LSQFIT_OK) return st;
    lsqfit_cuda_ctx* c = g->ctx[0];
    std::lock_guard<std::mutex> lock(c->mu);
    if ((st = group_combine(g, degree, flags)) != LSQFIT_OK) return st;
    LSQ_TRY(c, cudaMemcpyAsync(c->h_result, c->d_result, sizeof(lsqfit_result), cudaMemcpyDeviceToHost, c->stream));
    LSQ_TRY(c, cudaStreamSynchronize(c->stream));
    std::memcpy(result, c->h_result, sizeof(lsqfit_result));
    return result->status;
}

int lsqfit_cuda_group_fit_report_host(lsqfit_cuda_group* g, const double* xy, uint64_t n, int degree,
                                      lsqfit_result* result, lsqfit_diag* diag, double* residuals) {
    if (!g || !xy || !result || !diag || n == 0) return LSQFIT_EINVAL;
    if (check_degree(degree) != LSQFIT_OK) return LSQFIT_EINVAL;
    std::lock_guard<std::mutex> glock(g->mu);
    const int G = static_cast<int>(g->ctx.size());
    int st = group_run(g, [&](int d) { return group_shard_sums(g, d, xy, n, degree); });
    if (st != LSQFIT_OK) return st;
    lsqfit_cuda_ctx* c0 = g->ctx[0];
    {
        std::lock_guard<std::mutex> lock(c0->mu);
        if ((st = group_combine(g, degree, LSQFIT_SOLVE)) != LSQFIT_OK) return st;
        LSQ_TRY(c0, cudaMemcpyAsync(c0->h_result, c0->d_result, sizeof(lsqfit_result), cudaMemcpyDeviceToHost,
                                    c0->stream));
        LSQ_TRY(c0, cudaStreamSynchronize(c0->stream));
        std::memcpy(result, c0->h_result, sizeof(lsqfit_result));
    }
    if (result->status != LSQFIT_OK) return result->status;
    // diagnostics pass: every device evaluates its shard against the coefficients
    st = group_run(g, [&](int d) -> int {
        lsqfit_cuda_ctx* c = g->ctx[d];
        const uint64_t lo = n * uint64_t(d) / G, hi = n * uint64_t(d + 1) / G;
        if (hi == lo) {
            std::memset(&g->h_dparts[d], 0, sizeof(lsqfit_diag));
            return LSQFIT_OK;
        }
        std::lock_guard<std::mutex> lock(c->mu);
        LSQ_TRY(c, cudaSetDevice(c->device));
        double* d_coeffs = c->d_result->coeffs;
        LSQ_TRY(c, cudaMemcpyAsync(d_coeffs, result->coeffs, sizeof(double) * (degree + 1), cudaMemcpyHostToDevice,
                                   c->stream));
        LSQ_TRY(c, enqueue_report(c, xy + 2 * lo, hi - lo, degree, d_coeffs, nullptr,
                                  residuals ? residuals + lo : nullptr));
        LSQ_TRY(c, cudaMemcpyAsync(&g->h_dparts[d], c->d_diag, sizeof(lsqfit_diag), cudaMemcpyDeviceToHost, c->stream));
        LSQ_TRY(c, cudaStreamSynchronize(c->stream));
        return LSQFIT_OK;
    });
    if (st != LSQFIT_OK) return st;
    std::lock_guard<std::mutex> lock(c0->mu);
    LSQ_TRY(c0, cudaSetDevice(c0->device));
    LSQ_TRY(c0, cudaMemcpyAsync(g->d_dparts, g->h_dparts, sizeof(lsqfit_diag) * G, cudaMemcpyHostToDevice, c0->stream));
    lsq::diag_combine_kernel<<<1, 32, 0, c0->stream>>>(g->d_dparts, G, c0->d_diag);
    LSQ_TRY(c0, cudaGetLastError());
    LSQ_TRY(c0, cudaMemcpyAsync(c0->h_diag, c0->d_diag, sizeof(lsqfit_diag), cudaMemcpyDeviceToHost, c0->stream));
    LSQ_TRY(c0, cudaStreamSynchronize(c0->stream));
    std::memcpy(diag, c0->h_diag, sizeof(lsqfit_diag));
    return diag->status;
}

}  // extern "C"

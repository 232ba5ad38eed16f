// internal.hpp — host-side internals shared by the C-ABI translation units:
// the context object, error plumbing, grow-only buffers, the per-kernel launch
// dispatchers (each kernel family is instantiated in exactly one k_*.cu) and
// the host-input streaming helpers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <mutex>
#include <type_traits>

#include "host_staging.hpp"
#include "lsqfit_cuda.h"

// Scratch bounds of the power-sum kernel's dynamic tail (checked against
// power_sums.cuh in k_power_sums.cu): chunk records and the largest record
// width (degree LSQ_DYN_MAX <= 6: room for the A/B variants of tools/).
constexpr unsigned kPsDynMaxChunks = 4096;
constexpr int kPsDynMaxNV = 3 * 6 + 1;

// ---------------------------------------------------------------------------
// Context: one device, its streams and grow-only scratch.
// ---------------------------------------------------------------------------
struct lsqfit_cuda_ctx {
    int device = 0;
    int sm_count = 0;
    cudaStream_t stream = nullptr;  // host-path stream (kernels, D2H)
    // power sums: persistent grid per degree (0 = not configured yet: each
    // degree's kernel is configured, and so loaded, on first use), per-CTA dd
    // slots for up to slot_ctas CTAs, last-CTA ticket
    int ps_ctas[LSQFIT_MAX_DEGREE + 1] = {};
    int slot_ctas = 0;
    int qr_slot_ctas = 0;
    double2* d_slots = nullptr;
    unsigned* d_ticket = nullptr;
    // power sums' dynamic tail (power_sums.cuh, PsArgs): chunk records,
    // claim counter
    double2* d_dyn_chunks = nullptr;
    unsigned* d_dyn_counters = nullptr;
    lsqfit_result* d_result = nullptr;
    lsqfit_result* h_result = nullptr;  // pinned
    // batched
    int batch_ctas[LSQFIT_MAX_DEGREE + 1] = {};
    unsigned long long* d_batch_work = nullptr;  // warp kernel: curve claims, finished warps
    // diagnostics
    int diag_ctas = 0;
    double2* d_dslots = nullptr;
    unsigned* d_dticket = nullptr;
    lsqfit_diag* d_diag = nullptr;
    lsqfit_diag* h_diag = nullptr;  // pinned
    // TSQR
    int qr_ctas[LSQFIT_MAX_QR_DEGREE + 1] = {};
    double* d_qslots = nullptr;  // [max grid][55] packed factors
    int* d_qbad = nullptr;
    unsigned* d_qticket = nullptr;
    lsqfit_qr_result* d_qresult = nullptr;
    lsqfit_qr_result* h_qresult = nullptr;  // pinned
    // host-path device buffers (grow-only)
    double* d_buf = nullptr;  // single-chunk inputs, solve scratch
    size_t buf_bytes = 0;
    double* d_res = nullptr;  // residuals / batched outputs
    size_t res_bytes = 0;
    // out-of-core streaming of host inputs
    uint64_t chunk_points = 0;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_copied[2] = {nullptr, nullptr};
    cudaEvent_t ev_consumed[2] = {nullptr, nullptr};
    double* d_sbuf[2] = {nullptr, nullptr};
    size_t sbuf_bytes[2] = {0, 0};
    lsqfit_result* d_recs = nullptr;  // per-chunk records
    size_t recs_bytes = 0;
    lsqfit_diag* d_drecs = nullptr;
    size_t drecs_bytes = 0;
    lsqfit_qr_result* d_qrecs = nullptr;
    size_t qrecs_bytes = 0;
    double* d_oslots = nullptr;  // reference-order per-chunk slots
    size_t oslots_bytes = 0;
    double2* d_aparts = nullptr;  // any-degree partials
    size_t aparts_bytes = 0;
    double* d_aout = nullptr;  // any-degree s, t and status
    size_t aout_bytes = 0;
    lsq_host::Stager stager;  // pageable host <-> device copies
    // The scratch above (slots, tickets, records) is shared by every entry
    // point: the stream that used it last, and an event to chain a launch on
    // another stream behind it (claim_scratch).
    cudaStream_t scratch_stream = nullptr;
    bool scratch_used = false;
    cudaEvent_t ev_scratch = nullptr;
    std::mutex mu;  // serialises calls on this context (whole host-path calls; device-path enqueues)
    char last_error[256] = {0};
};

namespace lsq_impl {

constexpr uint64_t kDefaultStreamChunk = uint64_t(1) << 27;  // points (2 GiB per buffer)
constexpr int kQrSlotDoubles = (LSQFIT_MAX_QR_DEGREE + 2) * (LSQFIT_MAX_QR_DEGREE + 3) / 2;  // largest TSQR factor

inline int record(lsqfit_cuda_ctx* ctx, cudaError_t e) {
    if (e == cudaSuccess) return LSQFIT_OK;
    if (ctx)
        std::snprintf(ctx->last_error, sizeof ctx->last_error, "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? LSQFIT_ENOMEM : LSQFIT_ECUDA;
}

#define LSQ_TRY(ctx, expr)                                              \
    do {                                                                \
        const cudaError_t lsq_try_e_ = (expr);                          \
        if (lsq_try_e_ != cudaSuccess) return lsq_impl::record(ctx, lsq_try_e_); \
    } while (0)

// Device-path entry points run on the caller's stream, which belongs to the
// context's device; the caller's current device may differ (e.g. a tensor on
// cuda:1 while current_device() is 0). Switch to ctx->device for the enqueue
// and restore the caller's device on return.
class DeviceScope {
public:
    explicit DeviceScope(int device) {
        if (cudaGetDevice(&prev_) != cudaSuccess) prev_ = -1;
        err_ = (prev_ == device) ? cudaSuccess : cudaSetDevice(device);
        if (prev_ == device) prev_ = -1;  // nothing to restore
    }
    ~DeviceScope() {
        if (prev_ >= 0) cudaSetDevice(prev_);
    }
    cudaError_t error() const { return err_; }
    DeviceScope(const DeviceScope&) = delete;
    DeviceScope& operator=(const DeviceScope&) = delete;

private:
    int prev_ = -1;
    cudaError_t err_ = cudaSuccess;
};

#define LSQ_ON_DEVICE(ctx)                                   \
    lsq_impl::DeviceScope lsq_device_scope_((ctx)->device);  \
    LSQ_TRY(ctx, lsq_device_scope_.error())

// Make `st` wait for the context's previous scratch user when that was a
// different stream, so launches through one context never overlap on the
// device whatever streams the callers use. Call with ctx->mu held, then
// enqueue the launch before releasing it.
inline cudaError_t claim_scratch(lsqfit_cuda_ctx* ctx, cudaStream_t st) {
    if (ctx->scratch_used && ctx->scratch_stream != st) {
        cudaError_t e = cudaEventRecord(ctx->ev_scratch, ctx->scratch_stream);
        if (e != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(st, ctx->ev_scratch, 0)) != cudaSuccess) return e;
    }
    ctx->scratch_stream = st;
    ctx->scratch_used = true;
    return cudaSuccess;
}

cudaError_t ps_configure(int m, int sm_count, int* ctas);
cudaError_t batched_configure(int m, int sm_count, int* ctas);
cudaError_t qr_configure(int m, int sm_count, int* ctas);

// Per-degree launch configuration on first use (function attributes +
// occupancy: this also loads the kernel's module, so a context pays only for
// the kernels it runs). Call with ctx->mu held on ctx->device. The grid is
// clamped to the scratch sized at context creation.
inline cudaError_t ensure_ps(lsqfit_cuda_ctx* ctx, int m) {
    if (ctx->ps_ctas[m]) return cudaSuccess;
    int ctas = 0;
    const cudaError_t e = ps_configure(m, ctx->sm_count, &ctas);
    if (e == cudaSuccess) ctx->ps_ctas[m] = ctas < ctx->slot_ctas ? ctas : ctx->slot_ctas;
    return e;
}
inline cudaError_t ensure_batched(lsqfit_cuda_ctx* ctx, int m) {
    if (ctx->batch_ctas[m]) return cudaSuccess;
    return batched_configure(m, ctx->sm_count, &ctx->batch_ctas[m]);
}
inline cudaError_t ensure_qr(lsqfit_cuda_ctx* ctx, int m) {
    if (ctx->qr_ctas[m]) return cudaSuccess;
    int ctas = 0;
    const cudaError_t e = qr_configure(m, ctx->sm_count, &ctas);
    if (e == cudaSuccess) ctx->qr_ctas[m] = ctas < ctx->qr_slot_ctas ? ctas : ctx->qr_slot_ctas;
    return e;
}

inline int check_degree(int degree) {
    return (degree < 0 || degree > LSQFIT_MAX_DEGREE) ? LSQFIT_EINVAL : LSQFIT_OK;
}

// Grow-only device allocation (contents are not preserved).
template <class T>
cudaError_t grow(T** buf, size_t* cap, size_t bytes) {
    if (bytes <= *cap) return cudaSuccess;
    cudaFree(*buf);
    *buf = nullptr;
    *cap = 0;
    const cudaError_t e = cudaMalloc(reinterpret_cast<void**>(buf), bytes);
    if (e == cudaSuccess) *cap = bytes;
    return e;
}

// Runtime degree -> compile-time instance: f(std::integral_constant<int, m>{}).
template <int Lo, int Hi, class F>
cudaError_t dispatch_degree(int m, F&& f) {
    if constexpr (Lo > Hi) {
        return cudaErrorInvalidValue;
    } else {
        if (m == Lo) return f(std::integral_constant<int, Lo>{});
        return dispatch_degree<Lo + 1, Hi>(m, static_cast<F&&>(f));
    }
}

inline uint64_t n_chunks(const lsqfit_cuda_ctx* ctx, uint64_t n) {
    return (n + ctx->chunk_points - 1) / ctx->chunk_points;
}

// ---- kernel launch dispatchers (runtime degree -> template instance) -------
// k_power_sums.cu
cudaError_t ps_configure(int m, int sm_count, int* ctas);
int ps_error_levels(int m);
int ps_sum_terms(int m);
cudaError_t ps_launch(lsqfit_cuda_ctx* ctx, int m, const double* d_xy, uint64_t n, unsigned flags,
                      lsqfit_result* out, cudaStream_t st);
cudaError_t ps_combine(int m, const lsqfit_result* parts, int count, unsigned flags, lsqfit_result* out,
                       cudaStream_t st);
// k_diagnostics.cu
cudaError_t diag_launch(lsqfit_cuda_ctx* ctx, int m, const double* d_xy, uint64_t n, const double* d_coeffs,
                        const int32_t* d_gate, double shift, double* d_residuals, lsqfit_diag* out,
                        cudaStream_t st);
cudaError_t diag_combine(const lsqfit_diag* parts, int count, lsqfit_diag* out, cudaStream_t st);
// k_batched.cu
cudaError_t batched_configure(int m, int sm_count, int* ctas);
cudaError_t batched_launch(lsqfit_cuda_ctx* ctx, int m, const double* d_xy, uint64_t n_curves, uint32_t ppc,
                           double* d_coeffs, int32_t* d_status, cudaStream_t st);
cudaError_t batched_ragged_launch(lsqfit_cuda_ctx* ctx, int m, const double* d_xy, const uint64_t* d_offsets,
                                  uint64_t n_curves, uint64_t total_points, double* d_coeffs, int32_t* d_status,
                                  cudaStream_t st);
// k_qr.cu
cudaError_t qr_configure(int m, int sm_count, int* ctas);
cudaError_t qr_launch(lsqfit_cuda_ctx* ctx, int m, const double* d_xy, uint64_t n, unsigned flags,
                      lsqfit_qr_result* out, cudaStream_t st);
cudaError_t qr_combine(int m, const lsqfit_qr_result* parts, int count, unsigned flags, lsqfit_qr_result* out,
                       cudaStream_t st);
// k_ordered.cu (reference-order sums: accumulate_parallel's exact bits)
cudaError_t ordered_launch(lsqfit_cuda_ctx* ctx, int m, const double* d_xy, uint64_t n, uint64_t chunks,
                           unsigned flags, lsqfit_result* out, cudaStream_t st);
// k_misc.cu
cudaError_t synth_launch(int sm_count, double* d_xy, uint64_t n, uint64_t offset, uint64_t seed, int deg,
                         double sigma, cudaStream_t st);
cudaError_t synth_batched_launch(int sm_count, double* d_xy, uint64_t n_curves, uint32_t ppc, uint64_t seed,
                                 int deg, double sigma, cudaStream_t st);
cudaError_t solve_launch(const double* d_a, const double* d_b, int dim, double* d_x, int* d_status,
                         cudaStream_t st);

// k_anysums.cu (any degree): partials per (chunk, column, block), then the
// ordered final fold into s[0..2m], t[0..m] + a status word.
uint64_t anysums_blocks(const lsqfit_cuda_ctx* ctx, uint64_t n, int m);
cudaError_t anysums_partial(const lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n, int m, uint64_t B,
                            double2* parts, cudaStream_t st);
cudaError_t anysums_final(const double2* parts, int chunks, uint64_t B, int m, uint64_t n, double* out, int* status,
                          cudaStream_t st);
constexpr int kMaxAnyDegree = 16384;  // grid.y = 3m+1 <= 65535
// Reference-order (bit-exact) sums at any degree: per-chunk slots (3m+2
// doubles each), then the ascending combine into out[0..3m+1] + status.
cudaError_t ordered_any(const lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n, int m, uint64_t chunks,
                        double* slots, double* out, int* status, cudaStream_t st);

// ---- host inputs (api_host.cu) ---------------------------------------------
// Sums (+ solve per flags) of n host points into ctx->d_result: one H2D + one
// launch when n fits one streaming chunk, otherwise out of core (double-
// buffered H2D on the copy stream overlapping per-chunk kernels, ordered
// record combine).
// With `resident`, every chunk lands in its own slice of ctx->d_buf, so the
// points stay in HBM for a following pass (enqueue_report's d_resident).
cudaError_t enqueue_fit(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, int degree, unsigned flags,
                        bool resident = false);
// Diagnostics of host points against device coefficients into ctx->d_diag
// (y moments centred on `shift`, shared by every chunk); residuals copied back
// when non-null. d_resident: the same points already in HBM (no re-stream).
cudaError_t enqueue_report(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, int degree, const double* d_coeffs,
                           const int32_t* d_gate, double shift, double* residuals,
                           const double* d_resident = nullptr);
// Whether n points can stay resident in ctx->d_buf (with 4 GiB to spare).
bool can_keep_resident(lsqfit_cuda_ctx* ctx, uint64_t n);

// Run fn(k, d_points, count) on ctx->stream for every streaming chunk k.
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
    // Order the first two H2Ds after every kernel already enqueued on
    // ctx->stream: an earlier pass (e.g. fit_normal's sums pass before its
    // report pass, with no host sync between) may still be reading d_sbuf.
    {
        cudaError_t e = cudaEventRecord(ctx->ev_consumed[0], ctx->stream);
        if (e != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_consumed[0], 0)) != cudaSuccess) return e;
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

// As stream_points, but chunk k lands in slice k of ctx->d_buf (grown to all
// n points) and stays there: H2D of chunk k+1 on the copy stream overlaps fn
// on chunk k, and a later pass can read the points from HBM
// (for_resident_chunks) instead of over PCIe again.
template <class F>
cudaError_t stream_points_resident(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, F&& fn) {
    const uint64_t K = n_chunks(ctx, n);
    if (K == 1) return stream_points(ctx, xy, n, fn);  // already lands in ctx->d_buf
    const uint64_t C = ctx->chunk_points;
    cudaError_t e = grow(&ctx->d_buf, &ctx->buf_bytes, size_t(n) * 16);
    if (e != cudaSuccess) return e;
    // the copy stream must not overwrite d_buf before earlier readers finish
    if ((e = cudaEventRecord(ctx->ev_consumed[0], ctx->stream)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_consumed[0], 0)) != cudaSuccess) return e;
    for (uint64_t k = 0; k < K; ++k) {
        const uint64_t lo = k * C;
        const uint64_t cnt = (n - lo < C) ? (n - lo) : C;
        double* dst = ctx->d_buf + 2 * lo;
        if ((e = ctx->stager.h2d(dst, xy + 2 * lo, size_t(cnt) * 16, ctx->copy_stream)) != cudaSuccess) return e;
        if ((e = cudaEventRecord(ctx->ev_copied[k & 1], ctx->copy_stream)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(ctx->stream, ctx->ev_copied[k & 1], 0)) != cudaSuccess) return e;
        if ((e = fn(k, static_cast<const double*>(dst), cnt)) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// fn(k, d_points, count) on ctx->stream for every chunk of a resident dataset.
template <class F>
cudaError_t for_resident_chunks(lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n, F&& fn) {
    const uint64_t K = n_chunks(ctx, n);
    const uint64_t C = K == 1 ? n : ctx->chunk_points;
    for (uint64_t k = 0; k < K; ++k) {
        const uint64_t lo = k * C;
        const uint64_t cnt = (n - lo < C) ? (n - lo) : C;
        const cudaError_t e = fn(k, d_xy + 2 * lo, cnt);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace lsq_impl

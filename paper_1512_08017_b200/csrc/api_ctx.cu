// api_ctx.cu — context lifetime and error strings (include/lsqfit_cuda.h).
#include <cstring>
#include <new>

#include "internal.hpp"

using namespace lsq_impl;

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
    if ((e = cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device)) != cudaSuccess)
        return fail(e);
    // Kernels are configured per degree on first use (ensure_ps / _batched /
    // _qr): creating a context loads no kernel module. The reduction scratch
    // is sized for the largest grids those can ask for (persistent power-sum
    // grids are 1 CTA per SM; TSQR at most a few per SM).
    ctx->slot_ctas = ctx->sm_count * 4;
    ctx->qr_slot_ctas = ctx->sm_count * 16;
    const int max_ctas = ctx->slot_ctas;
    const int max_q = ctx->qr_slot_ctas;
#ifndef LSQ_DIAG_CTAS_PER_SM
#define LSQ_DIAG_CTAS_PER_SM 8
#endif
    ctx->diag_ctas = ctx->sm_count * LSQ_DIAG_CTAS_PER_SM;
    ctx->chunk_points = kDefaultStreamChunk;
    if ((e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking)) != cudaSuccess) return fail(e);
    if ((e = cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking)) != cudaSuccess) return fail(e);
    if ((e = cudaEventCreateWithFlags(&ctx->ev_scratch, cudaEventDisableTiming)) != cudaSuccess) return fail(e);
    for (int b = 0; b < 2; ++b) {
        if ((e = cudaEventCreateWithFlags(&ctx->ev_copied[b], cudaEventDisableTiming)) != cudaSuccess) return fail(e);
        if ((e = cudaEventCreateWithFlags(&ctx->ev_consumed[b], cudaEventDisableTiming)) != cudaSuccess) return fail(e);
    }
    struct Alloc {
        void** p;
        size_t bytes;
        bool zero;
    } const dev[] = {
        {reinterpret_cast<void**>(&ctx->d_slots), sizeof(double2) * size_t(max_ctas) * LSQFIT_MAX_NV, false},
        {reinterpret_cast<void**>(&ctx->d_ticket), sizeof(unsigned), true},
        {reinterpret_cast<void**>(&ctx->d_dyn_chunks), sizeof(double2) * size_t(kPsDynMaxChunks) * kPsDynMaxNV, false},
        {reinterpret_cast<void**>(&ctx->d_dyn_counters), sizeof(unsigned), true},
        {reinterpret_cast<void**>(&ctx->d_batch_work), 2 * sizeof(unsigned long long), true},
        {reinterpret_cast<void**>(&ctx->d_result), sizeof(lsqfit_result), true},
        {reinterpret_cast<void**>(&ctx->d_dslots), sizeof(double2) * size_t(ctx->diag_ctas) * 4, false},
        {reinterpret_cast<void**>(&ctx->d_dticket), sizeof(unsigned), true},
        {reinterpret_cast<void**>(&ctx->d_diag), sizeof(lsqfit_diag), true},
        {reinterpret_cast<void**>(&ctx->d_qslots), sizeof(double) * size_t(max_q) * kQrSlotDoubles, false},
        {reinterpret_cast<void**>(&ctx->d_qbad), sizeof(int) * size_t(max_q), false},
        {reinterpret_cast<void**>(&ctx->d_qticket), sizeof(unsigned), true},
        {reinterpret_cast<void**>(&ctx->d_qresult), sizeof(lsqfit_qr_result), true},
    };
    for (const Alloc& a : dev) {
        if ((e = cudaMalloc(a.p, a.bytes)) != cudaSuccess) return fail(e);
        if (a.zero && (e = cudaMemset(*a.p, 0, a.bytes)) != cudaSuccess) return fail(e);  // tickets start at 0
    }
    if ((e = cudaMallocHost(&ctx->h_result, sizeof(lsqfit_result))) != cudaSuccess) return fail(e);
    if ((e = cudaMallocHost(&ctx->h_diag, sizeof(lsqfit_diag))) != cudaSuccess) return fail(e);
    if ((e = cudaMallocHost(&ctx->h_qresult, sizeof(lsqfit_qr_result))) != cudaSuccess) return fail(e);
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return fail(e);
    *out = ctx;
    return LSQFIT_OK;
}

void lsqfit_cuda_destroy(lsqfit_cuda_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->copy_stream) cudaStreamSynchronize(ctx->copy_stream);
    if (ctx->scratch_used) cudaStreamSynchronize(ctx->scratch_stream);  // last device-path user
    void* const dev[] = {ctx->d_slots,  ctx->d_ticket,  ctx->d_result, ctx->d_dslots, ctx->d_dticket, ctx->d_diag,
                         ctx->d_qslots, ctx->d_qbad,    ctx->d_qticket, ctx->d_qresult, ctx->d_buf,   ctx->d_res,
                         ctx->d_sbuf[0], ctx->d_sbuf[1], ctx->d_recs,  ctx->d_drecs,  ctx->d_qrecs, ctx->d_oslots,
                         ctx->d_aparts, ctx->d_aout, ctx->d_dyn_chunks, ctx->d_dyn_counters,
                         ctx->d_batch_work};
    for (void* p : dev) cudaFree(p);
    void* const host[] = {ctx->h_result, ctx->h_diag, ctx->h_qresult};
    for (void* p : host)
        if (p) cudaFreeHost(p);
    if (ctx->ev_scratch) cudaEventDestroy(ctx->ev_scratch);
    for (int b = 0; b < 2; ++b) {
        if (ctx->ev_copied[b]) cudaEventDestroy(ctx->ev_copied[b]);
        if (ctx->ev_consumed[b]) cudaEventDestroy(ctx->ev_consumed[b]);
    }
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

int lsqfit_cuda_grid_size(lsqfit_cuda_ctx* ctx, int* ctas) {
    if (!ctx || !ctas) return LSQFIT_EINVAL;
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_ON_DEVICE(ctx);
    LSQ_TRY(ctx, ensure_ps(ctx, 3));
    *ctas = ctx->ps_ctas[3];
    return LSQFIT_OK;
}

int lsqfit_cuda_sum_error_levels(int degree) { return ps_error_levels(degree); }

int lsqfit_cuda_sum_terms(int degree) { return ps_sum_terms(degree); }

int lsqfit_cuda_release_buffers(lsqfit_cuda_ctx* ctx) {
    if (!ctx) return LSQFIT_EINVAL;
    std::lock_guard<std::mutex> lock(ctx->mu);
    LSQ_TRY(ctx, cudaSetDevice(ctx->device));
    // outstanding work on any stream that may touch the buffers
    LSQ_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    LSQ_TRY(ctx, cudaStreamSynchronize(ctx->copy_stream));
    if (ctx->scratch_used) LSQ_TRY(ctx, cudaStreamSynchronize(ctx->scratch_stream));
    struct Buf {
        void** p;
        size_t* cap;
    } const grow_only[] = {
        {reinterpret_cast<void**>(&ctx->d_buf), &ctx->buf_bytes},
        {reinterpret_cast<void**>(&ctx->d_res), &ctx->res_bytes},
        {reinterpret_cast<void**>(&ctx->d_sbuf[0]), &ctx->sbuf_bytes[0]},
        {reinterpret_cast<void**>(&ctx->d_sbuf[1]), &ctx->sbuf_bytes[1]},
        {reinterpret_cast<void**>(&ctx->d_recs), &ctx->recs_bytes},
        {reinterpret_cast<void**>(&ctx->d_drecs), &ctx->drecs_bytes},
        {reinterpret_cast<void**>(&ctx->d_qrecs), &ctx->qrecs_bytes},
        {reinterpret_cast<void**>(&ctx->d_oslots), &ctx->oslots_bytes},
        {reinterpret_cast<void**>(&ctx->d_aparts), &ctx->aparts_bytes},
        {reinterpret_cast<void**>(&ctx->d_aout), &ctx->aout_bytes},
    };
    for (const Buf& b : grow_only) {
        if (*b.p) LSQ_TRY(ctx, cudaFree(*b.p));
        *b.p = nullptr;
        *b.cap = 0;
    }
    ctx->stager.release();  // pinned staging buffers and the copy pool (re-created on demand)
    return LSQFIT_OK;
}

int lsqfit_cuda_set_stream_chunk(lsqfit_cuda_ctx* ctx, uint64_t points) {
    if (!ctx) return LSQFIT_EINVAL;
    std::lock_guard<std::mutex> lock(ctx->mu);
    ctx->chunk_points = points ? points : kDefaultStreamChunk;
    return LSQFIT_OK;
}

}  // extern "C"

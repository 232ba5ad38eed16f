// api_group.cu — device groups (include/lsqfit_cuda.h): one host dataset
// sharded over several GPUs of this process.
#include <cstring>
#include <new>
#include <thread>
#include <vector>

#include "internal.hpp"

using namespace lsq_impl;

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
    std::vector<char> resident;        // shard d still in ctx[d]->d_buf
    std::vector<cudaEvent_t> done;     // per device: its record has reached d_parts
    std::mutex mu;
};

namespace {

template <class F>
int group_run(lsqfit_cuda_group* g, F&& per_device) {
    const int G = static_cast<int>(g->ctx.size());
    std::vector<int> st(G, LSQFIT_OK);
    std::vector<std::thread> th;
    try {  // no exception may cross the C ABI
        for (int d = 1; d < G; ++d) th.emplace_back([&, d] { st[d] = per_device(d); });
    } catch (...) {
        for (auto& t : th) t.join();
        return LSQFIT_ENOMEM;
    }
    st[0] = per_device(0);
    for (auto& t : th) t.join();
    for (int d = 0; d < G; ++d)
        if (st[d] != LSQFIT_OK) return st[d];
    return LSQFIT_OK;
}

// Sums of shard d into g->h_parts[d] (an empty record for an empty shard).
// With `resident` the shard stays in its device's HBM when it fits
// (g->resident[d]) for the report pass.
int group_shard_sums(lsqfit_cuda_group* g, int d, const double* xy, uint64_t n, int degree, bool resident = false) {
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
    LSQ_TRY(c, claim_scratch(c, c->stream));
    g->resident[d] = resident && can_keep_resident(c, hi - lo);
    LSQ_TRY(c, enqueue_fit(c, xy + 2 * lo, hi - lo, degree, LSQFIT_SUMS, g->resident[d]));
    LSQ_TRY(c, cudaMemcpyAsync(&g->h_parts[d], c->d_result, sizeof(lsqfit_result), cudaMemcpyDeviceToHost, c->stream));
    LSQ_TRY(c, cudaStreamSynchronize(c->stream));
    return LSQFIT_OK;
}

// Combine the host records on device 0 into ctx[0]->d_result.
int group_combine(lsqfit_cuda_group* g, int degree, unsigned flags) {
    lsqfit_cuda_ctx* c = g->ctx[0];
    const int G = static_cast<int>(g->ctx.size());
    LSQ_TRY(c, cudaSetDevice(c->device));
    LSQ_TRY(c, claim_scratch(c, c->stream));
    LSQ_TRY(c, cudaMemcpyAsync(g->d_parts, g->h_parts, sizeof(lsqfit_result) * G, cudaMemcpyHostToDevice, c->stream));
    LSQ_TRY(c, ps_combine(degree, g->d_parts, G, flags, c->d_result, c->stream));
    return LSQFIT_OK;
}

}  // namespace

extern "C" {

int lsqfit_cuda_group_create(lsqfit_cuda_group** out, const int* devices, int count) {
    if (!out || !devices || count < 1 || count > 64) return LSQFIT_EINVAL;
    *out = nullptr;
    lsqfit_cuda_group* g = new (std::nothrow) lsqfit_cuda_group();
    if (!g) return LSQFIT_ENOMEM;
    try {  // no exception may cross the C ABI
        g->ctx.reserve(count);
        g->resident.assign(count, 0);
        g->done.assign(count, nullptr);
    } catch (...) {
        delete g;
        return LSQFIT_ENOMEM;
    }
    for (int d = 0; d < count; ++d) {
        lsqfit_cuda_ctx* c = nullptr;
        const int st = lsqfit_cuda_create(&c, devices[d]);
        if (st != LSQFIT_OK) {
            lsqfit_cuda_group_destroy(g);
            return st;
        }
        g->ctx.push_back(c);
        if (cudaEventCreateWithFlags(&g->done[d], cudaEventDisableTiming) != cudaSuccess) {
            lsqfit_cuda_group_destroy(g);
            return LSQFIT_ECUDA;
        }
        // direct NVLink copies of the records into device 0 where the pair allows it
        int can = 0;
        if (d > 0 && devices[d] != devices[0] && cudaDeviceCanAccessPeer(&can, devices[d], devices[0]) == cudaSuccess &&
            can) {
            const cudaError_t e = cudaDeviceEnablePeerAccess(devices[0], 0);
            if (e != cudaSuccess) cudaGetLastError();  // already enabled / unsupported: copies still work
        }
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
    for (size_t d = 0; d < g->done.size(); ++d)
        if (g->done[d]) {
            if (d < g->ctx.size()) cudaSetDevice(g->ctx[d]->device);
            cudaEventDestroy(g->done[d]);
        }
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

int lsqfit_cuda_group_fit_device(lsqfit_cuda_group* g, const double* const* d_xy_shards, const uint64_t* shard_n,
                                 int degree, unsigned flags, lsqfit_result* result) {
    if (!g || !d_xy_shards || !shard_n || !result) return LSQFIT_EINVAL;
    if (check_degree(degree) != LSQFIT_OK) return LSQFIT_EINVAL;
    const int G = static_cast<int>(g->ctx.size());
    for (int d = 0; d < G; ++d)
        if ((shard_n[d] > 0 && !d_xy_shards[d]) || reinterpret_cast<uintptr_t>(d_xy_shards[d]) % 16) return LSQFIT_EINVAL;
    std::lock_guard<std::mutex> glock(g->mu);
    lsqfit_cuda_ctx* c0 = g->ctx[0];
    // every device: fused sums of its resident shard, record -> device 0 (peer copy)
    for (int d = 0; d < G; ++d) {
        lsqfit_cuda_ctx* c = g->ctx[d];
        std::lock_guard<std::mutex> lock(c->mu);
        LSQ_TRY(c, cudaSetDevice(c->device));
        LSQ_TRY(c, claim_scratch(c, c->stream));
        LSQ_TRY(c, ps_launch(c, degree, d_xy_shards[d], shard_n[d], LSQFIT_SUMS, c->d_result, c->stream));
        LSQ_TRY(c, cudaMemcpyPeerAsync(g->d_parts + d, c0->device, c->d_result, c->device, sizeof(lsqfit_result),
                                       c->stream));
        LSQ_TRY(c, cudaEventRecord(g->done[d], c->stream));
    }
    // device 0: ascending-device combine + finite check + solve
    std::lock_guard<std::mutex> lock(c0->mu);
    LSQ_TRY(c0, cudaSetDevice(c0->device));
    LSQ_TRY(c0, claim_scratch(c0, c0->stream));
    for (int d = 0; d < G; ++d) LSQ_TRY(c0, cudaStreamWaitEvent(c0->stream, g->done[d], 0));
    LSQ_TRY(c0, ps_combine(degree, g->d_parts, G, flags, c0->d_result, c0->stream));
    LSQ_TRY(c0, cudaMemcpyAsync(c0->h_result, c0->d_result, sizeof(lsqfit_result), cudaMemcpyDeviceToHost,
                                c0->stream));
    LSQ_TRY(c0, cudaStreamSynchronize(c0->stream));
    std::memcpy(result, c0->h_result, sizeof(lsqfit_result));
    return result->status;
}

int lsqfit_cuda_group_fit_report_host(lsqfit_cuda_group* g, const double* xy, uint64_t n, int degree,
                                      lsqfit_result* result, lsqfit_diag* diag, double* residuals) {
    if (!g || !xy || !result || !diag || n == 0) return LSQFIT_EINVAL;
    if (check_degree(degree) != LSQFIT_OK) return LSQFIT_EINVAL;
    std::lock_guard<std::mutex> glock(g->mu);
    const int G = static_cast<int>(g->ctx.size());
    int st = group_run(g, [&](int d) { return group_shard_sums(g, d, xy, n, degree, true); });
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
            g->h_dparts[d].shift = xy[1];  // records combine under one shift
            return LSQFIT_OK;
        }
        std::lock_guard<std::mutex> lock(c->mu);
        LSQ_TRY(c, cudaSetDevice(c->device));
        LSQ_TRY(c, claim_scratch(c, c->stream));
        double* d_coeffs = c->d_result->coeffs;
        LSQ_TRY(c, cudaMemcpyAsync(d_coeffs, result->coeffs, sizeof(double) * (degree + 1), cudaMemcpyHostToDevice,
                                   c->stream));
        LSQ_TRY(c, enqueue_report(c, xy + 2 * lo, hi - lo, degree, d_coeffs, nullptr, xy[1],
                                  residuals ? residuals + lo : nullptr, g->resident[d] ? c->d_buf : nullptr));
        LSQ_TRY(c, cudaMemcpyAsync(&g->h_dparts[d], c->d_diag, sizeof(lsqfit_diag), cudaMemcpyDeviceToHost, c->stream));
        LSQ_TRY(c, cudaStreamSynchronize(c->stream));
        return LSQFIT_OK;
    });
    if (st != LSQFIT_OK) return st;
    std::lock_guard<std::mutex> lock(c0->mu);
    LSQ_TRY(c0, cudaSetDevice(c0->device));
    LSQ_TRY(c0, claim_scratch(c0, c0->stream));
    LSQ_TRY(c0, cudaMemcpyAsync(g->d_dparts, g->h_dparts, sizeof(lsqfit_diag) * G, cudaMemcpyHostToDevice, c0->stream));
    LSQ_TRY(c0, diag_combine(g->d_dparts, G, c0->d_diag, c0->stream));
    LSQ_TRY(c0, cudaMemcpyAsync(c0->h_diag, c0->d_diag, sizeof(lsqfit_diag), cudaMemcpyDeviceToHost, c0->stream));
    LSQ_TRY(c0, cudaStreamSynchronize(c0->stream));
    std::memcpy(diag, c0->h_diag, sizeof(lsqfit_diag));
    return diag->status;
}

}  // extern "C"

// k_anysums.cu — launches of the any-degree power sums (anysums.cuh).
#include "anysums.cuh"
#include "internal.hpp"

namespace lsq_impl {

uint64_t anysums_blocks(const lsqfit_cuda_ctx* ctx, uint64_t n, int m) {
    const uint64_t nc = uint64_t(3 * m + 1);
    uint64_t b = (uint64_t(ctx->sm_count) * 16 + nc - 1) / nc;  // ~16 blocks per SM in total
    const uint64_t by_n = (n + 4095) / 4096;                   // >= 4096 points per block
    if (b > by_n) b = by_n;
    return b ? b : 1;
}

cudaError_t anysums_partial(const lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n, int m, uint64_t B,
                            double2* parts, cudaStream_t st) {
    const dim3 grid(static_cast<unsigned>(B), static_cast<unsigned>(3 * m + 1));
    lsq::anysums_partial_kernel<<<grid, lsq::kAnyThreads, 0, st>>>(reinterpret_cast<const double2*>(d_xy), n, m,
                                                                   parts);
    return cudaGetLastError();
}

cudaError_t anysums_final(const double2* parts, int chunks, uint64_t B, int m, uint64_t n, double* out, int* status,
                          cudaStream_t st) {
    lsq::anysums_final_kernel<<<1, 256, 0, st>>>(parts, chunks, B, m, n, out, status);
    return cudaGetLastError();
}

cudaError_t ordered_any(const lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n, int m, uint64_t chunks,
                        double* slots, double* out, int* status, cudaStream_t st) {
    const uint64_t total = chunks * uint64_t(3 * m + 1);
    uint64_t blocks = (total + 127) / 128;
    const uint64_t cap = uint64_t(ctx->sm_count) * 16;
    if (blocks > cap) blocks = cap;
    lsq::ordered_any_kernel<<<static_cast<unsigned>(blocks ? blocks : 1), 128, 0, st>>>(
        reinterpret_cast<const double2*>(d_xy), n, chunks, m, slots);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    lsq::ordered_any_combine_kernel<<<1, 256, 0, st>>>(slots, chunks, m, out, status);
    return cudaGetLastError();
}

}  // namespace lsq_impl

// k_misc.cu — the synthetic generator and the standalone one-warp solve.
#include "internal.hpp"
#include "solve.cuh"
#include "synth.cuh"

namespace lsq {

// solve_gaussian (normal_backend.cpp:22-74) of a general dim x dim system.
__global__ void solve_kernel(const double* a, const double* b, int dim, double* x, int* status) {
    extern __shared__ double sm[];
    double* A = sm;
    double* B = A + dim * dim;
    double* X = B + dim;
    for (int i = threadIdx.x; i < dim * dim; i += 32) A[i] = a[i];
    for (int i = threadIdx.x; i < dim; i += 32) B[i] = b[i];
    __syncwarp();
    const int st = warp_solve_gaussian(A, B, X, dim);
    for (int i = threadIdx.x; i < dim; i += 32) x[i] = X[i];
    if (threadIdx.x == 0) *status = st;
}

// Systems too large for shared memory: the same warp solve directly on the
// (already copied, so consumable) system in global memory.
__global__ void solve_kernel_global(double* a, double* b, int dim, double* x, int* status) {
    const int st = warp_solve_gaussian(a, b, x, dim);
    if (threadIdx.x == 0) *status = st;
}

}  // namespace lsq

namespace lsq_impl {

cudaError_t synth_launch(int sm_count, double* d_xy, uint64_t n, uint64_t offset, uint64_t seed, int deg,
                         double sigma, cudaStream_t st) {
    uint64_t blocks = (n + 255) / 256;
    const uint64_t cap = uint64_t(sm_count) * 16;
    if (blocks > cap) blocks = cap;
    lsq::synth_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(reinterpret_cast<double2*>(d_xy), n, offset,
                                                                      seed, deg, sigma);
    return cudaGetLastError();
}

cudaError_t synth_batched_launch(int sm_count, double* d_xy, uint64_t n_curves, uint32_t ppc, uint64_t seed,
                                 int deg, double sigma, cudaStream_t st) {
    uint64_t blocks = (n_curves * 32 + 255) / 256;
    const uint64_t cap = uint64_t(sm_count) * 16;
    if (blocks > cap) blocks = cap;
    lsq::synth_batched_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(reinterpret_cast<double2*>(d_xy),
                                                                              n_curves, ppc, seed, deg, sigma);
    return cudaGetLastError();
}

cudaError_t solve_launch(const double* d_a, const double* d_b, int dim, double* d_x, int* d_status,
                         cudaStream_t st) {
    const size_t smem = (size_t(dim) * dim + 2 * size_t(dim)) * sizeof(double);
    if (smem > 200 * 1024) {  // the system is a private device copy: solve it in place
        lsq::solve_kernel_global<<<1, 32, 0, st>>>(const_cast<double*>(d_a), const_cast<double*>(d_b), dim, d_x,
                                                    d_status);
        return cudaGetLastError();
    }
    if (smem > 48 * 1024) {
        const cudaError_t e =
            cudaFuncSetAttribute(lsq::solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    lsq::solve_kernel<<<1, 32, smem, st>>>(d_a, d_b, dim, d_x, d_status);
    return cudaGetLastError();
}

}  // namespace lsq_impl

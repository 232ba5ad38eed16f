// synth.cuh — counter-based synthetic (x, y) generator, device side.
//
// Bit-identical twin of the oracle's host generator (oracle/lsqfit_oracle.c, test side):
// SplitMix64 jumped to a counter, uniforms from the top 53 bits as the
// reference's synthetic.cpp:13-15, truth coefficients -10 + 20u as
// synthetic.cpp:27, Horner evaluation as polynomial.cpp:5-11, noise a
// standardised Irwin-Hall(4) (no libm), every float op explicitly rounded.
// Unlike the reference's sequential mt19937_64 stream, any point can be
// generated independently, so each GPU (or shard) creates its own slice.
#pragma once

#include "common.cuh"

namespace lsq {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kStreamX = 0x5859ULL;
constexpr uint64_t kStreamTruth = 0x54525554ULL;
constexpr double kSqrt3 = 1.7320508075688772;

__host__ __device__ __forceinline__ uint64_t smix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t stream) {
    return smix(seed * kGolden + stream);
}
__device__ __forceinline__ double u53(uint64_t key, uint64_t ctr) {
    return __dmul_rn(static_cast<double>(smix(key + (ctr + 1) * kGolden) >> 11), 0x1.0p-53);
}

__device__ __forceinline__ void synth_truth(uint64_t seed, uint64_t curve, int deg, double* c) {
    const uint64_t key = stream_key(seed, kStreamTruth);
    for (int k = 0; k <= deg; ++k) c[k] = __dadd_rn(-10.0, __dmul_rn(20.0, u53(key, curve * 13 + k)));
}

__device__ __forceinline__ double2 synth_point(const double* c, int deg, double sigma, uint64_t key, uint64_t g) {
    const double x = __dsub_rn(__dmul_rn(2.0, u53(key, 5 * g)), 1.0);
    double acc = c[deg];
    for (int k = deg - 1; k >= 0; --k) acc = __dadd_rn(__dmul_rn(acc, x), c[k]);
    const double u1 = u53(key, 5 * g + 1), u2 = u53(key, 5 * g + 2);
    const double u3 = u53(key, 5 * g + 3), u4 = u53(key, 5 * g + 4);
    const double z = __dmul_rn(__dsub_rn(__dadd_rn(__dadd_rn(u1, u2), __dadd_rn(u3, u4)), 2.0), kSqrt3);
    return make_double2(x, __dadd_rn(acc, __dmul_rn(sigma, z)));
}

__global__ void synth_kernel(double2* __restrict__ xy, uint64_t n, uint64_t offset, uint64_t seed, int deg,
                             double sigma) {
    double c[LSQFIT_MAX_DEGREE + 1];
    synth_truth(seed, 0, deg, c);
    const uint64_t key = stream_key(seed, kStreamX);
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        xy[i] = synth_point(c, deg, sigma, key, offset + i);
}

// One warp per curve (curve-specific truth), lanes stride over its points.
__global__ void synth_batched_kernel(double2* __restrict__ xy, uint64_t n_curves, uint32_t ppc, uint64_t seed,
                                     int deg, double sigma) {
    const uint64_t key = stream_key(seed, kStreamX);
    const int lane = threadIdx.x & 31;
    const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t cv = gw; cv < n_curves; cv += nw) {
        double c[LSQFIT_MAX_DEGREE + 1];
        synth_truth(seed, cv, deg, c);
        for (uint32_t j = lane; j < ppc; j += 32) {
            const uint64_t g = cv * ppc + j;
            xy[g] = synth_point(c, deg, sigma, key, g);
        }
    }
}

}  // namespace lsq

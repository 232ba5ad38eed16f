// batched.cuh — many independent small fits per launch, one warp per curve.
//
// No reference counterpart (the reference fits one Dataset per call); the
// per-curve semantics are exactly accumulate -> build_normal_system ->
// solve_gaussian (power_sums.cpp:13-50, normal_backend.cpp:13-74), with
// curve c owning points [c*ppc, (c+1)*ppc) of one AoS array.
//
// Per curve: every lane streams its points with 256-bit non-allocating loads
// (2 AoS points per LDG, a warp instruction covers 1 KB contiguous), forms
// the reference's terms exactly (power *= x, power * y), sums them with a
// tree per 8-point chunk, adds chunk sums in order, then a shfl-down tree
// across lanes; the warp then solves its (m+1)^2 Hankel system in shared
// memory. Error bound per sum: (3 + ceil(ppc/256) + 5) u * sum|T|.
// Grid: persistent, warps stride over curves; each curve's arithmetic is
// independent of the mapping, so results are deterministic.
#pragma once

#include "common.cuh"
#include "solve.cuh"

namespace lsq {

constexpr int kBatchWarps = 8;
constexpr int kBatchThreads = kBatchWarps * 32;

template <int M>
struct BatchCfg {
    static constexpr int NS = 2 * M, NT = M + 1, NV = NS + NT, DIM = M + 1;
    // per-warp smem: s (2M+1) + t (M+1) + A + b + x
    static constexpr int SCRATCH = (2 * M + 1) + (M + 1) + DIM * DIM + 2 * DIM;
};

template <int M>
__device__ __forceinline__ void batch_terms(const double (&x)[8], const double (&y)[8], double (&acc)[3 * M + 1]) {
    double tmp[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) tmp[j] = y[j];
    acc[2 * M] = __dadd_rn(acc[2 * M], tree_sum<8>(tmp));
    if constexpr (M >= 1) {
        double pw[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) pw[j] = x[j];
#pragma unroll
        for (int k = 1; k <= 2 * M; ++k) {
            if (k > 1) {
#pragma unroll
                for (int j = 0; j < 8; ++j) pw[j] = __dmul_rn(pw[j], x[j]);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) tmp[j] = pw[j];
            acc[k - 1] = __dadd_rn(acc[k - 1], tree_sum<8>(tmp));
            if (k <= M) {
#pragma unroll
                for (int j = 0; j < 8; ++j) tmp[j] = __dmul_rn(pw[j], y[j]);
                acc[2 * M + k] = __dadd_rn(acc[2 * M + k], tree_sum<8>(tmp));
            }
        }
    }
}

template <int M, bool V256>
__global__ void __launch_bounds__(kBatchThreads) batched_fit_kernel(const double* __restrict__ xy, uint64_t n_curves,
                                                                    uint32_t ppc, double* __restrict__ coeffs,
                                                                    int32_t* __restrict__ status) {
    using C = BatchCfg<M>;
    constexpr int NV = C::NV, NS = C::NS, DIM = C::DIM;
    __shared__ double scratch[kBatchWarps][C::SCRATCH];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* s = scratch[warp];
    double* t = s + (2 * M + 1);
    double* A = t + (M + 1);
    double* b = A + DIM * DIM;
    double* xs = b + DIM;

    const uint64_t gw = uint64_t(blockIdx.x) * kBatchWarps + warp;
    const uint64_t nw = uint64_t(gridDim.x) * kBatchWarps;
    const uint32_t full_chunks = ppc / 256;  // 256 points = 8 per lane

    for (uint64_t c = gw; c < n_curves; c += nw) {
        const double* base = xy + c * uint64_t(ppc) * 2;
        double acc[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[v] = 0.0;

        for (uint32_t ch = 0; ch < full_chunks; ++ch) {
            double x[8], y[8];
            if constexpr (V256) {
                // 4 x 256-bit loads: lane owns points ch*256 + q*64 + 2*lane + {0,1}
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    ldg_2pts(base + (size_t(ch) * 256 + q * 64 + 2 * lane) * 2, x[2 * q], y[2 * q],
                             x[2 * q + 1], y[2 * q + 1]);
            } else {
                // curve base only 16-byte aligned (odd ppc): 8 x 128-bit loads
                const double2* b2 = reinterpret_cast<const double2*>(base) + size_t(ch) * 256;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const double2 v = __ldg(b2 + q * 32 + lane);
                    x[q] = v.x;
                    y[q] = v.y;
                }
            }
            batch_terms<M>(x, y, acc);
        }
        const uint32_t done = full_chunks * 256;
        if (done < ppc) {
            // ragged tail: zero points contribute exactly zero (s[0] is ppc)
            double x[8], y[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint32_t p = done + q * 32 + lane;
                x[q] = (p < ppc) ? base[size_t(p) * 2] : 0.0;
                y[q] = (p < ppc) ? base[size_t(p) * 2 + 1] : 0.0;
            }
            batch_terms<M>(x, y, acc);
        }
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[v] = warp_reduce_sum_down(acc[v]);

        int bad = 0;
        if (lane == 0) {
            s[0] = static_cast<double>(ppc);
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                if (v < NS)
                    s[v + 1] = acc[v];
                else
                    t[v - NS] = acc[v];
                bad |= !isfinite(acc[v]);
            }
        }
        bad = __shfl_sync(0xffffffffu, bad, 0);
        __syncwarp();
        int st = bad ? LSQFIT_EOVERFLOW : LSQFIT_OK;
        if (st == LSQFIT_OK) {
            warp_build_normal_system(s, t, M, A, b);
            st = warp_solve_gaussian(A, b, xs, DIM);
        }
        if (lane < DIM) coeffs[c * DIM + lane] = (st == LSQFIT_OK) ? xs[lane] : 0.0;
        if (lane == 0) status[c] = st;
        __syncwarp();
    }
}

}  // namespace lsq

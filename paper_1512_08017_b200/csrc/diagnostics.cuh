// diagnostics.cuh — the FitReport pass after the solve.
//
// Restates make_fit_report (reference proj/src/diagnostics.cpp:40-48):
//   residuals r_i = y_i - evaluate(poly, x_i)   (:14-19; Horner polynomial.cpp:5-11,
//                                                 explicitly rounded, no FMA)
//   non-finite residual -> OverflowError          (:42-44)
//   sse = sum r_i^2                               (:21-25)
//   R  = sqrt(max(0, 1 - sse/sst)), sst = sum (y_i - mean)^2, and the sst == 0
//        special case (:27-38)
// as one streaming pass. Every point contributes r^2, d = y - c and d^2 for a
// shift c (a data value: the first y of the whole dataset), so that
//   sst = sum d^2 - (sum d)^2 / n
// cancels only by the factor 1 + ((mean - c)/stddev)^2 instead of the
// reference's second pass over y; constant y gives d == 0 and sst == 0
// exactly. Each thread loads 8 points per batch (8 independent 16-byte loads
// in flight), sums the three columns with 8-point trees, pairs batches, and
// folds with magnitude-ordered Fast2Sum (the power-sum kernel's scheme); the
// grid reduces in a fixed order (last-CTA pattern). Batches are dealt to the
// CTAs round-robin, so the whole grid streams through one region of HBM at a
// time. Residuals are optionally written (8 B/pt, coalesced).
#pragma once

#include "common.cuh"

namespace lsq {

#ifndef LSQ_DIAG_STCS
#define LSQ_DIAG_STCS 0
#endif
#ifndef LSQ_DIAG_LDCS
#define LSQ_DIAG_LDCS 0
#endif
#ifndef LSQ_DIAG_GRIDSTRIDE
// A/B at n = 1e9: the grid sweeping the array together is 1.2x (read only)
// to 1.6x (with the residual write) faster than 8 contiguous ranges per SM
#define LSQ_DIAG_GRIDSTRIDE 1
#endif

constexpr int kDiagThreads = 256;
constexpr int kDiagWarps = kDiagThreads / 32;
constexpr int kDiagBatch = 8;

__device__ __forceinline__ void two_prod(double a, double b, double& p, double& e) {
    p = __dmul_rn(a, b);
    e = __fma_rn(a, b, -p);
}

// Final SSE / SST / R from the double-double partials {sum r^2, sum d,
// sum d^2} (d = y - shift), diagnostics.cpp:21-38.
static __device__ __noinline__ void diag_finalize(const double* part, double shift, uint64_t n, bool bad,
                                                  lsqfit_diag* out) {
    // Squares are >= 0, so a non-finite SSE with every residual finite means
    // some r^2 overflowed (|r| > ~1e154; Fast2Sum then turns inf into NaN):
    // the reference's plain sum is +inf there (diagnostics.cpp:21-25) and it
    // throws only for non-finite residuals (:42-44), so saturate, don't fail.
    double sse = __dadd_rn(part[0], part[1]);
    if (!isfinite(sse)) sse = bad ? sse : CUDART_INF;
    const double sd_h = part[2], sd_l = part[3];
    const double dn = static_cast<double>(n);
    double p_h, p_e;  // (sum d)^2 as a double-double
    two_prod(sd_h, sd_h, p_h, p_e);
    p_e = __dadd_rn(p_e, __dmul_rn(2.0, __dmul_rn(sd_h, sd_l)));
    const double q1 = __ddiv_rn(p_h, dn);
    double r1_h, r1_e;  // residual of q1 * n vs p
    two_prod(q1, dn, r1_h, r1_e);
    const double q2 = __ddiv_rn(__dadd_rn(__dsub_rn(__dsub_rn(p_h, r1_h), r1_e), p_e), dn);
    double st_h = part[4], st_l = part[5];
    dd_add(st_h, st_l, -q1, -q2);
    double sst = __dadd_rn(st_h, st_l);
    if (sst < 0.0) sst = 0.0;
    if (!isfinite(sst)) sst = CUDART_INF;  // (y - mean)^2 overflowed: the reference's sst is +inf too
    double r;
    if (sst == 0.0) {
        r = (sse <= __dmul_rn(1e-12, dn)) ? 1.0 : 0.0;
    } else {
        const double v = __dsub_rn(1.0, __ddiv_rn(sse, sst));
        r = __dsqrt_rn(v > 0.0 ? v : 0.0);
    }
    out->sse = sse;
    out->r = r;
    double sy_h = sd_h, sy_l = sd_l;  // sum y = sum d + n * shift
    double ns_h, ns_e;
    two_prod(dn, shift, ns_h, ns_e);
    dd_add(sy_h, sy_l, ns_h, ns_e);
    out->sum_y = __dadd_rn(sy_h, sy_l);
    out->sst = sst;
    for (int v = 0; v < 3; ++v) {
        out->part_hi[v] = part[2 * v];
        out->part_lo[v] = part[2 * v + 1];
    }
    out->shift = shift;
    out->n = n;
    out->status = bad ? LSQFIT_EOVERFLOW : LSQFIT_OK;
}

// M >= 0: compile-time degree (coefficients in static shared memory, Horner
// unrolled). M == kAnyDegree: the degree is m_rt (any polynomial the
// reference's residuals / make_fit_report accept), coefficients in dynamic
// shared memory.
constexpr int kAnyDegree = -1;

template <int M>
__global__ void __launch_bounds__(kDiagThreads) diagnostics_kernel(const double2* __restrict__ xy, uint64_t n,
                                                                   const double* __restrict__ coeffs_in,
                                                                   const int32_t* __restrict__ gate, double shift,
                                                                   double* __restrict__ residuals,
                                                                   double2* __restrict__ slots,
                                                                   unsigned* __restrict__ ticket,
                                                                   lsqfit_diag* __restrict__ out, int m_rt = 0) {
    __shared__ double c_static[M < 0 ? 1 : M + 1];
    extern __shared__ double c_dyn[];
    double* c = M < 0 ? c_dyn : c_static;
    const int mm = M < 0 ? m_rt : M;
    __shared__ double red[kDiagWarps][6];
    __shared__ int s_last;
    __shared__ int s_bad[kDiagWarps];
    if (gate && *gate != LSQFIT_OK) {
        if (blockIdx.x == 0 && threadIdx.x == 0) out->status = *gate;
        return;  // the fit failed: no report (uniform across the grid)
    }
    for (int k = threadIdx.x; k <= mm; k += kDiagThreads) c[k] = coeffs_in[k];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (isnan(shift)) shift = n ? __ldg(&xy[0].y) : 0.0;  // default: this array's first y

    double hi[3] = {0, 0, 0}, lo[3] = {0, 0, 0}, pend[3] = {0, 0, 0};
    bool have_pend = false;
    int bad = 0;
#if LSQ_DIAG_GRIDSTRIDE
    // batches of 8 x 256 coalesced points dealt round-robin to the CTAs (the
    // grid sweeps the array together)
    constexpr uint64_t kB = uint64_t(kDiagBatch) * kDiagThreads;
    const uint64_t hi_i = n;
    for (uint64_t base = uint64_t(blockIdx.x) * kB; base < n; base += uint64_t(gridDim.x) * kB) {
#else
    // contiguous range per CTA; inside it batches of 8 x 256 coalesced points
    const uint64_t per = (n + gridDim.x - 1) / gridDim.x;
    const uint64_t lo_i = per * blockIdx.x < n ? per * blockIdx.x : n;
    const uint64_t hi_i = lo_i + per < n ? lo_i + per : n;
    for (uint64_t base = lo_i; base < hi_i; base += uint64_t(kDiagBatch) * kDiagThreads) {
#endif
        double2 p[kDiagBatch];
#pragma unroll
        for (int q = 0; q < kDiagBatch; ++q) {
            const uint64_t i = base + uint64_t(q) * kDiagThreads + threadIdx.x;
#if LSQ_DIAG_LDCS
            p[q] = i < hi_i ? __ldcs(xy + i) : make_double2(0.0, shift);  // padding: r, d contribute 0
#else
            p[q] = i < hi_i ? __ldg(xy + i) : make_double2(0.0, shift);  // padding: r, d contribute 0
#endif
        }
        double e2[kDiagBatch], d1[kDiagBatch], d2[kDiagBatch];
#pragma unroll
        for (int q = 0; q < kDiagBatch; ++q) {
            const uint64_t i = base + uint64_t(q) * kDiagThreads + threadIdx.x;
            double acc = c[mm];
            if constexpr (M >= 0) {
#pragma unroll
                for (int k = M - 1; k >= 0; --k) acc = __dadd_rn(__dmul_rn(acc, p[q].x), c[k]);
            } else {
                for (int k = mm - 1; k >= 0; --k) acc = __dadd_rn(__dmul_rn(acc, p[q].x), c[k]);
            }
            double r = __dsub_rn(p[q].y, acc);
            if (i >= hi_i) r = 0.0;
            if (residuals && i < hi_i) {
#if LSQ_DIAG_STCS
                __stcs(residuals + i, r);  // streaming store: evict-first in L2
#else
                residuals[i] = r;
#endif
            }
            bad |= !isfinite(r);
            const double d = __dsub_rn(p[q].y, shift);
            e2[q] = __dmul_rn(r, r);
            d1[q] = d;
            d2[q] = __dmul_rn(d, d);
        }
        const double ts[3] = {tree_sum<kDiagBatch>(e2), tree_sum<kDiagBatch>(d1), tree_sum<kDiagBatch>(d2)};
        if (have_pend) {
#pragma unroll
            for (int v = 0; v < 3; ++v) fold_sorted(hi[v], lo[v], __dadd_rn(pend[v], ts[v]));
        } else {
#pragma unroll
            for (int v = 0; v < 3; ++v) pend[v] = ts[v];
        }
        have_pend = !have_pend;
    }
    if (have_pend) {
#pragma unroll
        for (int v = 0; v < 3; ++v) fold_sorted(hi[v], lo[v], pend[v]);
    }
#pragma unroll
    for (int v = 0; v < 3; ++v) warp_reduce_dd_down(hi[v], lo[v]);
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
#pragma unroll
        for (int v = 0; v < 3; ++v) {
            red[warp][2 * v] = hi[v];
            red[warp][2 * v + 1] = lo[v];
        }
        s_bad[warp] = bad;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        const int v = threadIdx.x;
        double h = red[0][2 * v], l = red[0][2 * v + 1];
        for (int w = 1; w < kDiagWarps; ++w) dd_add(h, l, red[w][2 * v], red[w][2 * v + 1]);
        slots[size_t(blockIdx.x) * 4 + v] = make_double2(h, l);
    }
    if (threadIdx.x == 3) {
        int b = 0;
        for (int w = 0; w < kDiagWarps; ++w) b |= s_bad[w];
        slots[size_t(blockIdx.x) * 4 + 3] = make_double2(b ? 1.0 : 0.0, 0.0);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (warp < 4) {
        double h = 0, l = 0;
        for (int i = lane; i < int(gridDim.x); i += 32) {
            const double2 r = __ldcg(&slots[size_t(i) * 4 + warp]);
            if (warp == 3)
                h = (h != 0.0 || r.x != 0.0) ? 1.0 : 0.0;
            else
                dd_add(h, l, r.x, r.y);
        }
        if (warp == 3) {
            h = __any_sync(0xffffffffu, h != 0.0) ? 1.0 : 0.0;
        } else {
            warp_reduce_dd_down(h, l);
        }
        if (lane == 0) {
            red[warp][0] = h;
            red[warp][1] = l;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        *ticket = 0u;
        const double part[6] = {red[0][0], red[0][1], red[1][0], red[1][1], red[2][0], red[2][1]};
        diag_finalize(part, shift, n, red[3][0] != 0.0, out);
    }
}

// Fold K diagnostics records (chunks or shards, ascending order; all computed
// with the same shift) and finish.
__global__ void diag_combine_kernel(const lsqfit_diag* parts, int count, lsqfit_diag* out) {
    if (threadIdx.x != 0) return;
    double part[6] = {0, 0, 0, 0, 0, 0};
    unsigned long long n = 0;
    bool bad = false;
    for (int i = 0; i < count; ++i) {
        for (int v = 0; v < 3; ++v) dd_add(part[2 * v], part[2 * v + 1], parts[i].part_hi[v], parts[i].part_lo[v]);
        n += parts[i].n;
        bad |= parts[i].status != LSQFIT_OK;
    }
    diag_finalize(part, count ? parts[0].shift : 0.0, n, bad, out);
}

}  // namespace lsq

// qr.cuh — TSQR cross-check backend: the least-squares fit
// by orthogonal factorisation instead of normal equations.
//
// The reference factors the n x (m+1) Vandermonde matrix with Householder
// reflections, transforming y alongside (qr_backend.cpp:34-103), then back-
// substitutes (solve_qr, :105-124). Here the same factorisation is computed as
// a communication-avoiding TSQR over the augmented rows [1, x, ..., x^m | y]:
//   * every thread folds its rows (x^j by incremental multiplication, as
//     build_vandermonde, qr_backend.cpp:13-32) into a private upper-triangular
//     C x C factor (C = m+2, registers) with Givens rotations;
//   * factors merge in a fixed binary tree (warp -> CTA -> last CTA, through
//     shared memory); a merge rotates the rows of one triangle into the other;
//   * the final R = [R_v | Q^T y; 0 | rho] gives the coefficients by back
//     substitution and the residual norm rho = sqrt(SSE).
// R is unique up to row signs (ours has a nonnegative diagonal, like the
// reference's normalised packed R), so |R(k,k)| and the column norms
// ||R e_j|| = ||V e_j|| reproduce the reference's rank test
// (sigma_k < 1e-12 * max column norm, qr_backend.cpp:43-56), and the
// coefficients agree with the reference's to roundoff times cond(V) — not
// cond(V)^2 as for the normal equations.
// Degrees up to LSQFIT_MAX_QR_DEGREE (12, the reference's whole range): the
// per-thread factor is (m+2)(m+3)/2 doubles of registers — it fits the 255-
// register budget up to m = 8; m = 9..12 spill part of it to local memory
// (L1-resident), which costs throughput, not correctness.
#pragma once

#include "common.cuh"

namespace lsq {

template <int M>
struct QrCfg {
    static constexpr int C = M + 2;            // columns: V (m+1) and y
    static constexpr int NT = C * (C + 1) / 2;  // packed upper triangle
    static constexpr int THREADS = (M <= 5) ? 256 : 128;
    static constexpr int WARPS = THREADS / 32;
    static constexpr size_t SMEM = size_t(THREADS) * NT * sizeof(double);  // one slot per thread
};

// Packed upper-triangular index of (i, j), i <= j.
template <int C>
__device__ __forceinline__ constexpr int tri(int i, int j) {
    return i * C - i * (i - 1) / 2 + (j - i);
}

// Rotate row v (entries start..C-1 significant) into the triangle R.
template <int C>
__device__ __forceinline__ void givens_add_row(double (&R)[C * (C + 1) / 2], double (&v)[C], int start) {
#pragma unroll
    for (int j = 0; j < C; ++j) {
        if (j < start) continue;
        const double a = R[tri<C>(j, j)];
        const double b = v[j];
        if (b == 0.0) continue;
        const double h = __fma_rn(a, a, __dmul_rn(b, b));
        const double inv = rsqrt(h);
        const double c = __dmul_rn(a, inv), s = __dmul_rn(b, inv);
        R[tri<C>(j, j)] = __dmul_rn(h, inv);
#pragma unroll
        for (int k = j + 1; k < C; ++k) {
            const double t = R[tri<C>(j, k)];
            R[tri<C>(j, k)] = __fma_rn(c, t, __dmul_rn(s, v[k]));
            v[k] = __fma_rn(c, v[k], -__dmul_rn(s, t));
        }
    }
}

// R <- qr([R; B]) for a packed triangle B in memory: rotate B's rows into R.
template <int C>
__device__ __forceinline__ void merge_from(double (&R)[C * (C + 1) / 2], const double* B) {
#pragma unroll
    for (int i = 0; i < C; ++i) {
        double v[C];
#pragma unroll
        for (int k = 0; k < C; ++k) v[k] = (k >= i) ? B[tri<C>(i, k)] : 0.0;
        givens_add_row<C>(R, v, i);
    }
}

// One warp: merge slots[0..count) (packed triangles in shared memory) into
// slots[0] by a fixed binary tree.
template <int C>
__device__ __forceinline__ void tree_merge_slots(double* slots, int count) {
    constexpr int NT = C * (C + 1) / 2;
    const int lane = threadIdx.x & 31;
    int width = 1;
    while (width < count) width <<= 1;
    for (int off = width >> 1; off >= 1; off >>= 1) {
        if (lane < off && lane + off < count) {
            double R[NT];
#pragma unroll
            for (int q = 0; q < NT; ++q) R[q] = slots[lane * NT + q];
            merge_from<C>(R, slots + (lane + off) * NT);
#pragma unroll
            for (int q = 0; q < NT; ++q) slots[lane * NT + q] = R[q];
        }
        __syncwarp();
    }
}

struct QrArgs {
    const double2* xy;
    uint64_t n;
    double* cta_slots;  // [gridDim.x][NT]
    int* cta_bad;       // [gridDim.x]
    unsigned* ticket;
    lsqfit_qr_result* out;
    unsigned flags;
};

// Finish from the merged factor (lane 0 of a warp): rank test, back
// substitution, record. Rp packed, n total points, bad: a Vandermonde entry
// overflowed (build_vandermonde's OverflowError, qr_backend.cpp:27-30).
template <int M>
__device__ void qr_finalize(const double* Rp, uint64_t n, bool bad, unsigned flags, lsqfit_qr_result* out) {
    constexpr int C = M + 2, D = M + 1;
    const int lane = threadIdx.x & 31;
    for (int i = lane; i < C * C; i += 32) {
        const int r = i / C, c = i % C;
        out->r[i] = (c >= r) ? Rp[tri<C>(r, c)] : 0.0;
    }
    if (lane != 0) return;
    out->n = n;
    out->degree = M;
    out->residual_norm = fabs(Rp[tri<C>(C - 1, C - 1)]);
    int status = bad ? LSQFIT_EOVERFLOW : LSQFIT_OK;
    if (status == LSQFIT_OK && n < uint64_t(D)) status = LSQFIT_ERANKDEF;  // qr_backend.cpp:37-38
    if (status == LSQFIT_OK) {
        double max_norm = 0.0;  // column norms of V == column norms of R_v
        for (int j = 0; j < D; ++j) {
            double ss = 0.0;
            for (int i = 0; i <= j; ++i) ss = __fma_rn(Rp[tri<C>(i, j)], Rp[tri<C>(i, j)], ss);
            max_norm = fmax(max_norm, __dsqrt_rn(ss));
        }
        if (max_norm == 0.0) status = LSQFIT_ERANKDEF;
        const double floor_ = __dmul_rn(1e-12, max_norm);
        for (int k = 0; k < D && status == LSQFIT_OK; ++k)
            if (fabs(Rp[tri<C>(k, k)]) < floor_) status = LSQFIT_ERANKDEF;
    }
    for (int i = 0; i < D; ++i) out->coeffs[i] = 0.0;
    if (status == LSQFIT_OK && (flags & LSQFIT_SOLVE)) {
        double p[D];
        for (int i = D - 1; i >= 0; --i) {
            double acc = Rp[tri<C>(i, C - 1)];
            for (int k = i + 1; k < D; ++k) acc = __dsub_rn(acc, __dmul_rn(Rp[tri<C>(i, k)], p[k]));
            p[i] = __ddiv_rn(acc, Rp[tri<C>(i, i)]);
        }
        for (int i = 0; i < D; ++i) {
            if (!isfinite(p[i])) status = LSQFIT_EOVERFLOW;  // qr_backend.cpp:120-122
            out->coeffs[i] = p[i];
        }
    }
    out->status = status;
}

template <int M>
__global__ void __launch_bounds__(QrCfg<M>::THREADS) qr_kernel(QrArgs a) {
    using Q = QrCfg<M>;
    constexpr int C = Q::C, NT = Q::NT, THREADS = Q::THREADS, WARPS = Q::WARPS;
    extern __shared__ __align__(16) double s_slots[];  // [THREADS][NT]
    __shared__ int s_bad[WARPS];
    __shared__ int s_last;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    double R[NT];
#pragma unroll
    for (int q = 0; q < NT; ++q) R[q] = 0.0;
    int bad = 0;
    // contiguous row range per CTA; coalesced rows inside it
    const uint64_t n = a.n, G = gridDim.x;
    const uint64_t lo = n * blockIdx.x / G, hi = n * (blockIdx.x + 1) / G;
    for (uint64_t i = lo + threadIdx.x; i < hi; i += THREADS) {
        const double2 p = __ldg(a.xy + i);
        double v[C];
        double pw = 1.0;  // build_vandermonde: power *= x (qr_backend.cpp:20-24)
#pragma unroll
        for (int j = 0; j <= M; ++j) {
            v[j] = pw;
            pw = __dmul_rn(pw, p.x);
        }
        v[C - 1] = p.y;
#pragma unroll
        for (int j = 0; j <= M; ++j) bad |= !isfinite(v[j]);
        givens_add_row<C>(R, v, 0);
    }
    // thread factors -> warp factor (slot 32*warp) -> CTA factor (slot 0)
    double* mine = s_slots + size_t(warp) * 32 * NT;
#pragma unroll
    for (int q = 0; q < NT; ++q) mine[lane * NT + q] = R[q];
    bad = __any_sync(0xffffffffu, bad);
    __syncwarp();
    tree_merge_slots<C>(mine, 32);
    if (lane == 0) s_bad[warp] = bad;
    __syncthreads();
    if (warp == 0) {
        // gather the warp factors into slots 0..WARPS-1 (slot 0 already holds warp 0's)
        for (int w = 1; w < WARPS; ++w)
            for (int q = lane; q < NT; q += 32) s_slots[w * NT + q] = s_slots[size_t(w) * 32 * NT + q];
        __syncwarp();
        tree_merge_slots<C>(s_slots, WARPS);
        if (lane == 0) {
            int b = 0;
            for (int w = 0; w < WARPS; ++w) b |= s_bad[w];
            a.cta_bad[blockIdx.x] = b;
        }
        for (int q = lane; q < NT; q += 32) a.cta_slots[size_t(blockIdx.x) * NT + q] = s_slots[q];
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(a.ticket, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last || warp != 0) return;
    __threadfence();
    // last CTA: lane l merges CTA factors l, l+32, ... (ascending), then a tree
    double F[NT];
#pragma unroll
    for (int q = 0; q < NT; ++q) F[q] = 0.0;
    int fb = 0;
    for (int c = lane; c < int(G); c += 32) {
        double T[NT];
#pragma unroll
        for (int q = 0; q < NT; ++q) T[q] = __ldcg(&a.cta_slots[size_t(c) * NT + q]);
        merge_from<C>(F, T);
        fb |= __ldcg(&a.cta_bad[c]);
    }
#pragma unroll
    for (int q = 0; q < NT; ++q) s_slots[lane * NT + q] = F[q];
    fb = __any_sync(0xffffffffu, fb);
    __syncwarp();
    tree_merge_slots<C>(s_slots, 32);
    if (lane == 0) *a.ticket = 0u;
    qr_finalize<M>(s_slots, n, fb != 0, a.flags, a.out);
}

// Merge per-shard / per-chunk factors (ascending order) and finish (one warp).
template <int M>
__global__ void qr_combine_kernel(const lsqfit_qr_result* parts, int count, unsigned flags, lsqfit_qr_result* out) {
    constexpr int C = M + 2, NT = QrCfg<M>::NT;
    __shared__ double s_F[NT];
    __shared__ unsigned long long s_n;
    __shared__ int s_bad;
    if (threadIdx.x == 0) {
        double F[NT];
        for (int q = 0; q < NT; ++q) F[q] = 0.0;
        unsigned long long n = 0;
        int bad = 0;
        for (int i = 0; i < count; ++i) {
            double T[NT];
            for (int r = 0; r < C; ++r)
                for (int c = r; c < C; ++c) T[tri<C>(r, c)] = parts[i].r[r * C + c];
            merge_from<C>(F, T);
            n += parts[i].n;
            bad |= parts[i].status == LSQFIT_EOVERFLOW;
        }
        for (int q = 0; q < NT; ++q) s_F[q] = F[q];
        s_n = n;
        s_bad = bad;
    }
    __syncwarp();
    if (threadIdx.x < 32) qr_finalize<M>(s_F, s_n, s_bad != 0, flags, out);
}

}  // namespace lsq

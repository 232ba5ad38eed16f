// solve.cuh — one-warp Gaussian elimination with partial pivoting.
//
// Device restatement of lsqfit::solve_gaussian (reference
// proj/src/normal_backend.cpp:22-74), operation for operation:
//   * max_entry = max |a| over all entries (NaN ignored, as std::max is) :29-30
//   * zero matrix -> SingularSystemError                                 :31-32
//   * pivot_floor = 1e-12 * max_entry                                    :33
//   * pivot = first row of maximal |a(r,col)| (strict '>' in row order)  :35-43
//   * pivot < floor -> SingularSystemError                               :44-48
//   * row swap from column col                                           :49-53
//   * factor = a(r,col)/a(col,col); factor == 0 rows skipped;
//     a(r,k) -= factor*a(col,k); b[r] -= factor*b[col]                   :54-61
//   * back substitution acc -= a(i,k)*x[k] in ascending k, x = acc/a(i,i) :64-69
//   * non-finite x -> OverflowError                                      :70-72
// Every product/difference/quotient is an explicitly rounded binary64 op
// (__dmul_rn/__dsub_rn/__ddiv_rn, no contraction), so given identical inputs
// the coefficients are bit-identical to the reference's x86-64 build.
//
// Parallel shape: lanes own rows (row r -> lane r % 32) during elimination;
// the per-row update order does not affect any single result bit, so it is
// exactly the sequential computation. Back substitution is a dependency
// chain and runs on lane 0.
#pragma once

#include "common.cuh"

namespace lsq {

// All 32 lanes of the warp must call. A (dim*dim, row-major), b (dim) and x
// (dim) live in shared memory; A and b are consumed. Returns an LSQFIT_* code
// (warp-uniform).
static __device__ __noinline__ int warp_solve_gaussian(double* A, double* b, double* x, int dim) {
    const int lane = threadIdx.x & 31;

    double mx = 0.0;
    for (int i = lane; i < dim * dim; i += 32) {
        const double v = fabs(A[i]);
        mx = (mx < v) ? v : mx;
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, mx, off);
        mx = (mx < o) ? o : mx;
    }
    if (mx == 0.0) return LSQFIT_ESINGULAR;
    const double pivot_floor = __dmul_rn(1e-12, mx);

    for (int col = 0; col < dim; ++col) {
        const double diag = fabs(A[col * dim + col]);
        int prow = col;
        double piv = diag;
        if (!isnan(diag)) {
            // Lane-local scan of owned rows in ascending order, then a
            // (max value, lowest row) butterfly: the same row the reference's
            // strict-'>' sequential scan selects. NaN candidates never win.
            double bv = -1.0;
            int bi = 0x7fffffff;
            for (int r = col + lane; r < dim; r += 32) {
                double c = fabs(A[r * dim + col]);
                if (isnan(c)) c = -1.0;
                if (c > bv) {
                    bv = c;
                    bi = r;
                }
            }
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
                if (ov > bv || (ov == bv && oi < bi)) {
                    bv = ov;
                    bi = oi;
                }
            }
            piv = bv;
            prow = bi;
        }
        if (piv < pivot_floor) return LSQFIT_ESINGULAR;
        if (prow != col) {
            for (int k = col + lane; k < dim; k += 32) {
                const double tmp = A[col * dim + k];
                A[col * dim + k] = A[prow * dim + k];
                A[prow * dim + k] = tmp;
            }
            if (lane == 0) {
                const double tb = b[col];
                b[col] = b[prow];
                b[prow] = tb;
            }
        }
        __syncwarp();
        const double pv = A[col * dim + col];
        const double bc = b[col];
        for (int r = col + 1 + lane; r < dim; r += 32) {
            const double factor = __ddiv_rn(A[r * dim + col], pv);
            if (factor == 0.0) continue;
            A[r * dim + col] = 0.0;
            for (int k = col + 1; k < dim; ++k)
                A[r * dim + k] = __dsub_rn(A[r * dim + k], __dmul_rn(factor, A[col * dim + k]));
            b[r] = __dsub_rn(b[r], __dmul_rn(factor, bc));
        }
        __syncwarp();
    }

    int bad = 0;
    if (lane == 0) {
        for (int i = dim; i-- > 0;) {
            double acc = b[i];
            for (int k = i + 1; k < dim; ++k) acc = __dsub_rn(acc, __dmul_rn(A[i * dim + k], x[k]));
            x[i] = __ddiv_rn(acc, A[i * dim + i]);
        }
        for (int i = 0; i < dim; ++i) bad |= !isfinite(x[i]);
    }
    __syncwarp();
    bad = __shfl_sync(0xffffffffu, bad, 0);
    return bad ? LSQFIT_EOVERFLOW : LSQFIT_OK;
}

// The same elimination for a compile-time DIM <= 32 with the system in
// registers: lane r holds row r (and b[r]); the pivot row travels by
// shuffles, so a column step costs a few shuffles plus one correctly rounded
// division and DIM-col rounded mul/sub per lane, instead of shared-memory
// round trips. A, b are read from shared memory (not modified); x is written
// there. Identical operation sequence, hence identical bits.
#ifndef LSQ_SOLVE_INLINE
#define LSQ_SOLVE_INLINE 1  // A/B (tools/ab.py): inlined 1.4-2.8% faster at n = 1e6 for m = 1..3, neutral at m >= 5 and 1e8
#endif
#if LSQ_SOLVE_INLINE
#define LSQ_SOLVE_LINKAGE __forceinline__
#else
#define LSQ_SOLVE_LINKAGE __noinline__
#endif
template <int DIM>
static __device__ LSQ_SOLVE_LINKAGE int warp_solve_gaussian_reg(const double* A, const double* b, double* x) {
    static_assert(DIM >= 1 && DIM <= 32, "one row per lane");
    const unsigned FULL = 0xffffffffu;
    // butterflies over the first P2 >= DIM lanes only (the others hold
    // neutral values), then a broadcast from lane 0: log2(P2) + 1 shuffle
    // steps per reduction instead of 5 for small systems
    constexpr int P2 = DIM <= 1 ? 1 : DIM <= 2 ? 2 : DIM <= 4 ? 4 : DIM <= 8 ? 8 : DIM <= 16 ? 16 : 32;
    const int lane = threadIdx.x & 31;
    const bool own = lane < DIM;
    double a[DIM];
    double bb = own ? b[lane] : 0.0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) a[k] = own ? A[lane * DIM + k] : 0.0;
    // max |a| over the whole matrix (NaN ignored, as std::max)
    double mx = 0.0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
        const double v = fabs(a[k]);
        mx = (mx < v) ? v : mx;
    }
#pragma unroll
    for (int off = P2 / 2; off >= 1; off >>= 1) {
        const double o = __shfl_xor_sync(FULL, mx, off);
        mx = (mx < o) ? o : mx;
    }
    if constexpr (P2 < 32) mx = __shfl_sync(FULL, mx, 0);
    if (mx == 0.0) return LSQFIT_ESINGULAR;
    const double pivot_floor = __dmul_rn(1e-12, mx);
#pragma unroll
    for (int col = 0; col < DIM; ++col) {
        const double diag = __shfl_sync(FULL, fabs(a[col]), col);
        int prow = col;
        double piv = diag;
        if (!isnan(diag)) {
            // (value, lowest row) argmax over rows >= col: the row the
            // reference's strict-'>' scan from row col selects; NaN never wins
            double bv = -1.0;
            int bi = 0x7fffffff;
            if (own && lane >= col) {
                const double c = fabs(a[col]);
                bv = isnan(c) ? -1.0 : c;
                bi = lane;
            }
#pragma unroll
            for (int off = P2 / 2; off >= 1; off >>= 1) {
                const double ov = __shfl_xor_sync(FULL, bv, off);
                const int oi = __shfl_xor_sync(FULL, bi, off);
                if (ov > bv || (ov == bv && oi < bi)) {
                    bv = ov;
                    bi = oi;
                }
            }
            if constexpr (P2 < 32) {
                bv = __shfl_sync(FULL, bv, 0);
                bi = __shfl_sync(FULL, bi, 0);
            }
            piv = bv;
            prow = bi;
        }
        if (piv < pivot_floor) return LSQFIT_ESINGULAR;  // warp-uniform
        if (prow != col) {
            const int src = lane == col ? prow : (lane == prow ? col : lane);
#pragma unroll
            for (int k = col; k < DIM; ++k) a[k] = __shfl_sync(FULL, a[k], src);
            bb = __shfl_sync(FULL, bb, src);
        }
        const double pv = __shfl_sync(FULL, a[col], col);
        const double bc = __shfl_sync(FULL, bb, col);
        double prow_k[DIM];
#pragma unroll
        for (int k = col + 1; k < DIM; ++k) prow_k[k] = __shfl_sync(FULL, a[k], col);
        if (own && lane > col) {
            const double factor = __ddiv_rn(a[col], pv);
            if (factor != 0.0) {
                a[col] = 0.0;
#pragma unroll
                for (int k = col + 1; k < DIM; ++k) a[k] = __dsub_rn(a[k], __dmul_rn(factor, prow_k[k]));
                bb = __dsub_rn(bb, __dmul_rn(factor, bc));
            }
        }
    }
    // back substitution, x[DIM-1] first; row i sums k ascending (the
    // reference's order) once x[i+1..] are known
    double xs[DIM];
    int bad = 0;
#pragma unroll
    for (int i = DIM - 1; i >= 0; --i) {
        double xi = 0.0;
        if (lane == i) {
            double acc = bb;
#pragma unroll
            for (int k = i + 1; k < DIM; ++k) acc = __dsub_rn(acc, __dmul_rn(a[k], xs[k]));
            xi = __ddiv_rn(acc, a[i]);
        }
        xs[i] = __shfl_sync(FULL, xi, i);
        bad |= !isfinite(xs[i]);
    }
    if (lane < DIM) {
#pragma unroll
        for (int k = 0; k < DIM; ++k)
            if (k == lane) x[k] = xs[k];
    }
    __syncwarp();
    return bad ? LSQFIT_EOVERFLOW : LSQFIT_OK;
}

#ifndef LSQ_WARP_SOLVE_REG
#define LSQ_WARP_SOLVE_REG 1
#endif
// The solve for a compile-time dimension (A, b consumed or not; x written).
template <int DIM>
__device__ __forceinline__ int warp_solve(double* A, double* b, double* x) {
#if LSQ_WARP_SOLVE_REG
    return warp_solve_gaussian_reg<DIM>(A, b, x);
#else
    return warp_solve_gaussian(A, b, x, DIM);
#endif
}

// Hankel system from power sums (build_normal_system, normal_backend.cpp:13-20):
// a(j,k) = s[j+k], b = t. Warp-cooperative, shared-memory destinations.
__device__ __forceinline__ void warp_build_normal_system(const double* s, const double* t, int degree, double* A,
                                                         double* b) {
    const int lane = threadIdx.x & 31;
    const int dim = degree + 1;
    for (int i = lane; i < dim * dim; i += 32) A[i] = s[i / dim + i % dim];
    for (int j = lane; j < dim; j += 32) b[j] = t[j];
    __syncwarp();
}

}  // namespace lsq

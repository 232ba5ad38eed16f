// batched.cuh — many independent small fits per launch: one warp per curve,
// or one thread per curve for short curves (batched_small_kernel; the system
// in registers up to m = 6, in shared memory beyond).
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

#include <type_traits>

#include "common.cuh"
#include "solve.cuh"

namespace lsq {

constexpr int kBatchWarps = 8;
#ifndef LSQ_BATCH_DYN
#define LSQ_BATCH_DYN 1  // warp kernel: dynamic curve claims (0: static grid-stride deal, for A/B)
#endif
#ifndef LSQ_BATCH_MIN_BLOCKS
#define LSQ_BATCH_MIN_BLOCKS 0  // __launch_bounds__ min blocks per SM, m <= 2 (0: none). A/B at C4: 3 (no spills, 80 regs) 4.8% slower, 4 equal
#endif
#ifndef LSQ_BATCH_CHUNK_UNROLL
#define LSQ_BATCH_CHUNK_UNROLL 1  // 256-point chunks per unrolled loop body (A/B at C4: 2 or 4 are 28-30% slower: occupancy)
#endif
#define LSQ_STR_(x) #x
#define LSQ_UNROLL(n) _Pragma(LSQ_STR_(unroll n))
#ifndef LSQ_BATCH_CLAIM
#define LSQ_BATCH_CLAIM 2  // consecutive curves per claim (A/B 1 / 2 / 4 / 8: 2 best)
#endif
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

// offsets != nullptr: ragged batch, curve c = points [offsets[c], offsets[c+1])
// (then V256 must be false: curve bases are only 16-byte aligned).
template <int M, bool V256, bool RAGGED = false>
__global__ void __launch_bounds__(kBatchThreads, (M <= 2 ? LSQ_BATCH_MIN_BLOCKS : 0)) batched_fit_kernel(const double* __restrict__ xy, uint64_t n_curves,
                                                                    uint32_t ppc_uniform, double* __restrict__ coeffs,
                                                                    int32_t* __restrict__ status,
                                                                    const uint64_t* __restrict__ offsets,
                                                                    unsigned long long* __restrict__ work) {
    static_assert(!(RAGGED && V256), "ragged curve bases are only 16-byte aligned");
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

    // uniform batches keep 32-bit per-curve counts (the measured-fast loop);
    // ragged ones read each curve's range
    using Count = typename std::conditional<RAGGED, uint64_t, uint32_t>::type;
    // Curves after the first one per warp are claimed from work[0] (per-SM
    // HBM bandwidth is not fair, so a static deal finishes on the slowest
    // SM); the claim for the next block of LSQ_BATCH_CLAIM curves is issued
    // before this block's loads and consumed after them. Each curve's result depends only on its own points,
    // so the schedule cannot change any result. work[1] counts finished
    // warps; the last one re-arms both counters for the next launch.
    constexpr uint64_t CL = LSQ_BATCH_DYN ? LSQ_BATCH_CLAIM : 1;
    uint64_t blk = gw;  // claim block: curves [blk * CL, blk * CL + CL); the first one is static
    while (blk * CL < n_curves) {
        unsigned long long claim = 0;
        if (LSQ_BATCH_DYN && lane == 0) claim = atomicAdd(&work[0], 1ull);
        const uint64_t c_end = (blk + 1) * CL < n_curves ? (blk + 1) * CL : n_curves;
        for (uint64_t c = blk * CL; c < c_end; ++c) {
            const uint64_t first = RAGGED ? offsets[c] : c * uint64_t(ppc_uniform);
            const Count ppc = RAGGED ? Count(offsets[c + 1] - first) : Count(ppc_uniform);
            const Count full_chunks = ppc / 256;  // 256 points = 8 per lane
            const double* base = xy + first * 2;
            double acc[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) acc[v] = 0.0;

            LSQ_UNROLL(LSQ_BATCH_CHUNK_UNROLL)
            for (Count ch = 0; ch < full_chunks; ++ch) {
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
            const Count done = full_chunks * 256;
            if (done < ppc) {
                // ragged tail: zero points contribute exactly zero (s[0] is ppc)
                double x[8], y[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const Count p = done + q * 32 + lane;
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
                // the shared-memory warp solve: the register variant's footprint
                // costs this kernel occupancy at high degree (A/B: m = 12, ppc = 4096
                // 8.5 vs 10.0 ms); the solve is amortised over a long curve here
                st = warp_solve_gaussian(A, b, xs, DIM);
            }
            if (lane < DIM) coeffs[c * DIM + lane] = (st == LSQFIT_OK) ? xs[lane] : 0.0;
            if (lane == 0) status[c] = st;
            __syncwarp();
        }
        blk = LSQ_BATCH_DYN ? nw + __shfl_sync(0xffffffffu, claim, 0) : blk + nw;
    }
    if (LSQ_BATCH_DYN && lane == 0 && atomicAdd(&work[1], 1ull) == nw - 1) {
        work[0] = 0ull;
        work[1] = 0ull;
    }
}

// ---------------------------------------------------------------------------
// Short curves: one THREAD per curve. With a warp per curve, curves of a few
// dozen points leave most lanes idle and the per-curve warp reduction and
// warp solve dominate (~7e8 curves/s whatever ppc). Here every thread streams
// its own curve (adjacent threads read adjacent curves, so a warp's loads
// cover one contiguous region; L1 serves the rest of each line), sums the
// reference's terms with 8-point trees added in order, and solves its
// (m+1)x(m+1) system in registers with the scalar restatement below.
// Error bound per sum: (10 + ceil(ppc/64)) u * sum|T| (8-point trees, 8 per
// block partial, block partials in order).
// ---------------------------------------------------------------------------

constexpr int kSmallThreads = 128;

// solve_gaussian (normal_backend.cpp:22-74) for one thread: the same
// operation sequence as warp_solve_gaussian / the reference (first row of
// maximal |a(r,col)| by strict '>', pivot floor 1e-12*max|a|, factor == 0
// rows skipped, rounded mul/sub, correctly rounded division, ascending back
// substitution). The matrix lives in registers (RegMat, compile-time indices;
// row swaps are selects) or, for the larger systems, in shared memory
// (SmemMat: element (i,j) of thread t at [(i*DIM + j)*T + t], so a warp's
// accesses are consecutive words).
template <int DIM>
struct RegMat {
    double (&a)[DIM][DIM];
    double (&v)[DIM];
    __device__ __forceinline__ double& operator()(int i, int j) const { return a[i][j]; }
    __device__ __forceinline__ double& b(int i) const { return v[i]; }
};
template <int DIM, int T>
struct SmemMat {
    double* p;  // this thread's element (0, 0)
    __device__ __forceinline__ double& operator()(int i, int j) const { return p[(i * DIM + j) * T]; }
    __device__ __forceinline__ double& b(int i) const { return p[(DIM * DIM + i) * T]; }
};

template <int DIM, class Mat>
__device__ __forceinline__ int thread_solve_gaussian_m(const Mat& A, double (&x)[DIM]) {
    double mx = 0.0;
#pragma unroll
    for (int i = 0; i < DIM; ++i)
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
            const double v = fabs(A(i, k));
            mx = (mx < v) ? v : mx;  // std::max: NaN never replaces
        }
    if (mx == 0.0) return LSQFIT_ESINGULAR;
    const double pivot_floor = __dmul_rn(1e-12, mx);
#pragma unroll
    for (int col = 0; col < DIM; ++col) {
        int prow = col;
        double piv = fabs(A(col, col));
#pragma unroll
        for (int r = col + 1; r < DIM; ++r) {
            const double c = fabs(A(r, col));
            if (c > piv) {
                piv = c;
                prow = r;
            }
        }
        if (piv < pivot_floor) return LSQFIT_ESINGULAR;
#pragma unroll
        for (int r = col + 1; r < DIM; ++r) {
            if (r == prow) {
#pragma unroll
                for (int k = col; k < DIM; ++k) {
                    const double tmp = A(col, k);
                    A(col, k) = A(r, k);
                    A(r, k) = tmp;
                }
                const double tb = A.b(col);
                A.b(col) = A.b(r);
                A.b(r) = tb;
            }
        }
#pragma unroll
        for (int r = col + 1; r < DIM; ++r) {
            const double factor = __ddiv_rn(A(r, col), A(col, col));
            if (factor != 0.0) {
                A(r, col) = 0.0;
#pragma unroll
                for (int k = col + 1; k < DIM; ++k) A(r, k) = __dsub_rn(A(r, k), __dmul_rn(factor, A(col, k)));
                A.b(r) = __dsub_rn(A.b(r), __dmul_rn(factor, A.b(col)));
            }
        }
    }
    bool bad = false;
#pragma unroll
    for (int i = DIM - 1; i >= 0; --i) {
        double acc = A.b(i);
#pragma unroll
        for (int k = i + 1; k < DIM; ++k) acc = __dsub_rn(acc, __dmul_rn(A(i, k), x[k]));
        x[i] = __ddiv_rn(acc, A(i, i));
    }
#pragma unroll
    for (int i = 0; i < DIM; ++i) bad |= !isfinite(x[i]);
    return bad ? LSQFIT_EOVERFLOW : LSQFIT_OK;
}

// The same sequence with runtime loops over a shared-memory system (no
// unrolling: indices stay dynamic, register use stays flat).
template <int DIM, int T>
__device__ __forceinline__ int thread_solve_gaussian_smem(const SmemMat<DIM, T>& A, double (&x)[DIM]) {
    double mx = 0.0;
#pragma unroll 1
    for (int i = 0; i < DIM * DIM; ++i) {
        const double v = fabs(A.p[i * T]);
        mx = (mx < v) ? v : mx;  // std::max: NaN never replaces
    }
    if (mx == 0.0) return LSQFIT_ESINGULAR;
    const double pivot_floor = __dmul_rn(1e-12, mx);
#pragma unroll 1
    for (int col = 0; col < DIM; ++col) {
        int prow = col;
        double piv = fabs(A(col, col));
#pragma unroll 1
        for (int r = col + 1; r < DIM; ++r) {
            const double c = fabs(A(r, col));
            if (c > piv) {
                piv = c;
                prow = r;
            }
        }
        if (piv < pivot_floor) return LSQFIT_ESINGULAR;
        if (prow != col) {
#pragma unroll 1
            for (int k = col; k < DIM; ++k) {
                const double tmp = A(col, k);
                A(col, k) = A(prow, k);
                A(prow, k) = tmp;
            }
            const double tb = A.b(col);
            A.b(col) = A.b(prow);
            A.b(prow) = tb;
        }
        const double pv = A(col, col), bc = A.b(col);
#pragma unroll 1
        for (int r = col + 1; r < DIM; ++r) {
            const double factor = __ddiv_rn(A(r, col), pv);
            if (factor != 0.0) {
                A(r, col) = 0.0;
#pragma unroll 4
                for (int k = col + 1; k < DIM; ++k) A(r, k) = __dsub_rn(A(r, k), __dmul_rn(factor, A(col, k)));
                A.b(r) = __dsub_rn(A.b(r), __dmul_rn(factor, bc));
            }
        }
    }
    // back substitution: x goes to the (now free) b column, then registers
    bool bad = false;
#pragma unroll 1
    for (int i = DIM - 1; i >= 0; --i) {
        double acc = A.b(i);
#pragma unroll 1
        for (int k = i + 1; k < DIM; ++k) acc = __dsub_rn(acc, __dmul_rn(A(i, k), A.b(k)));
        A.b(i) = __ddiv_rn(acc, A(i, i));
    }
#pragma unroll
    for (int i = 0; i < DIM; ++i) {
        x[i] = A.b(i);
        bad |= !isfinite(x[i]);
    }
    return bad ? LSQFIT_EOVERFLOW : LSQFIT_OK;
}

template <int DIM>
__device__ __forceinline__ int thread_solve_gaussian(double (&A)[DIM][DIM], double (&b)[DIM], double (&x)[DIM]) {
    return thread_solve_gaussian_m<DIM>(RegMat<DIM>{A, b}, x);
}

// STAGED (ppc >= 16): per warp, the next 8 points of its 32 curves — one
// 128-byte slice per curve — are loaded line by line (lane l of load q takes
// point l % 8 of slice 4q + l / 8) into shared memory and read back row-wise
// (a 16-byte pad per row keeps the row reads conflict-free): 5.5-5.8 TB/s at
// m = 2 vs ~4 TB/s for direct per-thread loads, which stay better for curves
// shorter than a slice (A/B, tools/batched_sweep.py).
// SMEM_SOLVE (m >= 7): the (m+1)^2 system lives in dynamic shared memory
// (SmemMat) instead of registers; 64-thread CTAs.
template <bool SMEM_SOLVE>
__host__ __device__ constexpr int small_threads() {
    return SMEM_SOLVE ? 64 : kSmallThreads;
}
template <int M>
__host__ __device__ constexpr size_t small_solve_smem() {
    return size_t((M + 1) * (M + 1) + (M + 1)) * small_threads<true>() * sizeof(double);
}

template <int M, bool STAGED, bool SMEM_SOLVE = false>
__global__ void __launch_bounds__(small_threads<SMEM_SOLVE>()) batched_small_kernel(
    const double2* __restrict__ xy, uint64_t n_curves, uint32_t ppc_uniform, double* __restrict__ coeffs,
    int32_t* __restrict__ status, const uint64_t* __restrict__ offsets = nullptr) {
    // offsets (ragged batch; the direct-load variant only): curve c = points
    // [offsets[c], offsets[c+1]); else c * ppc_uniform + [0, ppc_uniform)
    constexpr int NV = 3 * M + 1, NS = 2 * M, DIM = M + 1;
    constexpr int THREADS = small_threads<SMEM_SOLVE>();
    constexpr int WARPS = THREADS / 32;
    __shared__ double2 stage[STAGED ? WARPS : 1][32][9];
    extern __shared__ double solve_smem[];  // SMEM_SOLVE only
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // curves are dealt to warps in groups of 32 (lane = curve within the group)
    const uint64_t gstride = uint64_t(gridDim.x) * THREADS;
    for (uint64_t c0 = (uint64_t(blockIdx.x) * WARPS + warp) * 32; c0 < n_curves; c0 += gstride) {
        const uint64_t c = c0 + lane;
        if (!STAGED && c >= n_curves) break;
        const uint64_t first = (!STAGED && offsets) ? offsets[c] : c * uint64_t(ppc_uniform);
        const uint64_t ppc = (!STAGED && offsets) ? offsets[c + 1] - first : uint64_t(ppc_uniform);
        // 8-point trees are added into a block partial over 64 points, block
        // partials into the running sums
        double acc[NV], blk[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[v] = blk[v] = 0.0;
        for (uint64_t p0 = 0; p0 < ppc; p0 += 8) {
            double x[8], y[8];
            if constexpr (STAGED) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int row = 4 * q + (lane >> 3), pt = lane & 7;
                    const uint64_t cr = c0 + row;
                    stage[warp][row][pt] = (cr < n_curves && p0 + pt < ppc)
                                               ? __ldg(xy + cr * ppc + p0 + pt)
                                               : make_double2(0.0, 0.0);  // zero points add exactly 0
                }
                __syncwarp();
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const double2 v = stage[warp][lane][j];
                    x[j] = v.x;
                    y[j] = v.y;
                }
                __syncwarp();
            } else {
                const double2* base = xy + first;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const double2 v = (p0 + j < ppc) ? __ldg(base + p0 + j) : make_double2(0.0, 0.0);
                    x[j] = v.x;
                    y[j] = v.y;
                }
            }
            batch_terms<M>(x, y, blk);
            if ((p0 & 63) == 56 || p0 + 8 >= ppc) {
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    acc[v] = __dadd_rn(acc[v], blk[v]);
                    blk[v] = 0.0;
                }
            }
        }
        if (c >= n_curves) continue;  // (staged: after the warp-cooperative loads)
        double xs[DIM];
        bool bad = false;
#pragma unroll
        for (int v = 0; v < NV; ++v) bad |= !isfinite(acc[v]);
        int st = LSQFIT_EOVERFLOW;
        // build_normal_system: a(j,k) = s[j+k] (s[0] = ppc, s[k>=1] = acc[k-1]), b = t
        if constexpr (SMEM_SOLVE) {
            const SmemMat<DIM, THREADS> A{solve_smem + threadIdx.x};
#pragma unroll
            for (int j = 0; j < DIM; ++j) {
#pragma unroll
                for (int k = 0; k < DIM; ++k) A(j, k) = (j + k == 0) ? static_cast<double>(ppc) : acc[j + k - 1];
                A.b(j) = acc[NS + j];
            }
            if (!bad) st = thread_solve_gaussian_smem<DIM, THREADS>(A, xs);
        } else {
            double A[DIM][DIM], b[DIM];
#pragma unroll
            for (int j = 0; j < DIM; ++j) {
#pragma unroll
                for (int k = 0; k < DIM; ++k) A[j][k] = (j + k == 0) ? static_cast<double>(ppc) : acc[j + k - 1];
                b[j] = acc[NS + j];
            }
            if (!bad) st = thread_solve_gaussian<DIM>(A, b, xs);
        }
#pragma unroll
        for (int k = 0; k < DIM; ++k) coeffs[c * DIM + k] = (st == LSQFIT_OK) ? xs[k] : 0.0;
        status[c] = st;
    }
}

}  // namespace lsq

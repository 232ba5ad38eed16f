/*
 * lsqfit_cuda.h — C ABI of the B200 (sm_100a) normal-equation fit hot path.
 *
 * This is the drop-in boundary between host code and the CUDA kernels. It
 * replaces the reference's O(n·m) accumulation and its tiny solve:
 *
 *   reference (paths relative to /root/reference/proj)      replaced by
 *   ------------------------------------------------------   ---------------------------------
 *   lsqfit::accumulate            include/lsqfit/power_sums.hpp:23     lsqfit_cuda_fit_host (SUMS)
 *   lsqfit::accumulate_parallel   include/lsqfit/power_sums.hpp:31     lsqfit_cuda_fit_host (SUMS)
 *     (hot loop accumulate_into   src/power_sums.cpp:13-26,
 *      require_finite             src/power_sums.cpp:28-35)
 *   lsqfit::build_normal_system   include/lsqfit/normal_backend.hpp:17 fused into the fit kernels
 *   lsqfit::solve_gaussian        include/lsqfit/normal_backend.hpp:22 lsqfit_cuda_solve_host
 *   lsqfit::fit_normal (sums+solve part)
 *                                 include/lsqfit/normal_backend.hpp:27 lsqfit_cuda_fit_host (SOLVE)
 *   (no reference counterpart)   batched curves, sharded partials      lsqfit_cuda_fit_batched_device,
 *                                                                      lsqfit_cuda_combine_device
 *
 * Plain C: pointers, sizes, status codes. No exception crosses this ABI; the
 * C++ drop-in layer (include/lsqfit/*.hpp, liblsqfit_b200.so) maps status
 * codes to the reference's exception types (errors.hpp:10-68).
 *
 * Data layout: points are AoS pairs (x0, y0, x1, y1, ...) of IEEE binary64,
 * i.e. exactly the memory image of std::vector<lsqfit::Point> (dataset.hpp:10-13,36).
 * Device pointers must be 16-byte aligned. "stream" arguments are cudaStream_t
 * values passed as void* (NULL = legacy default stream).
 */
#ifndef LSQFIT_CUDA_H
#define LSQFIT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Highest supported degree: kMaxDegree, include/lsqfit/diagnostics.hpp:13. */
#define LSQFIT_MAX_DEGREE 12
/* Number of compensated running sums: s[1..2m] and t[0..m] (s[0] = n is an integer count). */
#define LSQFIT_MAX_NV (3 * LSQFIT_MAX_DEGREE + 1)
/* Largest general system lsqfit_cuda_solve_host accepts (one warp; the matrix in shared memory up to
 * ~160x160, in place in global memory beyond). */
#define LSQFIT_MAX_SOLVE_DIM 4096

/* Status codes. */
#define LSQFIT_OK 0
#define LSQFIT_EINVAL 1    /* std::invalid_argument (power_sums.cpp:40,53-54; normal_backend.cpp:26-27,77) */
#define LSQFIT_EOVERFLOW 2 /* OverflowError (power_sums.cpp:28-35; normal_backend.cpp:70-72) */
#define LSQFIT_ESINGULAR 3 /* SingularSystemError (normal_backend.cpp:31-32,45-48) */
#define LSQFIT_EDEGREE 4   /* DegreeTooHighError (normal_backend.cpp:78-80) */
#define LSQFIT_ECUDA 5     /* CUDA runtime failure (std::runtime_error) */
#define LSQFIT_ENOMEM 6    /* device allocation failed (std::bad_alloc) */
#define LSQFIT_ERANKDEF 7  /* RankDeficientError (qr_backend.cpp:37-38,43-56) */

/* Highest degree of the TSQR cross-check backend (per-thread factor in registers). */
#define LSQFIT_MAX_QR_DEGREE 12

/* Flags for the fit entry points. */
#define LSQFIT_SUMS 0u      /* power sums only (accumulate) */
#define LSQFIT_SOLVE 1u     /* sums, then build_normal_system + solve_gaussian on device */

/*
 * Result of one fit, written by the device (or copied back by the host entry
 * points). Plain-old-data, fixed size, identical on host and device.
 *   s[0..2m], t[0..m]   the reference's PowerSums vectors (power_sums.hpp:13-18);
 *                       s[0] == n exactly (an integer count converted once).
 *   coeffs[0..m]        solve_gaussian's Polynomial coefficients (ascending), if SOLVE.
 *   part_hi/part_lo     the same 3m+1 sums s[1..2m], t[0..m] as unevaluated
 *                       double-double pairs (hi + lo); this is what shards exchange.
 *   status              LSQFIT_OK, LSQFIT_EOVERFLOW or LSQFIT_ESINGULAR.
 */
typedef struct lsqfit_result {
    double s[2 * LSQFIT_MAX_DEGREE + 1];
    double t[LSQFIT_MAX_DEGREE + 1];
    double coeffs[LSQFIT_MAX_DEGREE + 1];
    double part_hi[LSQFIT_MAX_NV];
    double part_lo[LSQFIT_MAX_NV];
    uint64_t n;
    int32_t degree;
    int32_t status;
} lsqfit_result;

/*
 * FitReport diagnostics (make_fit_report, diagnostics.cpp:40-48): SSE, R and
 * the pieces R is formed from. status: LSQFIT_OK or LSQFIT_EOVERFLOW
 * (non-finite residual, diagnostics.cpp:42-44).
 */
typedef struct lsqfit_diag {
    double sse;
    double r;
    double sum_y;
    double sst;
    /* double-double partials (sum r^2, sum d, sum d^2) with d = y - shift,
     * the shift (a data value; records combine only with equal shifts) and
     * the point count: what chunked / sharded report passes combine */
    double part_hi[3];
    double part_lo[3];
    double shift;
    uint64_t n;
    int32_t status;
    int32_t pad;
} lsqfit_diag;

/*
 * TSQR cross-check fit (the QR backend's role, qr_backend.cpp:105-133): the
 * R factor of the augmented Vandermonde rows [1, x, .., x^m | y]
 * (row-major (m+2) x (m+2), upper triangular, nonnegative diagonal), the
 * coefficients by back substitution, and rho = |R(m+1, m+1)| = sqrt(SSE).
 * status: OK, EOVERFLOW, ERANKDEF. Records combine across chunks / shards.
 */
typedef struct lsqfit_qr_result {
    double r[(LSQFIT_MAX_DEGREE + 2) * (LSQFIT_MAX_DEGREE + 2)];
    double coeffs[LSQFIT_MAX_DEGREE + 1];
    double residual_norm;
    uint64_t n;
    int32_t degree;
    int32_t status;
} lsqfit_qr_result;

typedef struct lsqfit_cuda_ctx lsqfit_cuda_ctx;

/* Context: one CUDA device, grow-only scratch, a private stream for the host path. */
int lsqfit_cuda_create(lsqfit_cuda_ctx** out, int device);
/*
 * Host-path streaming granule (points). Host inputs larger than this are
 * processed out of core: double-buffered H2D chunks on a copy stream
 * overlapped with per-chunk kernels, then an ordered combine, so device
 * memory use is bounded (2 chunks) and n may exceed HBM. 0 restores the
 * default (2^27 points = 2 GiB per buffer). Results are a deterministic
 * function of (data, degree, chunk size).
 */
int lsqfit_cuda_set_stream_chunk(lsqfit_cuda_ctx* ctx, uint64_t points);
void lsqfit_cuda_destroy(lsqfit_cuda_ctx* ctx);
const char* lsqfit_cuda_strerror(int status);
/* Text of the last CUDA error seen by this context ("" if none). */
const char* lsqfit_cuda_last_error(lsqfit_cuda_ctx* ctx);
/* Persistent grid of the power-sum kernel on this device (CTAs), for reporting. */
int lsqfit_cuda_grid_size(lsqfit_cuda_ctx* ctx, int* ctas);
/* The stated accuracy of the power sums (lsqfit_result.s / .t) at `degree`:
 * every sum S satisfies |S - S_exact| <= L * 2^-53 * sum|T_i| + ulp(S_exact)
 * (+ O(n 2^-106 sum|T_i|)), where the T_i are exactly the terms the fused
 * kernel forms at that degree (lsqfit_cuda_sum_terms) and L is returned. -1
 * for a degree outside [0, LSQFIT_MAX_DEGREE]. (No reference counterpart:
 * the reference's plain sums carry no bound beyond SPEC.md:146's 1e-9.) */
int lsqfit_cuda_sum_error_levels(int degree);
/* Which terms the fused kernel sums at `degree` (-1 outside [0, 12]):
 *   LSQFIT_TERMS_REFERENCE  exactly the reference's: power *= x, and the
 *                           rounded power * y (power_sums.cpp:20-24);
 *   LSQFIT_TERMS_PRODUCTS   degrees >= 3: s[k] = sum of the
 *                           reference's power for k <= degree and of the
 *                           EXACT product pw_{k/2} * pw_{k-k/2} above it;
 *                           t[j] = sum of the exact products pw_j * y (fused
 *                           multiply-add). Each differs from the reference's
 *                           term by at most ~k ulps, below the reference's own
 *                           rounding of x^k; the reference-order mode
 *                           (lsqfit_cuda_fit_ordered_*) always uses the
 *                           reference's terms. */
#define LSQFIT_TERMS_REFERENCE 0
#define LSQFIT_TERMS_PRODUCTS 1
int lsqfit_cuda_sum_terms(int degree);
/* Free the context's grow-only buffers (host-input staging, resident datasets,
 * streaming records, residual buffers): they are re-allocated on demand by the
 * next call that needs them. For long-running processes after a large fit.
 * (No reference counterpart: the reference allocates per call.) */
int lsqfit_cuda_release_buffers(lsqfit_cuda_ctx* ctx);

/*
 * accumulate / accumulate_parallel (power_sums.hpp:20-31, power_sums.cpp:39-90)
 * and, with LSQFIT_SOLVE, build_normal_system + solve_gaussian
 * (normal_backend.hpp:17-22) on a host dataset — the call behind the drop-in
 * lsqfit::accumulate. xy is host memory (pageable or pinned), n >= 1.
 * Copies H2D into context-owned device memory, runs the fused kernel, copies
 * the result back. Synchronous. flags: LSQFIT_SUMS or LSQFIT_SOLVE.
 * Returns EOVERFLOW for non-finite sums; with SOLVE also ESINGULAR/EOVERFLOW
 * from the solve (result->status carries the same value).
 */
int lsqfit_cuda_fit_host(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, int degree,
                         unsigned flags, lsqfit_result* result);

/*
 * Whole fit_normal (normal_backend.cpp:76-85) on the device: H2D, fused
 * sums + solve, then the diagnostics pass (residuals written back to
 * `residuals` when non-NULL, n doubles). Returns the first failing status.
 */
int lsqfit_cuda_fit_report_host(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, int degree,
                                lsqfit_result* result, lsqfit_diag* diag, double* residuals);

/*
 * make_fit_report / residuals / correlation_coefficient (diagnostics.cpp:14-48)
 * for a given host polynomial coeffs[0..degree]: H2D of the points, one device
 * diagnostics pass, residuals copied back when non-NULL. Returns OK or
 * EOVERFLOW (non-finite residual; diag->status carries it too).
 */
int lsqfit_cuda_report_host(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, const double* coeffs,
                            int degree, lsqfit_diag* diag, double* residuals);

/* Batched mode from host memory (lsqfit_cuda_fit_batched_device semantics; per
 * curve accumulate -> build_normal_system -> solve_gaussian, power_sums.cpp:39-50
 * and normal_backend.cpp:13-74 — no reference counterpart for the batch). */
int lsqfit_cuda_fit_batched_host(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n_curves,
                                 uint32_t points_per_curve, int degree, double* coeffs, int32_t* status);

/*
 * Power sums for ANY degree >= 0 (s[0..2m], t[0..m]; host arrays of 2m+1 and
 * m+1 doubles): the reference's accumulate / accumulate_parallel have no
 * degree cap (power_sums.hpp:20-31). Degrees <= LSQFIT_MAX_DEGREE run the
 * fused kernel; above it a generic kernel forms every term with the
 * reference's exact multiplication chain and sums it compensated (slower:
 * O(m) multiplies per term). Status as accumulate: LSQFIT_EOVERFLOW for
 * non-finite sums (require_finite). Degrees up to 16384.
 */
int lsqfit_cuda_power_sums_host(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, int degree, double* s,
                                double* t);
/* Reference order at any degree: exactly the reference's
 * accumulate_parallel(d, m, chunks) bits (power_sums.cpp:52-90; chunks = 1:
 * accumulate, :39-50), s[0..2m]
 * and t[0..m] host arrays; degrees <= LSQFIT_MAX_DEGREE use the specialised
 * reference-order kernels (lsqfit_cuda_fit_ordered_host). */
int lsqfit_cuda_power_sums_ordered_host(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, int degree,
                                        uint64_t chunks, double* s, double* t);
/* Device-resident variant of lsqfit_cuda_power_sums_host (accumulate,
 * power_sums.hpp:20-23): d_st receives s[0..2m] then t[0..m] (3m+2 doubles),
 * *d_status the status; asynchronous on `stream`. */
int lsqfit_cuda_power_sums_device(lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n, int degree, double* d_st,
                                  int32_t* d_status, void* stream);

/*
 * Device-resident path (the benchmarked one): d_xy holds n AoS points on the
 * context's device; d_result is a device lsqfit_result. One launch: streaming
 * power sums -> deterministic grid reduction -> finite check -> (SOLVE) Hankel
 * build + Gaussian elimination. Asynchronous on `stream`; only argument
 * validation is reported through the return value, numeric status lands in
 * d_result->status. n may be 0 (used by empty shards).
 * The launch uses the context's grid-reduction scratch: a launch on a
 * different stream than the context's previous one (device or host path) is
 * chained behind it with an event, so launches through one context never
 * overlap on the device. Thread-safe; for truly concurrent fits use one
 * context per stream.
 */
int lsqfit_cuda_fit_device(lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n, int degree,
                           unsigned flags, lsqfit_result* d_result, void* stream);

/*
 * Reference-order sums: bit-identical to the reference's
 * accumulate_parallel(dataset, degree, chunks) (power_sums.cpp:52-90), i.e.
 * the same chunk boundaries, the same sequential per-chunk operation order
 * and the same ascending combine, replayed by one GPU thread per chunk
 * (fast when chunks >= ~1e4; exact for any chunks >= 1, chunks == 1 being
 * accumulate() itself). part_lo is zero. flags as lsqfit_cuda_fit_device.
 */
int lsqfit_cuda_fit_ordered_device(lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n, int degree,
                                   uint64_t chunks, unsigned flags, lsqfit_result* d_result, void* stream);
/* Host-resident form (the points must fit in device memory). */
int lsqfit_cuda_fit_ordered_host(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, int degree,
                                 uint64_t chunks, unsigned flags, lsqfit_result* result);

/*
 * Sharded combine: d_parts holds n_parts lsqfit_result records (one per shard,
 * e.g. after an NCCL all-gather), combined in ascending shard order with
 * double-double arithmetic; then finite check and (SOLVE) the solve.
 */
int lsqfit_cuda_combine_device(lsqfit_cuda_ctx* ctx, const lsqfit_result* d_parts, int n_parts,
                               int degree, unsigned flags, lsqfit_result* d_result, void* stream);

/*
 * Diagnostics pass on device data: residuals (optional, n doubles), SSE, R
 * for the polynomial d_coeffs[0..degree] (device memory). If d_gate is not
 * NULL the pass is skipped unless *d_gate == LSQFIT_OK (e.g. point it at
 * d_result->status of the preceding fit). `shift` centres the y moments
 * (sst = sum d^2 - (sum d)^2/n, d = y - shift): pass one data value shared by
 * every shard, or NaN for this array's first y.
 */
int lsqfit_cuda_diagnostics_device(lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n, int degree,
                                   const double* d_coeffs, const int32_t* d_gate, double shift,
                                   double* d_residuals, lsqfit_diag* d_out, void* stream);

/*
 * TSQR fit (no reference counterpart on the GPU; semantics of fit_qr /
 * solve_qr, qr_backend.cpp:105-133): device-resident points, one launch
 * (per-thread Givens factors -> fixed merge tree -> last-CTA finalize).
 * degree <= LSQFIT_MAX_QR_DEGREE. flags: LSQFIT_SOLVE for coefficients.
 */
int lsqfit_cuda_qr_fit_device(lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n, int degree,
                              unsigned flags, lsqfit_qr_result* d_result, void* stream);
/* Merge n_parts TSQR records in ascending order and finish. */
int lsqfit_cuda_qr_combine_device(lsqfit_cuda_ctx* ctx, const lsqfit_qr_result* d_parts, int n_parts,
                                  int degree, unsigned flags, lsqfit_qr_result* d_result, void* stream);
/* Host-resident TSQR fit (streamed out of core like lsqfit_cuda_fit_host). */
int lsqfit_cuda_qr_fit_host(lsqfit_cuda_ctx* ctx, const double* xy, uint64_t n, int degree,
                            lsqfit_qr_result* result);

/*
 * Device groups (single process, several GPUs): one host dataset sharded
 * contiguously ([n*g/G, n*(g+1)/G), the chunk formula of power_sums.cpp:69-70)
 * over G devices, each streaming its shard over its own PCIe link; the G
 * partial records are combined in ascending device order on the first device
 * (the exchange is G x 1016 bytes through the host). Same results contract as
 * the single-device host path.
 */
typedef struct lsqfit_cuda_group lsqfit_cuda_group;
int lsqfit_cuda_group_create(lsqfit_cuda_group** out, const int* devices, int count);
void lsqfit_cuda_group_destroy(lsqfit_cuda_group* group);
int lsqfit_cuda_group_size(lsqfit_cuda_group* group);
int lsqfit_cuda_group_fit_host(lsqfit_cuda_group* group, const double* xy, uint64_t n, int degree,
                               unsigned flags, lsqfit_result* result);
/*
 * Device-resident shards in one process (SURVEY §8e's single-process model):
 * shard d (shard_n[d] points, 16-byte aligned) lives on the group's device d.
 * Every device reduces its shard with the fused kernel; the 1016-byte records
 * go to device 0 by peer copy (NVLink where the pair allows it) and are folded
 * in ascending device order, then finite check and (LSQFIT_SOLVE) the solve.
 * result is host memory. Empty shards (shard_n[d] == 0) are allowed.
 */
int lsqfit_cuda_group_fit_device(lsqfit_cuda_group* g, const double* const* d_xy_shards, const uint64_t* shard_n,
                                 int degree, unsigned flags, lsqfit_result* result);
int lsqfit_cuda_group_fit_report_host(lsqfit_cuda_group* group, const double* xy, uint64_t n, int degree,
                                      lsqfit_result* result, lsqfit_diag* diag, double* residuals);

/*
 * build_normal_system + solve_gaussian from power sums (normal_backend.cpp:13-74):
 * s[0..2m], t[0..m] host arrays -> coeffs[0..m]. Status as lsqfit_cuda_solve_host
 * (ESINGULAR, EOVERFLOW as the reference's exceptions; ENOMEM if the host
 * Hankel matrix cannot be allocated).
 */
int lsqfit_cuda_solve_sums_host(lsqfit_cuda_ctx* ctx, const double* s, const double* t, int degree, double* coeffs);
/*
 * solve_gaussian (normal_backend.cpp:22-74) for a general dim x dim row-major
 * system, computed on the device by one warp, operation-for-operation as the
 * reference (no FMA contraction), so identical inputs give identical bits.
 * Returns OK, EINVAL (dim < 1 or > LSQFIT_MAX_SOLVE_DIM), ESINGULAR, EOVERFLOW.
 */
int lsqfit_cuda_solve_host(lsqfit_cuda_ctx* ctx, const double* a, const double* b, int dim,
                           double* x);

/*
 * Batched mode: n_curves independent curves, curve c owning the
 * points_per_curve AoS points starting at point c*points_per_curve. One warp
 * per curve: sums, solve, write coeffs[c*(degree+1) + k] and status[c].
 */
int lsqfit_cuda_fit_batched_device(lsqfit_cuda_ctx* ctx, const double* d_xy, uint64_t n_curves,
                                   uint32_t points_per_curve, int degree, double* d_coeffs,
                                   int32_t* d_status, void* stream);

/*
 * Ragged batch: curve c = points [d_offsets[c], d_offsets[c+1]) of d_xy
 * (d_offsets: n_curves + 1 non-decreasing device values; curves may be empty,
 * which gives LSQFIT_ESINGULAR like any curve with fewer than degree+1
 * distinct x). Per-curve semantics of lsqfit_cuda_fit_batched_device;
 * total_points (= d_offsets[n] - d_offsets[0]) only selects the kernel
 * (thread per curve for short mean lengths, warp per curve otherwise).
 */
int lsqfit_cuda_fit_batched_ragged_device(lsqfit_cuda_ctx* ctx, const double* d_xy, const uint64_t* d_offsets,
                                          uint64_t n_curves, uint64_t total_points, int degree, double* d_coeffs,
                                          int32_t* d_status, void* stream);
/* Ragged batch from host memory: offsets (n_curves + 1, host, non-decreasing)
 * index xy; coeffs (n_curves*(degree+1)) and status (n_curves) are host
 * outputs. Synchronous. */
int lsqfit_cuda_fit_batched_ragged_host(lsqfit_cuda_ctx* ctx, const double* xy, const uint64_t* offsets,
                                        uint64_t n_curves, int degree, double* coeffs, int32_t* status);

/*
 * Counter-based synthetic generator (identical bits on host: oracle/lsqfit_oracle.c).
 * Point i (global index offset+i): x = 2u-1 in [-1,1), y = truth(x) + sigma*z,
 * z = standardised Irwin-Hall(4); truth has truth_degree+1 coefficients U[-10,10]
 * keyed by (seed, curve). Single-curve form uses curve 0.
 */
int lsqfit_cuda_synth_device(lsqfit_cuda_ctx* ctx, double* d_xy, uint64_t n, uint64_t offset,
                             uint64_t seed, int truth_degree, double sigma, void* stream);
/* Batched form: curve c = (offset+i) / points_per_curve picks the truth polynomial. */
int lsqfit_cuda_synth_batched_device(lsqfit_cuda_ctx* ctx, double* d_xy, uint64_t n_curves,
                                     uint32_t points_per_curve, uint64_t seed, int truth_degree,
                                     double sigma, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* LSQFIT_CUDA_H */

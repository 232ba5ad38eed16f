/*
 * lsqfit_oracle.h — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A plain-C restatement of the reference's normal-equation path, used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg to check
 * the CUDA path. Citations are relative to /root/reference/proj.
 *
 * Pinned against the compiled reference (oracle/_ref, built by oracle/Makefile
 * from the reference's own sources) and against tests/golden/ JSON fixtures
 * produced from that build by oracle/make_golden.py.
 */
#ifndef LSQFIT_ORACLE_H
#define LSQFIT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes mirror include/lsqfit_cuda.h. */
enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_EOVERFLOW = 2, ORC_ESINGULAR = 3, ORC_EDEGREE = 4 };

/* accumulate (src/power_sums.cpp:39-50 over accumulate_into :13-26, require_finite :28-35). */
int orc_accumulate(const double* xy, uint64_t n, int degree, double* s, double* t);
/* accumulate_parallel (src/power_sums.cpp:52-90): chunked, OpenMP, ascending combine. */
int orc_accumulate_parallel(const double* xy, uint64_t n, int degree, int chunks, double* s,
                            double* t);
/* build_normal_system (src/normal_backend.cpp:13-20): a is (m+1)^2 row-major. */
void orc_build_normal_system(const double* s, int degree, double* a);
/* solve_gaussian (src/normal_backend.cpp:22-74). a, b are consumed (modified). */
int orc_solve_gaussian(double* a, double* b, int dim, double* x);
/* fit_normal's numeric part (src/normal_backend.cpp:76-85): degree checks, sums, solve. */
int orc_fit_normal(const double* xy, uint64_t n, int degree, int chunks, double* coeffs);

/*
 * Exact-sum oracle: double-double sums of exactly the terms the reference
 * forms (power *= x, power * y rounded; power_sums.cpp:20-24), plus sum|term|.
 * Outputs are length 2m+1 (s) and m+1 (t); index 0 of s is n. Threads fixed
 * chunks combined in ascending order (deterministic).
 */
int orc_exact_sums(const double* xy, uint64_t n, int degree, double* s_hi, double* s_lo,
                   double* s_abs, double* t_hi, double* t_lo, double* t_abs);

/*
 * Exact sums of both term families the CUDA kernel may form: the reference's
 * plain powers / rounded moments, and the exact products pw_a * pw_b
 * (a = k/2, b = k - a) / pw_j * y of its fused multiply-add mode.
 */
int orc_exact_sums_terms(const double* xy, uint64_t n, int degree, double* sp_hi, double* sp_lo,
                         double* sp_abs, double* sx_hi, double* sx_lo, double* sx_abs, double* tr_hi,
                         double* tr_lo, double* tr_abs, double* tx_hi, double* tx_lo, double* tx_abs);

/* Residual moments {sum r^2, sum (y-shift), sum (y-shift)^2}, r = y - Horner(x) as
 * the reference (diagnostics.cpp:14-19, polynomial.cpp:5-11), summed exactly. */
void orc_residual_moments(const double* xy, uint64_t n, const double* coeffs, int degree, double shift,
                          double* out);

/* tests/support/oracles.hpp:40-51 accumulate_oracle: std::pow + Kahan. */
void orc_kahan_pow_sums(const double* xy, uint64_t n, int degree, double* s, double* t);

/* Batched reference loop: per curve accumulate -> build -> solve (no reference batched API). */
void orc_fit_batched(const double* xy, uint64_t n_curves, uint32_t ppc, int degree,
                     double* coeffs, int32_t* status);

/* Counter-based generator, bit-identical to the device generator (csrc/synth.cuh). */
void orc_synth(double* xy, uint64_t n, uint64_t offset, uint64_t seed, int truth_degree,
               double sigma);
void orc_synth_batched(double* xy, uint64_t n_curves, uint32_t ppc, uint64_t seed,
                       int truth_degree, double sigma);
void orc_synth_truth(uint64_t seed, uint64_t curve, int truth_degree, double* coeffs);

/* generate_synthetic (src/synthetic.cpp:13-56): mt19937_64 + Box-Muller on [0,1). */
int orc_generate_synthetic(uint64_t n, int degree, double sigma, uint64_t seed, double* xy);

/* Number of OpenMP threads the oracle uses (for reporting cores). */
int orc_max_threads(void);

#ifdef __cplusplus
}
#endif
#endif

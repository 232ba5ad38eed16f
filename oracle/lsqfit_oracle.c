/*
 * lsqfit_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's normal-equation path (the checker the
 * CUDA path is compared against). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product (paper_1512_08017_b200/) never links or calls it.
 *
 * Every function cites the reference lines it restates (relative to
 * /root/reference/proj). Build: oracle/Makefile, gcc -O3 -fopenmp
 * -ffp-contract=off (x86-64 SSE2: no FMA, no extended precision — the same
 * arithmetic the reference's Release build performs).
 */
#include "lsqfit_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---------------------------------------------------------------------------
 * Power sums.
 * ------------------------------------------------------------------------- */

/* accumulate_into, src/power_sums.cpp:13-26: per point, power starts at 1 and
 * is multiplied by x after each term; s[k] += power; t[k] += power*y for k<=m. */
static void accumulate_into(const double* xy, uint64_t lo, uint64_t hi, int degree, double* s,
                            double* t) {
    const int top = 2 * degree;
    for (uint64_t i = lo; i < hi; ++i) {
        const double x = xy[2 * i];
        const double y = xy[2 * i + 1];
        double power = 1.0;
        for (int k = 0; k <= top; ++k) {
            s[k] += power;
            if (k <= degree) t[k] += power * y;
            power *= x;
        }
    }
}

/* require_finite, src/power_sums.cpp:28-35. */
static int require_finite(const double* s, const double* t, int degree) {
    for (int k = 0; k <= 2 * degree; ++k)
        if (!isfinite(s[k])) return ORC_EOVERFLOW;
    for (int j = 0; j <= degree; ++j)
        if (!isfinite(t[j])) return ORC_EOVERFLOW;
    return ORC_OK;
}

/* accumulate, src/power_sums.cpp:39-50. */
int orc_accumulate(const double* xy, uint64_t n, int degree, double* s, double* t) {
    if (degree < 0) return ORC_EINVAL;
    memset(s, 0, sizeof(double) * (size_t)(2 * degree + 1));
    memset(t, 0, sizeof(double) * (size_t)(degree + 1));
    accumulate_into(xy, 0, n, degree, s, t);
    return require_finite(s, t, degree);
}

/* accumulate_parallel, src/power_sums.cpp:52-90: `chunks` contiguous slices
 * [n*c/C, n*(c+1)/C) (:68-70), one slot of stride 3m+2 per chunk (:59,63,71),
 * OpenMP static schedule (:66), ascending element-wise combine (:80-87). */
int orc_accumulate_parallel(const double* xy, uint64_t n, int degree, int chunks, double* s,
                            double* t) {
    if (degree < 0) return ORC_EINVAL;
    if (chunks < 1) return ORC_EINVAL;
    const size_t s_len = (size_t)(2 * degree) + 1;
    const size_t t_len = (size_t)degree + 1;
    const size_t stride = s_len + t_len;
    double* partials = (double*)calloc((size_t)chunks * stride, sizeof(double));
    if (!partials) return ORC_EINVAL;
#pragma omp parallel for schedule(static)
    for (int c = 0; c < chunks; ++c) {
        const uint64_t uc = (uint64_t)c;
        const uint64_t lo = n * uc / (uint64_t)chunks;
        const uint64_t hi = n * (uc + 1) / (uint64_t)chunks;
        double* slot = partials + uc * stride;
        accumulate_into(xy, lo, hi, degree, slot, slot + s_len);
    }
    memcpy(s, partials, sizeof(double) * s_len);
    memcpy(t, partials + s_len, sizeof(double) * t_len);
    for (int c = 1; c < chunks; ++c) {
        const double* slot = partials + (size_t)c * stride;
        for (size_t k = 0; k < s_len; ++k) s[k] += slot[k];
        for (size_t j = 0; j < t_len; ++j) t[j] += slot[s_len + j];
    }
    free(partials);
    return require_finite(s, t, degree);
}

/* ---------------------------------------------------------------------------
 * Normal system and Gaussian elimination.
 * ------------------------------------------------------------------------- */

/* build_normal_system, src/normal_backend.cpp:13-20: a(j,k) = s[j+k]. */
void orc_build_normal_system(const double* s, int degree, double* a) {
    const int dim = degree + 1;
    for (int j = 0; j < dim; ++j)
        for (int k = 0; k < dim; ++k) a[j * dim + k] = s[j + k];
}

/* solve_gaussian, src/normal_backend.cpp:22-74. */
int orc_solve_gaussian(double* a, double* b, int dim, double* x) {
    if (dim <= 0) return ORC_EINVAL;
    double max_entry = 0.0;
    for (int i = 0; i < dim * dim; ++i) {
        const double v = fabs(a[i]);
        /* std::max(max_entry, v) == (max_entry < v) ? v : max_entry */
        if (max_entry < v) max_entry = v;
    }
    if (max_entry == 0.0) return ORC_ESINGULAR; /* :31-32 */
    const double pivot_floor = 1e-12 * max_entry; /* :33 */

    for (int col = 0; col < dim; ++col) {
        int pivot_row = col;
        double pivot = fabs(a[col * dim + col]);
        for (int r = col + 1; r < dim; ++r) { /* :37-43, strict '>' keeps the upper row */
            const double candidate = fabs(a[r * dim + col]);
            if (candidate > pivot) {
                pivot = candidate;
                pivot_row = r;
            }
        }
        if (pivot < pivot_floor) return ORC_ESINGULAR; /* :44-47 */
        if (pivot_row != col) {                          /* :49-53 */
            for (int k = col; k < dim; ++k) {
                const double tmp = a[col * dim + k];
                a[col * dim + k] = a[pivot_row * dim + k];
                a[pivot_row * dim + k] = tmp;
            }
            const double tb = b[col];
            b[col] = b[pivot_row];
            b[pivot_row] = tb;
        }
        for (int r = col + 1; r < dim; ++r) { /* :54-61 */
            const double factor = a[r * dim + col] / a[col * dim + col];
            if (factor == 0.0) continue;
            a[r * dim + col] = 0.0;
            for (int k = col + 1; k < dim; ++k) a[r * dim + k] -= factor * a[col * dim + k];
            b[r] -= factor * b[col];
        }
    }
    for (int i = dim; i-- > 0;) { /* :64-69 back substitution */
        double acc = b[i];
        for (int k = i + 1; k < dim; ++k) acc -= a[i * dim + k] * x[k];
        x[i] = acc / a[i * dim + i];
    }
    for (int i = 0; i < dim; ++i) /* :70-72 */
        if (!isfinite(x[i])) return ORC_EOVERFLOW;
    return ORC_OK;
}

/* fit_normal numeric part, src/normal_backend.cpp:76-85 (kMaxDegree = 12,
 * include/lsqfit/diagnostics.hpp:13). */
int orc_fit_normal(const double* xy, uint64_t n, int degree, int chunks, double* coeffs) {
    if (degree < 0) return ORC_EINVAL;
    if (degree > 12) return ORC_EDEGREE;
    double s[25], t[13], a[169];
    const int st = chunks == 1 ? orc_accumulate(xy, n, degree, s, t)
                               : orc_accumulate_parallel(xy, n, degree, chunks, s, t);
    if (st != ORC_OK) return st;
    orc_build_normal_system(s, degree, a);
    return orc_solve_gaussian(a, t, degree + 1, coeffs);
}

/* ---------------------------------------------------------------------------
 * Exact-sum oracle (double-double over the reference's own terms).
 * ------------------------------------------------------------------------- */

static inline void two_sum(double a, double b, double* s, double* e) {
    const double ss = a + b;
    const double bb = ss - a;
    *e = (a - (ss - bb)) + (b - bb);
    *s = ss;
}

static inline void dd_add(double* hi, double* lo, double bhi, double blo) {
    double s, e;
    two_sum(*hi, bhi, &s, &e);
    e += *lo + blo;
    const double h = s + e;
    *lo = e - (h - s);
    *hi = h;
}

#define ORC_EXACT_CHUNKS 256

int orc_exact_sums(const double* xy, uint64_t n, int degree, double* s_hi, double* s_lo,
                   double* s_abs, double* t_hi, double* t_lo, double* t_abs) {
    if (degree < 0 || degree > 16384) return ORC_EINVAL; /* any degree the library accepts */
    const int ns = 2 * degree + 1, nt = degree + 1, nv = ns + nt;
    double* part = (double*)calloc((size_t)ORC_EXACT_CHUNKS * nv * 3, sizeof(double));
    double* scratch = (double*)calloc((size_t)ORC_EXACT_CHUNKS * nv * 3, sizeof(double));
    if (!part || !scratch) {
        free(part);
        free(scratch);
        return ORC_EINVAL;
    }
#pragma omp parallel for schedule(dynamic, 1)
    for (int c = 0; c < ORC_EXACT_CHUNKS; ++c) {
        const uint64_t lo = n * (uint64_t)c / ORC_EXACT_CHUNKS;
        const uint64_t hi = n * (uint64_t)(c + 1) / ORC_EXACT_CHUNKS;
        double* h = scratch + (size_t)c * nv * 3; /* per-chunk running sums (zeroed by calloc) */
        double* l = h + nv;
        double* ab = l + nv;
        for (uint64_t i = lo; i < hi; ++i) {
            const double x = xy[2 * i], y = xy[2 * i + 1];
            double power = 1.0;
            for (int k = 0; k < ns; ++k) {
                double sum, err;
                two_sum(h[k], power, &sum, &err);
                h[k] = sum;
                l[k] += err;
                ab[k] += fabs(power);
                if (k < nt) {
                    const double term = power * y; /* rounded exactly as power_sums.cpp:22 */
                    two_sum(h[ns + k], term, &sum, &err);
                    h[ns + k] = sum;
                    l[ns + k] += err;
                    ab[ns + k] += fabs(term);
                }
                power *= x;
            }
        }
        double* slot = part + (size_t)c * nv * 3;
        for (int v = 0; v < nv; ++v) {
            /* renormalise the chunk's (hi, lo) */
            const double hh = h[v] + l[v];
            slot[v] = hh;
            slot[nv + v] = l[v] - (hh - h[v]);
            slot[2 * nv + v] = ab[v];
        }
    }
    for (int v = 0; v < nv; ++v) {
        double hi = 0.0, lo = 0.0, ab = 0.0;
        for (int c = 0; c < ORC_EXACT_CHUNKS; ++c) {
            const double* slot = part + (size_t)c * nv * 3;
            dd_add(&hi, &lo, slot[v], slot[nv + v]);
            ab += slot[2 * nv + v];
        }
        if (v < ns) {
            s_hi[v] = hi; s_lo[v] = lo; s_abs[v] = ab;
        } else {
            t_hi[v - ns] = hi; t_lo[v - ns] = lo; t_abs[v - ns] = ab;
        }
    }
    free(part);
    free(scratch);
    return ORC_OK;
}

/*
 * Exact sums of BOTH term families the CUDA kernel may form (no reference
 * counterpart: the reference forms only the first family):
 *   s_plain[k] = sum pw_k                 pw_k = the reference's power (power *= x)
 *   s_prod[k]  = sum pw_a * pw_b (exact)  a = k / 2, b = k - a  (k >= 2; = s_plain below)
 *   t_round[j] = sum fl(pw_j * y)         the reference's rounded moment term
 *   t_exact[j] = sum pw_j * y (exact)     the fused multiply-add term
 * each as a double-double plus sum|term|. Exact products via fma (TwoProd).
 * Layout of every output group: [hi(2m+1 or m+1)] etc., as orc_exact_sums.
 */
int orc_exact_sums_terms(const double* xy, uint64_t n, int degree, double* sp_hi, double* sp_lo,
                         double* sp_abs, double* sx_hi, double* sx_lo, double* sx_abs, double* tr_hi,
                         double* tr_lo, double* tr_abs, double* tx_hi, double* tx_lo, double* tx_abs) {
    if (degree < 0 || degree > 4096) return ORC_EINVAL;
    const int ns = 2 * degree + 1, nt = degree + 1;
    const int nv = 2 * ns + 2 * nt; /* [s_plain | s_prod | t_round | t_exact] */
    double* part = (double*)calloc((size_t)ORC_EXACT_CHUNKS * nv * 3, sizeof(double));
    double* scratch = (double*)calloc((size_t)ORC_EXACT_CHUNKS * nv * 3, sizeof(double));
    double* pws = (double*)calloc((size_t)ORC_EXACT_CHUNKS * ns, sizeof(double));
    if (!part || !scratch || !pws) {
        free(part);
        free(scratch);
        free(pws);
        return ORC_EINVAL;
    }
#pragma omp parallel for schedule(dynamic, 1)
    for (int c = 0; c < ORC_EXACT_CHUNKS; ++c) {
        const uint64_t lo = n * (uint64_t)c / ORC_EXACT_CHUNKS;
        const uint64_t hi = n * (uint64_t)(c + 1) / ORC_EXACT_CHUNKS;
        double* h = scratch + (size_t)c * nv * 3;
        double* l = h + nv;
        double* ab = l + nv;
        double* pw = pws + (size_t)c * ns;
        for (uint64_t i = lo; i < hi; ++i) {
            const double x = xy[2 * i], y = xy[2 * i + 1];
            pw[0] = 1.0;
            for (int k = 1; k < ns; ++k) pw[k] = pw[k - 1] * x; /* power *= x (power_sums.cpp:24) */
            for (int k = 0; k < ns; ++k) {
                double sum, err;
                two_sum(h[k], pw[k], &sum, &err); /* plain power */
                h[k] = sum;
                l[k] += err;
                ab[k] += fabs(pw[k]);
                const int a = k / 2, b = k - a;
                const double p = pw[a] * pw[b];
                const double pe = k >= 2 ? fma(pw[a], pw[b], -p) : 0.0; /* exact: p + pe */
                const double pv = k >= 2 ? p : pw[k];
                two_sum(h[ns + k], pv, &sum, &err);
                h[ns + k] = sum;
                l[ns + k] += err + pe;
                ab[ns + k] += fabs(pv);
            }
            for (int j = 0; j < nt; ++j) {
                double sum, err;
                const double p = pw[j] * y; /* rounded as power_sums.cpp:22 */
                two_sum(h[2 * ns + j], p, &sum, &err);
                h[2 * ns + j] = sum;
                l[2 * ns + j] += err;
                ab[2 * ns + j] += fabs(p);
                const double pe = fma(pw[j], y, -p);
                two_sum(h[2 * ns + nt + j], p, &sum, &err);
                h[2 * ns + nt + j] = sum;
                l[2 * ns + nt + j] += err + pe;
                ab[2 * ns + nt + j] += fabs(p);
            }
        }
        double* slot = part + (size_t)c * nv * 3;
        for (int v = 0; v < nv; ++v) {
            const double hh = h[v] + l[v];
            slot[v] = hh;
            slot[nv + v] = l[v] - (hh - h[v]);
            slot[2 * nv + v] = ab[v];
        }
    }
    double* outs[4][3] = {{sp_hi, sp_lo, sp_abs}, {sx_hi, sx_lo, sx_abs}, {tr_hi, tr_lo, tr_abs},
                          {tx_hi, tx_lo, tx_abs}};
    for (int v = 0; v < nv; ++v) {
        double hi = 0.0, lo = 0.0, ab = 0.0;
        for (int c = 0; c < ORC_EXACT_CHUNKS; ++c) {
            const double* slot = part + (size_t)c * nv * 3;
            dd_add(&hi, &lo, slot[v], slot[nv + v]);
            ab += slot[2 * nv + v];
        }
        const int g = v < ns ? 0 : v < 2 * ns ? 1 : v < 2 * ns + nt ? 2 : 3;
        const int idx = v - (g == 0 ? 0 : g == 1 ? ns : g == 2 ? 2 * ns : 2 * ns + nt);
        outs[g][0][idx] = hi;
        outs[g][1][idx] = lo;
        outs[g][2][idx] = ab;
    }
    free(part);
    free(scratch);
    free(pws);
    return ORC_OK;
}

/*
 * Residual moments for checking make_fit_report (diagnostics.cpp:14-48) at
 * scale: residuals r = y - evaluate(poly, x) with the reference's Horner
 * (polynomial.cpp:5-11, no contraction), d = y - shift; out = the exact
 * (double-double, rounded) sums {sum r^2, sum d, sum d^2}. OpenMP over fixed
 * chunks combined in order.
 */
void orc_residual_moments(const double* xy, uint64_t n, const double* coeffs, int degree, double shift,
                          double* out) {
    double part[ORC_EXACT_CHUNKS][6];
#pragma omp parallel for schedule(dynamic, 1)
    for (int c = 0; c < ORC_EXACT_CHUNKS; ++c) {
        const uint64_t lo = n * (uint64_t)c / ORC_EXACT_CHUNKS;
        const uint64_t hi = n * (uint64_t)(c + 1) / ORC_EXACT_CHUNKS;
        double h[3] = {0, 0, 0}, l[3] = {0, 0, 0};
        for (uint64_t i = lo; i < hi; ++i) {
            const double x = xy[2 * i], y = xy[2 * i + 1];
            double acc = coeffs[degree];
            for (int k = degree - 1; k >= 0; --k) acc = acc * x + coeffs[k];
            const double r = y - acc, d = y - shift;
            const double v[3] = {r * r, d, d * d};
            for (int j = 0; j < 3; ++j) {
                double sum, err;
                two_sum(h[j], v[j], &sum, &err);
                h[j] = sum;
                l[j] += err;
            }
        }
        for (int j = 0; j < 3; ++j) {
            part[c][2 * j] = h[j];
            part[c][2 * j + 1] = l[j];
        }
    }
    for (int j = 0; j < 3; ++j) {
        double hi = 0.0, lo = 0.0;
        for (int c = 0; c < ORC_EXACT_CHUNKS; ++c) dd_add(&hi, &lo, part[c][2 * j], part[c][2 * j + 1]);
        out[j] = hi + lo;
    }
}

/* tests/support/oracles.hpp:19-51: KahanSum of std::pow(x, k) and pow(x, j)*y. */
void orc_kahan_pow_sums(const double* xy, uint64_t n, int degree, double* s, double* t) {
    const int ns = 2 * degree + 1, nt = degree + 1;
    double sc[25], tc[13];
    for (int k = 0; k < ns; ++k) s[k] = sc[k] = 0.0;
    for (int j = 0; j < nt; ++j) t[j] = tc[j] = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        const double x = xy[2 * i], yv = xy[2 * i + 1];
        for (int k = 0; k < ns; ++k) {
            const double v = pow(x, k);
            const double yk = v - sc[k];
            const double tt = s[k] + yk;
            sc[k] = (tt - s[k]) - yk;
            s[k] = tt;
        }
        for (int j = 0; j < nt; ++j) {
            const double v = pow(x, j) * yv;
            const double yk = v - tc[j];
            const double tt = t[j] + yk;
            tc[j] = (tt - t[j]) - yk;
            t[j] = tt;
        }
    }
}

/* Batched reference: per curve accumulate -> build_normal_system -> solve_gaussian. */
void orc_fit_batched(const double* xy, uint64_t n_curves, uint32_t ppc, int degree,
                     double* coeffs, int32_t* status) {
    const int dim = degree + 1;
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < (int64_t)n_curves; ++c) {
        double s[25], t[13], a[169], x[13];
        const double* base = xy + (size_t)c * ppc * 2;
        int st = orc_accumulate(base, ppc, degree, s, t);
        if (st == ORC_OK) {
            orc_build_normal_system(s, degree, a);
            st = orc_solve_gaussian(a, t, dim, x);
        }
        status[c] = st;
        for (int k = 0; k < dim; ++k) coeffs[(size_t)c * dim + k] = st == ORC_OK ? x[k] : 0.0;
    }
}

/* ---------------------------------------------------------------------------
 * Counter-based synthetic generator (host twin of csrc/synth.cuh). SplitMix64
 * jumped to a counter; uniforms from the top 53 bits as synthetic.cpp:13-15.
 * Only integer ops and correctly rounded + - x (no libm, no contraction).
 * ------------------------------------------------------------------------- */

#define GOLDEN 0x9E3779B97F4A7C15ULL
#define STREAM_X 0x5859ULL
#define STREAM_TRUTH 0x54525554ULL
#define SQRT3 1.7320508075688772

static inline uint64_t smix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
    return smix(seed * GOLDEN + stream);
}
static inline double u53(uint64_t key, uint64_t ctr) {
    return (double)(smix(key + (ctr + 1) * GOLDEN) >> 11) * 0x1.0p-53;
}

void orc_synth_truth(uint64_t seed, uint64_t curve, int truth_degree, double* coeffs) {
    const uint64_t key = stream_key(seed, STREAM_TRUTH);
    for (int k = 0; k <= truth_degree; ++k)
        coeffs[k] = -10.0 + 20.0 * u53(key, curve * 13 + (uint64_t)k); /* synthetic.cpp:27 */
}

static inline double synth_y(const double* c, int truth_degree, double x, double sigma,
                             uint64_t key, uint64_t g) {
    double acc = c[truth_degree];
    for (int k = truth_degree - 1; k >= 0; --k) acc = acc * x + c[k];
    const double u1 = u53(key, 5 * g + 1), u2 = u53(key, 5 * g + 2);
    const double u3 = u53(key, 5 * g + 3), u4 = u53(key, 5 * g + 4);
    const double z = (((u1 + u2) + (u3 + u4)) - 2.0) * SQRT3;
    return acc + sigma * z;
}

void orc_synth(double* xy, uint64_t n, uint64_t offset, uint64_t seed, int truth_degree,
               double sigma) {
    double c[13];
    orc_synth_truth(seed, 0, truth_degree, c);
    const uint64_t key = stream_key(seed, STREAM_X);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) {
        const uint64_t g = offset + (uint64_t)i;
        const double x = 2.0 * u53(key, 5 * g) - 1.0;
        xy[2 * i] = x;
        xy[2 * i + 1] = synth_y(c, truth_degree, x, sigma, key, g);
    }
}

void orc_synth_batched(double* xy, uint64_t n_curves, uint32_t ppc, uint64_t seed,
                       int truth_degree, double sigma) {
    const uint64_t key = stream_key(seed, STREAM_X);
#pragma omp parallel for schedule(static)
    for (int64_t cv = 0; cv < (int64_t)n_curves; ++cv) {
        double c[13];
        orc_synth_truth(seed, (uint64_t)cv, truth_degree, c);
        for (uint32_t j = 0; j < ppc; ++j) {
            const uint64_t g = (uint64_t)cv * ppc + j;
            const double x = 2.0 * u53(key, 5 * g) - 1.0;
            xy[2 * g] = x;
            xy[2 * g + 1] = synth_y(c, truth_degree, x, sigma, key, g);
        }
    }
}

/* ---------------------------------------------------------------------------
 * generate_synthetic restatement (src/synthetic.cpp:13-56) with a C
 * mt19937_64 (Matsumoto & Nishimura 2004; the parameters std::mt19937_64
 * fixes in [rand.predef]).
 * ------------------------------------------------------------------------- */

typedef struct {
    uint64_t mt[312];
    int mti;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->mti = 312;
}

static uint64_t mt64_next(mt64* g) {
    static const uint64_t mag[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (g->mti >= 312) {
        int i;
        uint64_t x;
        for (i = 0; i < 312 - 156; ++i) {
            x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
            g->mt[i] = g->mt[i + 156] ^ (x >> 1) ^ mag[x & 1ULL];
        }
        for (; i < 311; ++i) {
            x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
            g->mt[i] = g->mt[i + (156 - 312)] ^ (x >> 1) ^ mag[x & 1ULL];
        }
        x = (g->mt[311] & UM) | (g->mt[0] & LM);
        g->mt[311] = g->mt[155] ^ (x >> 1) ^ mag[x & 1ULL];
        g->mti = 0;
    }
    uint64_t x = g->mt[g->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

static double mt_uniform01(mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; }

static double mt_standard_normal(mt64* g) { /* synthetic.cpp:19-23 */
    const double u1 = 1.0 - mt_uniform01(g);
    const double u2 = mt_uniform01(g);
    const double pi = 3.141592653589793;
    return sqrt(-2.0 * log(u1)) * cos(2.0 * pi * u2);
}

int orc_generate_synthetic(uint64_t n, int degree, double sigma, uint64_t seed, double* xy) {
    if (n < 2 || degree < 0 || !(sigma >= 0.0)) return ORC_EINVAL;
    mt64* g = (mt64*)malloc(sizeof(mt64));
    if (!g) return ORC_EINVAL;
    mt64_seed(g, seed);
    double c[64];
    if (degree > 63) { free(g); return ORC_EINVAL; }
    for (int k = 0; k <= degree; ++k) c[k] = -10.0 + 20.0 * mt_uniform01(g); /* :25-29 */
    for (uint64_t i = 0; i < n; ++i) xy[2 * i] = mt_uniform01(g);         /* :50 */
    for (uint64_t i = 0; i < n; ++i) {                                     /* :51-54 */
        const double x = xy[2 * i];
        double acc = c[degree]; /* evaluate(), src/polynomial.cpp:5-11 */
        for (int k = degree - 1; k >= 0; --k) acc = acc * x + c[k];
        double y = acc;
        if (sigma > 0.0) y += sigma * mt_standard_normal(g);
        xy[2 * i + 1] = y;
    }
    free(g);
    return ORC_OK;
}

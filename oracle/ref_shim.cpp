// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers around the reference's own C++ API so Python tests,
// oracle/make_golden.py and bench.py's reference arm can call the compiled
// reference (oracle/_ref/libref_lsqfit.so, built by oracle/Makefile from the
// unmodified sources under /root/reference/proj/src). No reference code is
// copied here; this file only calls it.
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <vector>

#include "lsqfit/dataset.hpp"
#include "lsqfit/diagnostics.hpp"
#include "lsqfit/errors.hpp"
#include "lsqfit/normal_backend.hpp"
#include "lsqfit/qr_backend.hpp"
#include "lsqfit/power_sums.hpp"
#include "lsqfit/synthetic.hpp"
#include "support/oracles.hpp"

namespace {

enum { OK = 0, EINVAL_ = 1, EOVERFLOW_ = 2, ESINGULAR_ = 3, EDEGREE_ = 4, ERANKDEF_ = 7, EOTHER_ = 9 };

template <class F>
int guarded(F&& f) {
    try {
        f();
        return OK;
    } catch (const lsqfit::OverflowError&) {
        return EOVERFLOW_;
    } catch (const lsqfit::SingularSystemError&) {
        return ESINGULAR_;
    } catch (const lsqfit::DegreeTooHighError&) {
        return EDEGREE_;
    } catch (const lsqfit::RankDeficientError&) {
        return ERANKDEF_;
    } catch (const std::invalid_argument&) {
        return EINVAL_;
    } catch (...) {
        return EOTHER_;
    }
}

std::vector<lsqfit::Point> to_points(const double* xy, std::uint64_t n) {
    const auto* p = reinterpret_cast<const lsqfit::Point*>(xy);  // same AoS layout (dataset.hpp:10-13)
    return std::vector<lsqfit::Point>(p, p + n);                   // one copying pass, no zero-fill
}

void copy_sums(const lsqfit::PowerSums& p, double* s, double* t) {
    std::memcpy(s, p.s.data(), p.s.size() * sizeof(double));
    std::memcpy(t, p.t.data(), p.t.size() * sizeof(double));
}

}  // namespace

extern "C" {

// A Dataset built once (untimed) so timed calls exclude the O(n) copy+validation.
void* ref_dataset_new(const double* xy, std::uint64_t n) {
    try {
        return new lsqfit::Dataset(to_points(xy, n));
    } catch (...) {
        return nullptr;
    }
}
void ref_dataset_free(void* d) { delete static_cast<lsqfit::Dataset*>(d); }

int ref_accumulate_ds(void* d, int degree, double* s, double* t) {
    return guarded([&] { copy_sums(lsqfit::accumulate(*static_cast<lsqfit::Dataset*>(d), degree), s, t); });
}

int ref_accumulate_parallel_ds(void* d, int degree, int chunks, double* s, double* t) {
    return guarded([&] {
        copy_sums(lsqfit::accumulate_parallel(*static_cast<lsqfit::Dataset*>(d), degree, chunks), s, t);
    });
}

// accumulate_parallel -> build_normal_system -> solve_gaussian (the fit's numeric core).
int ref_fit_sums_solve_ds(void* d, int degree, int chunks, double* s, double* t, double* coeffs) {
    return guarded([&] {
        const auto& ds = *static_cast<lsqfit::Dataset*>(d);
        const lsqfit::PowerSums p = chunks == 1 ? lsqfit::accumulate(ds, degree)
                                                : lsqfit::accumulate_parallel(ds, degree, chunks);
        copy_sums(p, s, t);
        const lsqfit::Polynomial poly = lsqfit::solve_gaussian(lsqfit::build_normal_system(p));
        std::memcpy(coeffs, poly.coefficients().data(), poly.coefficients().size() * sizeof(double));
    });
}

// fit_normal (normal_backend.cpp:76-85) on a prebuilt Dataset: sums + solve +
// make_fit_report (residual vector, SSE, R).
int ref_fit_normal_ds(void* d, int degree, int chunks, double* coeffs, double* sse, double* r) {
    return guarded([&] {
        const lsqfit::FitReport rep = lsqfit::fit_normal(*static_cast<lsqfit::Dataset*>(d), degree, chunks);
        const auto& c = rep.polynomial.coefficients();
        std::memcpy(coeffs, c.data(), c.size() * sizeof(double));
        *sse = rep.sse;
        *r = rep.r;
    });
}

int ref_accumulate(const double* xy, std::uint64_t n, int degree, double* s, double* t) {
    return guarded([&] { copy_sums(lsqfit::accumulate(lsqfit::Dataset(to_points(xy, n)), degree), s, t); });
}

int ref_accumulate_parallel(const double* xy, std::uint64_t n, int degree, int chunks, double* s,
                            double* t) {
    return guarded([&] {
        copy_sums(lsqfit::accumulate_parallel(lsqfit::Dataset(to_points(xy, n)), degree, chunks), s, t);
    });
}

int ref_solve_gaussian(const double* a, const double* b, int dim, double* x) {
    return guarded([&] {
        lsqfit::NormalSystem sys;
        sys.degree = dim - 1;
        sys.a = lsqfit::DenseMatrix(static_cast<std::size_t>(dim), static_cast<std::size_t>(dim));
        for (int i = 0; i < dim; ++i)
            for (int j = 0; j < dim; ++j) sys.a(i, j) = a[i * dim + j];
        sys.b.assign(b, b + dim);
        const lsqfit::Polynomial p = lsqfit::solve_gaussian(std::move(sys));
        std::memcpy(x, p.coefficients().data(), static_cast<std::size_t>(dim) * sizeof(double));
    });
}

// Solve from given power sums (s: 2m+1, t: m+1), via build_normal_system.
int ref_solve_from_sums(const double* s, const double* t, int degree, double* x) {
    return guarded([&] {
        lsqfit::PowerSums p;
        p.degree = degree;
        p.s.assign(s, s + 2 * degree + 1);
        p.t.assign(t, t + degree + 1);
        p.n = static_cast<std::size_t>(s[0]);
        const lsqfit::Polynomial poly = lsqfit::solve_gaussian(lsqfit::build_normal_system(p));
        std::memcpy(x, poly.coefficients().data(), static_cast<std::size_t>(degree + 1) * sizeof(double));
    });
}

int ref_fit_normal(const double* xy, std::uint64_t n, int degree, int chunks, double* coeffs,
                   double* sse, double* r) {
    return guarded([&] {
        const lsqfit::FitReport rep = lsqfit::fit_normal(lsqfit::Dataset(to_points(xy, n)), degree, chunks);
        const auto& c = rep.polynomial.coefficients();
        std::memcpy(coeffs, c.data(), c.size() * sizeof(double));
        *sse = rep.sse;
        *r = rep.r;
    });
}

// fit_qr (qr_backend.cpp:126-133): Householder QR cross-check backend.
int ref_fit_qr(const double* xy, std::uint64_t n, int degree, double* coeffs, double* sse, double* r) {
    return guarded([&] {
        const lsqfit::FitReport rep = lsqfit::fit_qr(lsqfit::Dataset(to_points(xy, n)), degree);
        const auto& c = rep.polynomial.coefficients();
        std::memcpy(coeffs, c.data(), c.size() * sizeof(double));
        *sse = rep.sse;
        *r = rep.r;
    });
}

int ref_generate_synthetic(std::uint64_t n, int degree, double sigma, std::uint64_t seed, double* xy) {
    return guarded([&] {
        const lsqfit::Dataset d = lsqfit::generate_synthetic(n, degree, sigma, seed);
        std::memcpy(xy, d.points().data(), n * sizeof(lsqfit::Point));
    });
}

// The batched CPU baseline: the reference has no batched
// API, so an OpenMP loop over curves runs its per-curve path — Dataset (the
// curve's points copied in, 16 B/pt, included in the time), accumulate,
// build_normal_system, solve_gaussian. Status per curve: 0 ok, else the
// guarded() code (2 overflow, 3 singular, ...).
void ref_fit_batched(const double* xy, std::uint64_t n_curves, std::uint32_t ppc, int degree, double* coeffs,
                     std::int32_t* status) {
    const std::size_t dim = static_cast<std::size_t>(degree) + 1;
#pragma omp parallel for schedule(static)
    for (std::int64_t c = 0; c < static_cast<std::int64_t>(n_curves); ++c) {
        double* out = coeffs + static_cast<std::size_t>(c) * dim;
        status[c] = guarded([&] {
            const lsqfit::Dataset d(to_points(xy + 2 * static_cast<std::size_t>(c) * ppc, ppc));
            const lsqfit::Polynomial poly =
                lsqfit::solve_gaussian(lsqfit::build_normal_system(lsqfit::accumulate(d, degree)));
            std::memcpy(out, poly.coefficients().data(), dim * sizeof(double));
        });
        if (status[c] != OK)
            for (std::size_t k = 0; k < dim; ++k) out[k] = 0.0;
    }
}

// tests/support/oracles.hpp:40-51
int ref_accumulate_oracle(const double* xy, std::uint64_t n, int degree, double* s, double* t) {
    return guarded([&] {
        const testsupport::OracleSums o = testsupport::accumulate_oracle(lsqfit::Dataset(to_points(xy, n)), degree);
        std::memcpy(s, o.s.data(), o.s.size() * sizeof(double));
        std::memcpy(t, o.t.data(), o.t.size() * sizeof(double));
    });
}

}  // extern "C"

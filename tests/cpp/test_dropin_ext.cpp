// tests/cpp/test_dropin_ext.cpp — checks of the B200 drop-in that the
// reference suites do not reach: the lsqfit::cuda extensions (device
// selection, batched fit), the diagnostics entry points and the error
// mapping. Built by the top-level Makefile, run by tests/test_gpu_dropin.py.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "lsqfit/cuda.hpp"
#include "lsqfit/diagnostics.hpp"
#include "lsqfit/errors.hpp"
#include "lsqfit/normal_backend.hpp"
#include "lsqfit/power_sums.hpp"

using namespace lsqfit;

namespace {
std::vector<Point> line_points(std::size_t n, double a0, double a1) {
    std::vector<Point> pts(n);
    for (std::size_t i = 0; i < n; ++i) {
        const double x = -1.0 + 2.0 * static_cast<double>(i) / static_cast<double>(n);
        pts[i] = {x, a0 + a1 * x};
    }
    return pts;
}
}  // namespace

TEST_CASE("device selection and a basic fit") {
    cuda::set_device(0);
    const FitReport rep = fit_normal(Dataset(line_points(1000, 2.0, -3.0)), 1);
    CHECK(std::fabs(rep.polynomial.coefficients()[0] - 2.0) <= 1e-12);
    CHECK(std::fabs(rep.polynomial.coefficients()[1] + 3.0) <= 1e-12);
    CHECK(rep.sse <= 1e-20);
    CHECK(rep.r == doctest::Approx(1.0));
    CHECK(rep.n_points == 1000);
    CHECK(rep.residuals.size() == 1000);
}

TEST_CASE("batched fit: exact lines per curve, singular and overflow flags") {
    const std::size_t curves = 300;
    const std::uint32_t ppc = 256;
    std::vector<Point> pts;
    pts.reserve(curves * ppc);
    for (std::size_t c = 0; c < curves; ++c) {
        const auto line = line_points(ppc, static_cast<double>(c), 0.5);
        pts.insert(pts.end(), line.begin(), line.end());
    }
    for (std::uint32_t j = 0; j < ppc; ++j) pts[ppc + j].x = 0.25;  // curve 1: one distinct x
    pts[2 * ppc].x = 1e200;                                          // curve 2: overflow
    const cuda::BatchedFit b = cuda::fit_batched(pts, curves, ppc, 1);
    REQUIRE(b.status.size() == curves);
    CHECK(b.status[0] == 0);
    CHECK(b.status[1] == 3);
    CHECK(b.status[2] == 2);
    for (std::size_t c = 3; c < curves; ++c) {
        CHECK(b.status[c] == 0);
        CHECK(std::fabs(b.coeffs[2 * c] - static_cast<double>(c)) <= 1e-11 * (1.0 + c));
        CHECK(std::fabs(b.coeffs[2 * c + 1] - 0.5) <= 1e-11 * (1.0 + c));
    }
    CHECK_THROWS_AS(cuda::fit_batched(pts, curves + 1, ppc, 1), std::invalid_argument);
}

TEST_CASE("diagnostics entry points") {
    const Dataset d({{0.0, 1.0}, {1.0, 2.0}, {2.0, 4.0}, {3.0, 5.0}});
    const Polynomial p({1.0, 1.0});
    const std::vector<double> r = residuals(d, p);
    REQUIRE(r.size() == 4);
    CHECK(r[0] == 0.0);
    CHECK(r[2] == 1.0);
    CHECK(r[3] == 1.0);
    CHECK(sum_squared_error(r) == 2.0);
    const double rr = correlation_coefficient(d, 2.0);  // mean 3, sst = 10
    CHECK(rr == doctest::Approx(std::sqrt(1.0 - 2.0 / 10.0)).epsilon(1e-14));
    const FitReport rep = make_fit_report(d, p, FitBackend::HouseholderQR);
    CHECK(rep.sse == 2.0);
    CHECK(std::string(backend_name(rep.backend)) == "qr");
    const Dataset constant({{0.0, 3.0}, {1.0, 3.0}});
    CHECK(correlation_coefficient(constant, 0.0) == 1.0);
    CHECK(correlation_coefficient(constant, 1.0) == 0.0);
    CHECK_THROWS_AS(make_fit_report(Dataset({{1e300, 1.0}}), Polynomial({0.0, 0.0, 1.0}), FitBackend::NormalEquations),
                    OverflowError);
}

TEST_CASE("TSQR cross-check fit") {
    const FitReport rep = cuda::fit_qr_tsqr(Dataset(line_points(4096, -1.5, 0.25)), 3);
    CHECK(rep.backend == FitBackend::HouseholderQR);
    CHECK(std::fabs(rep.polynomial.coefficients()[0] + 1.5) <= 1e-12);
    CHECK(std::fabs(rep.polynomial.coefficients()[1] - 0.25) <= 1e-12);
    CHECK(std::fabs(rep.polynomial.coefficients()[2]) <= 1e-12);
    CHECK(std::fabs(rep.polynomial.coefficients()[3]) <= 1e-12);
    CHECK_THROWS_AS(cuda::fit_qr_tsqr(Dataset({{2.0, 1.0}, {2.0, 2.0}, {2.0, 3.0}}), 1), RankDeficientError);
    CHECK_THROWS_AS(cuda::fit_qr_tsqr(Dataset({{0.0, 1.0}, {1.0, 2.0}}), 13), DegreeTooHighError);
}

TEST_CASE("device groups shard host datasets (emulated with repeated device ids)") {
    std::vector<Point> pts(1000003);
    for (std::size_t i = 0; i < pts.size(); ++i) {
        const double x = -1.0 + 2.0 * static_cast<double>((i * 7919) % pts.size()) / static_cast<double>(pts.size());
        pts[i] = {x, 1.0 + x - 0.5 * x * x * x};
    }
    const Dataset d(pts);
    cuda::set_devices({0});
    const PowerSums one = accumulate(d, 3);
    const FitReport f1 = fit_normal(d, 3);
    for (const std::vector<int>& devs : {std::vector<int>{0, 0}, std::vector<int>{0, 0, 0}}) {
        cuda::set_devices(devs);
        const PowerSums g = accumulate(d, 3);
        CHECK(g.n == pts.size());
        CHECK(g.s[0] == static_cast<double>(pts.size()));
        for (std::size_t k = 0; k < g.s.size(); ++k)
            CHECK(std::fabs(g.s[k] - one.s[k]) <= 1e-13 * (1.0 + std::fabs(one.s[k])));
        const FitReport fg = fit_normal(d, 3);
        for (int k = 0; k < 4; ++k)
            CHECK(std::fabs(fg.polynomial.coefficients()[k] - f1.polynomial.coefficients()[k]) <= 1e-12);
        CHECK(fg.residuals.size() == pts.size());
        CHECK(std::fabs(fg.sse - f1.sse) <= 1e-9 * (1.0 + f1.sse));
        CHECK(fg.r == doctest::Approx(f1.r).epsilon(1e-12));
    }
    cuda::set_device(0);
}

TEST_CASE("reference-order mode reproduces the reference's bits (Table I golden values)") {
    const Dataset t1({{39.206, 751.912}, {29.74, 567.121}, {21.31, 403.746},
                      {12.087, 221.738}, {1.812, 18.8418}, {0.001, 1.88672}});
    cuda::set_reference_order(true);
    const PowerSums p = accumulate(t1, 3);
    // the reference's degree-3 sums and coefficients on Table I
    const std::vector<double> s = {6, 104.15600000000001, 3025.07305, 98017.038830648002, 3372567.5558183366,
                                   120550025.81553388, 4420414550.8308372};
    const std::vector<double> t = {1965.2455199999999, 57663.758106319998, 1873176.2942356199, 64529583.154778928};
    CHECK(p.s == s);
    CHECK(p.t == t);
    const FitReport r = fit_normal(t1, 3);
    const std::vector<double> c = {-4.7551083966032817, 17.51093799773647, 0.10857202524918211,
                                   -0.0016173860909198452};
    CHECK(r.polynomial.coefficients() == c);
    CHECK(r.sse == doctest::Approx(128.1995753700682).epsilon(1e-12));
    cuda::set_reference_order(false);
}

TEST_CASE("accumulate above the fused kernels' degree cap (the reference has none)") {
    const Dataset d({{0.5, 1.0}, {-0.25, 2.0}, {1.0, -1.0}});
    const PowerSums p = accumulate(d, 15);
    CHECK(p.degree == 15);
    CHECK(p.s.size() == 31);
    CHECK(p.t.size() == 16);
    CHECK(p.s[0] == 3.0);
    // x in {0.5, -0.25, 1}: every term is a power of two, the sums are exact
    double xk[3] = {1.0, 1.0, 1.0};
    const double x[3] = {0.5, -0.25, 1.0}, y[3] = {1.0, 2.0, -1.0};
    for (int k = 1; k <= 30; ++k) {
        double s = 0.0, t = 0.0;
        for (int i = 0; i < 3; ++i) {
            xk[i] *= x[i];
            s += xk[i];
            t += xk[i] * y[i];
        }
        CHECK(p.s[k] == s);
        if (k <= 15) CHECK(p.t[k] == t);
    }
    CHECK(accumulate_parallel(d, 15, 4).s == p.s);
    // the report pass takes any degree too: residuals bit-identical to Horner
    std::vector<double> c(21);
    for (int k = 0; k <= 20; ++k) c[k] = 1.0 / (k + 1);
    const Polynomial poly(c);
    const std::vector<double> r = residuals(d, poly);
    for (int i = 0; i < 3; ++i) CHECK(r[i] == y[i] - evaluate(poly, x[i]));
    const FitReport rep = make_fit_report(d, poly, FitBackend::NormalEquations);
    CHECK(rep.residuals == r);
}

TEST_CASE("fit_batched_ragged: curves of different lengths") {
    // curve 0: 4 points on y = 1 + 2x; curve 1: empty; curve 2: 3 points on y = -x + 0.5x^2 (m = 2: exact);
    // curve 3: 2 points on y = 3 (m = 1)
    std::vector<Point> pts = {{0.0, 1.0}, {1.0, 3.0}, {2.0, 5.0}, {3.0, 7.0},
                              {0.0, 0.0}, {1.0, -0.5}, {2.0, 0.0},
                              {-1.0, 3.0}, {1.0, 3.0}};
    const std::vector<std::uint64_t> offsets = {0, 4, 4, 7, 9};
    const cuda::BatchedFit f1 = cuda::fit_batched_ragged(pts, offsets, 1);
    CHECK(f1.status[0] == 0);
    CHECK(f1.coeffs[0] == doctest::Approx(1.0).epsilon(1e-12));
    CHECK(f1.coeffs[1] == doctest::Approx(2.0).epsilon(1e-12));
    CHECK(f1.status[1] == 3);  // empty curve: singular, as a reference Dataset of no points cannot be fitted
    CHECK(f1.status[3] == 0);
    CHECK(f1.coeffs[6] == doctest::Approx(3.0).epsilon(1e-12));
    const cuda::BatchedFit f2 = cuda::fit_batched_ragged(pts, offsets, 2);
    CHECK(f2.status[2] == 0);
    CHECK(f2.coeffs[6] == doctest::Approx(0.0).epsilon(1e-12));
    CHECK(f2.coeffs[7] == doctest::Approx(-1.0).epsilon(1e-12));
    CHECK(f2.coeffs[8] == doctest::Approx(0.5).epsilon(1e-12));
    CHECK(f2.status[3] == 3);  // 2 points, 3 unknowns
    CHECK_THROWS_AS(cuda::fit_batched_ragged(pts, {0, 5, 4}, 1), std::invalid_argument);
}

TEST_CASE("error mapping of the C ABI statuses") {
    const Dataset d({{0.0, 0.0}, {1.0, 1.0}});
    CHECK_THROWS_AS(accumulate(d, -1), std::invalid_argument);
    CHECK_THROWS_AS(accumulate(d, 16385), std::invalid_argument);  // past the any-degree kernel's range
    CHECK_THROWS_AS(fit_normal(d, 13), DegreeTooHighError);
    CHECK_THROWS_AS(accumulate(Dataset({{1e200, 1.0}, {1.0, 1.0}}), 2), OverflowError);
    NormalSystem bad;
    bad.a = DenseMatrix(2, 3);
    bad.b = {1.0, 2.0};
    CHECK_THROWS_AS(solve_gaussian(bad), std::invalid_argument);
}

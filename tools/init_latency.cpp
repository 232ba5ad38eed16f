// Dev probe (C++ drop-in): first fit_normal wall time in a fresh process.
#include <chrono>
#include <cstdio>
#include "lsqfit/normal_backend.hpp"
int main() {
    using C = std::chrono::steady_clock;
    const auto t0 = C::now();
    const lsqfit::Dataset d({{39.206, 751.912}, {29.74, 567.121}, {21.31, 403.746}, {12.087, 221.738}, {1.812, 18.8418}, {0.001, 1.88672}});
    const auto rep = lsqfit::fit_normal(d, 1);
    const auto t1 = C::now();
    const auto rep2 = lsqfit::fit_normal(d, 1);
    const auto t2 = C::now();
    std::printf("first_fit_s %.4f second_fit_ms %.4f a0 %.10f a1 %.10f\n", std::chrono::duration<double>(t1 - t0).count(),
                std::chrono::duration<double, std::milli>(t2 - t1).count(), rep2.polynomial.coefficients()[0],
                rep.polynomial.coefficients()[1]);
}

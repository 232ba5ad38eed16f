// Dev probe: where the first call's wall time goes in a fresh process (the
// reference acceptance harness's degree-1 criterion allows < 1 s including
// CUDA initialisation, acceptance.cpp:125-140).
//   g++ -O2 -Iinclude -I/usr/local/cuda/include tools/init_breakdown.cpp -o tools/init_breakdown \
//       -Lpaper_1512_08017_b200/lib -llsqfit_cuda -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_1512_08017_b200/lib
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>

#include "lsqfit_cuda.h"

int main() {
    using C = std::chrono::steady_clock;
    auto ms = [](C::time_point a, C::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const double xy[12] = {39.206, 751.912, 29.74, 567.121, 21.31, 403.746, 12.087, 221.738, 1.812, 18.8418, 0.001, 1.88672};
    const auto t0 = C::now();
    cudaFree(nullptr);
    const auto t1 = C::now();
    lsqfit_cuda_ctx* ctx = nullptr;
    int st = lsqfit_cuda_create(&ctx, 0);
    const auto t2 = C::now();
    lsqfit_result r{};
    lsqfit_diag d{};
    double res[6];
    st |= lsqfit_cuda_fit_report_host(ctx, xy, 6, 1, &r, &d, res);
    const auto t3 = C::now();
    st |= lsqfit_cuda_fit_report_host(ctx, xy, 6, 1, &r, &d, res);
    const auto t4 = C::now();
    st |= lsqfit_cuda_fit_report_host(ctx, xy, 6, 2, &r, &d, res);
    const auto t5 = C::now();
    std::printf("{\"cuda_init_ms\": %.2f, \"ctx_create_ms\": %.2f, \"first_fit_report_ms\": %.2f, "
                "\"second_fit_report_ms\": %.3f, \"first_m2_ms\": %.3f, \"status\": %d, \"a1\": %.12g}\n",
                ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4), ms(t4, t5), st, r.coeffs[1]);
    lsqfit_cuda_destroy(ctx);
    return st;
}

// Dev probe: cudaFree(0) wall time with only cudart linked (compare
// tools/init_breakdown, which also links liblsqfit_cuda.so and its fatbin).
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
int main() {
    const auto t0 = std::chrono::steady_clock::now();
    cudaFree(nullptr);
    const auto t1 = std::chrono::steady_clock::now();
    std::printf("{\"cudart_only_cudaFree0_ms\": %.2f}\n", std::chrono::duration<double, std::milli>(t1 - t0).count());
}

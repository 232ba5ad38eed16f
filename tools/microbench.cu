// tools/microbench.cu — measures the roofline denominators this path needs
// that MEASURED_PEAKS.json lacks: FP64 pipe throughput (DFMA, DADD) and a
// read-only HBM streaming ceiling (LDG.128, 16 B/elem, sum-reduce). Not product code.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
        x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
        x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void dadd_loop(double* out, int iters, double a) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
        x0 = __dadd_rn(x0, a); x1 = __dadd_rn(x1, a); x2 = __dadd_rn(x2, a); x3 = __dadd_rn(x3, a);
        x4 = __dadd_rn(x4, a); x5 = __dadd_rn(x5, a); x6 = __dadd_rn(x6, a); x7 = __dadd_rn(x7, a);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void read_stream(const double2* __restrict__ in, size_t n, double* out) {
    double acc = 0;
    size_t stride = size_t(gridDim.x) * blockDim.x;
    size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n; i += 4 * stride) {
        double2 a = __ldg(in + i), b = __ldg(in + i + stride), c = __ldg(in + i + 2 * stride), d = __ldg(in + i + 3 * stride);
        acc += a.x + a.y + b.x + b.y + c.x + c.y + d.x + d.y;
    }
    for (; i < n; i += stride) { double2 a = __ldg(in + i); acc += a.x + a.y; }
    if (acc == 1234.5) out[0] = acc;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 1 << 16;
    for (int pass = 0; pass < 2; ++pass) {
        for (int which = 0; which < 2; ++which) {
            cudaEventRecord(e0);
            if (which == 0) dfma_loop<<<sms * 8, 256>>>(out, iters, 0.999, 1e-3);
            else dadd_loop<<<sms * 8, 256>>>(out, iters, 1e-3);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double ops = double(sms) * 8 * 256 * iters * 8;
            if (pass == 1)
                printf("{\"probe\": \"%s\", \"ops_per_s\": %.4e, \"per_sm_per_clk_at_max\": %.2f}\n",
                       which == 0 ? "dfma" : "dadd", ops / (ms * 1e-3), ops / (ms * 1e-3) / sms / (clk * 1e3));
        }
    }
    size_t n = size_t(1) << 31;  // 2^31 points = 32 GiB
    double2* in; if (cudaMalloc(&in, n * 16) != cudaSuccess) { n >>= 2; cudaMalloc(&in, n * 16); }
    cudaMemset(in, 0, n * 16);
    float best = 1e30;
    for (int r = 0; r < 6; ++r) {
        cudaEventRecord(e0);
        read_stream<<<sms * 8, 256>>>(in, n, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
    }
    printf("{\"probe\": \"read_stream_ldg128\", \"bytes\": %zu, \"GB_per_s\": %.1f}\n", n * 16, n * 16 / (best * 1e-3) / 1e9);
    printf("{\"probe\": \"device\", \"sms\": %d, \"clock_khz\": %d, \"err\": \"%s\"}\n", sms, clk, cudaGetErrorString(cudaGetLastError()));
    return 0;
}

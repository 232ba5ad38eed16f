// Dev probe: dependent-chain latency of DADD / DMUL and of an LDS -> DADD
// chain on sm_100a (one thread, clock64). nvcc -O3 -arch=sm_100a --fmad=false
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(double* out, long long* cyc, double a, double b, int iters) {
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 32; ++k) x = __dadd_rn(x, b);
    }
    long long t1 = clock64();
    double y = a;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 32; ++k) y = __dmul_rn(y, b);
    }
    long long t2 = clock64();
    __shared__ double s[64];
    if (threadIdx.x < 64) s[threadIdx.x] = b * threadIdx.x;
    __syncwarp();
    double z = a;
    long long t3 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 32; ++k) z = __dadd_rn(z, s[(k + i) & 63]);
    }
    long long t4 = clock64();
    out[0] = x + y + z;
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t4 - t3;
}

int main() {
    double* d;
    long long* c;
    cudaMalloc(&d, 8);
    cudaMalloc(&c, 24);
    const int iters = 1 << 14;
    chain<<<1, 32>>>(d, c, 1.0, 1e-300, iters);
    chain<<<1, 32>>>(d, c, 1.0, 1e-300, iters);
    long long h[3];
    cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
    const double n = 32.0 * iters;
    printf("{\"dadd_dep_latency_cyc\": %.2f, \"dmul_dep_latency_cyc\": %.2f, \"lds_fed_dadd_chain_cyc\": %.2f}\n",
           h[0] / n, h[1] / n, h[2] / n);
    return 0;
}

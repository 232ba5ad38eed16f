// tools/stream_balance.cu — dev probe, not product code. Does a persistent
// TMA-ring read stream (the power_sums_kernel feed: 1 CTA/SM, producer lane +
// 7 consumer warps, 56 KB tiles, 3-4 stage ring) lose time to per-SM bandwidth
// unfairness under a STATIC tile partition? Compares static round-robin,
// static contiguous and dynamic (atomic tile counter) dealing of the same
// tiles, and reports each CTA's finish-time spread.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/stream_balance tools/stream_balance.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int kCW = 7, kThreads = 256, kP = 16, kTile = kCW * 32 * kP;  // points (16 B each)
constexpr int kStages = 3;

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t ph) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(ok)
                     : "r"(sa(b)), "r"(ph)
                     : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(d)),
                 "l"(s), "r"(bytes), "r"(sa(b))
                 : "memory");
}
__device__ __forceinline__ uint64_t gtime() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// mode 0: round-robin static, 1: contiguous static, 2: dynamic counter
__global__ void __launch_bounds__(kThreads, 1)
    stream(const double2* xy, uint64_t n_tiles, int mode, unsigned* counter, double* out, uint64_t* fin,
           uint64_t n_static, int K) {
    extern __shared__ __align__(128) unsigned char sm[];
    double2* ring = reinterpret_cast<double2*>(sm);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + kStages * kTile * 16);
    uint64_t* empty = full + kStages;
    long long* tid_of = reinterpret_cast<long long*>(empty + kStages);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t G = gridDim.x, b = blockIdx.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) { bar_init(&full[s], 1); bar_init(&empty[s], kCW); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint64_t cb = n_tiles * b / G, ce = n_tiles * (b + 1) / G;
    if (warp == kCW) {
        if (lane == 0) {
            int chunk_left = 0;
            uint64_t chunk_next = 0;
            for (uint64_t it = 0;; ++it) {
                const int s = int(it % kStages);
                if (it >= kStages) bar_wait(&empty[s], uint32_t((it / kStages - 1) & 1));
                long long t;
                if (mode == 0) t = (b + it * G < n_tiles) ? (long long)(b + it * G) : -1;
                else if (mode == 1) t = (cb + it < ce) ? (long long)(cb + it) : -1;
                else if (mode == 2) { const unsigned c = atomicAdd(counter, 1u); t = c < n_tiles ? (long long)c : -1; }
                else {  // mode 3: static round-robin prefix, then dynamic chunks of K tiles
                    const uint64_t ns = (n_static > b) ? (n_static - 1 - b) / G + 1 : 0;
                    if (it < ns) t = (long long)(b + it * G);
                    else {
                        if (chunk_left == 0) {
                            const unsigned c = atomicAdd(counter, 1u);
                            chunk_next = n_static + uint64_t(c) * K;
                            chunk_left = chunk_next < n_tiles ? K : 0;
                        }
                        if (chunk_left > 0 && chunk_next < n_tiles) { t = (long long)chunk_next++; --chunk_left; }
                        else t = -1;
                    }
                }
                tid_of[s] = t;
                if (t < 0) { bar_arrive(&full[s]); break; }
                bar_expect(&full[s], kTile * 16);
                const unsigned char* src = reinterpret_cast<const unsigned char*>(xy + uint64_t(t) * kTile);
                for (int off = 0; off < kTile * 16; off += 16384)
                    bulk(reinterpret_cast<unsigned char*>(ring + s * kTile) + off, src + off,
                         uint32_t(kTile * 16 - off < 16384 ? kTile * 16 - off : 16384), &full[s]);
            }
        }
        return;
    }
    double acc = 0.0;
    for (uint64_t it = 0;; ++it) {
        const int s = int(it % kStages);
        bar_wait(&full[s], uint32_t((it / kStages) & 1));
        if (tid_of[s] < 0) break;
        const double2* p = ring + s * kTile + warp * 32 * kP + lane;  // conflict-free
#pragma unroll
        for (int i = 0; i < kP; ++i) acc += p[32 * i].x * p[32 * i].y;
        __syncwarp();
        if (lane == 0) bar_arrive(&empty[s]);
    }
    if (acc == 1234.5) out[0] = acc;
    if (threadIdx.x == 0) fin[b] = gtime();
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint64_t n = uint64_t(1) << 31;  // 32 GiB of points
    const uint64_t n_tiles = n / kTile;
    double2* xy;
    if (cudaMalloc(&xy, n * 16) != cudaSuccess) return 1;
    cudaMemset(xy, 0, n * 16);
    unsigned* counter;
    double* out;
    uint64_t* fin;
    cudaMalloc(&counter, 4);
    cudaMalloc(&out, 8);
    cudaMalloc(&fin, 8 * sms);
    const int smem = kStages * kTile * 16 + 2 * kStages * 8 + kStages * 8;
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[4] = {"static round-robin", "static contiguous", "dynamic counter", "hybrid"};
    struct V { int mode; double f; int K; };
    const V vs[] = {{0, 0, 0}, {1, 0, 0}, {2, 0, 0}, {3, .1, 8}, {3, .2, 8}, {3, .3, 8}, {3, .2, 4}, {3, .2, 16}, {3, .3, 16}};
    for (int pass = 0; pass < 3; ++pass)
        for (const V& v : vs) {
            const int mode = v.mode;
            const uint64_t n_static = uint64_t(n_tiles * (1.0 - v.f));
            cudaMemset(counter, 0, 4);
            uint64_t t0h;
            cudaEventRecord(e0);
            stream<<<sms, kThreads, smem>>>(xy, n_tiles, mode, counter, out, fin, n_static, v.K);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            std::vector<uint64_t> f(sms);
            cudaMemcpy(f.data(), fin, 8 * sms, cudaMemcpyDeviceToHost);
            std::sort(f.begin(), f.end());
            t0h = f[0];
            if (pass > 0)
                printf("{\"mode\": \"%s f=%.2f K=%d\", \"ms\": %.3f, \"GB_per_s\": %.1f, \"finish_spread_us\": %.1f, \"median_minus_first_us\": %.1f}\n",
                       names[mode], v.f, v.K, ms, n_tiles * double(kTile) * 16 / (ms * 1e6), (f[sms - 1] - t0h) / 1e3,
                       (f[sms / 2] - t0h) / 1e3);
        }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    return 0;
}

// Dev probe: per-fit device time of K back-to-back lsqfit_cuda_fit_device
// launches captured in one CUDA graph and replayed (no host launch path in
// the measurement), and the same K launches issued directly from C++.
//   usage: tools/graph_bench n[,n..] m[,m..] [K]
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "lsqfit_cuda.h"

static std::vector<double> parse(const char* s) {
    std::vector<double> v;
    std::string str(s);
    size_t p = 0;
    while (p < str.size()) {
        size_t q = str.find(',', p);
        if (q == std::string::npos) q = str.size();
        v.push_back(std::atof(str.substr(p, q - p).c_str()));
        p = q + 1;
    }
    return v;
}

#define CK(x)                                                                                 \
    do {                                                                                      \
        cudaError_t e_ = (x);                                                                 \
        if (e_ != cudaSuccess) {                                                              \
            std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            return 1;                                                                         \
        }                                                                                     \
    } while (0)

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    const std::vector<double> ns = parse(argv[1]), ms = parse(argv[2]);
    const int K = argc > 3 ? std::atoi(argv[3]) : 50;
    const uint64_t nmax = uint64_t(*std::max_element(ns.begin(), ns.end()));
    lsqfit_cuda_ctx* ctx = nullptr;
    if (lsqfit_cuda_create(&ctx, 0) != LSQFIT_OK) return 1;
    double* xy = nullptr;
    lsqfit_result* out = nullptr;
    CK(cudaMalloc(&xy, nmax * 16));
    CK(cudaMalloc(&out, sizeof(lsqfit_result)));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    if (lsqfit_cuda_synth_device(ctx, xy, nmax, 0, 1, 3, 0.1, s) != LSQFIT_OK) return 1;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (double mv : ms) {
        const int m = int(mv);
        for (double nv : ns) {
            const uint64_t n = uint64_t(nv);
            for (int w = 0; w < 3; ++w)
                if (lsqfit_cuda_fit_device(ctx, xy, n, m, LSQFIT_SOLVE, out, s) != LSQFIT_OK) return 1;
            CK(cudaStreamSynchronize(s));
            // direct launches
            std::vector<float> direct;
            for (int r = 0; r < 7; ++r) {
                CK(cudaEventRecord(e0, s));
                for (int k = 0; k < K; ++k) lsqfit_cuda_fit_device(ctx, xy, n, m, LSQFIT_SOLVE, out, s);
                CK(cudaEventRecord(e1, s));
                CK(cudaEventSynchronize(e1));
                float ms_;
                CK(cudaEventElapsedTime(&ms_, e0, e1));
                direct.push_back(ms_ * 1e3f / K);
            }
            // graph
            cudaGraph_t g;
            cudaGraphExec_t ge;
            CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            for (int k = 0; k < K; ++k)
                if (lsqfit_cuda_fit_device(ctx, xy, n, m, LSQFIT_SOLVE, out, s) != LSQFIT_OK) return 1;
            CK(cudaStreamEndCapture(s, &g));
            size_t nodes = 0;
            CK(cudaGraphGetNodes(g, nullptr, &nodes));
            CK(cudaGraphInstantiate(&ge, g, 0));
            std::vector<float> graph;
            for (int r = 0; r < 9; ++r) {
                CK(cudaEventRecord(e0, s));
                CK(cudaGraphLaunch(ge, s));
                CK(cudaEventRecord(e1, s));
                CK(cudaEventSynchronize(e1));
                float ms_;
                CK(cudaEventElapsedTime(&ms_, e0, e1));
                if (r >= 2) graph.push_back(ms_ * 1e3f / K);
            }
            lsqfit_result h;
            CK(cudaMemcpy(&h, out, sizeof h, cudaMemcpyDeviceToHost));
            std::sort(direct.begin(), direct.end());
            std::sort(graph.begin(), graph.end());
            const double gu = graph[graph.size() / 2];
            std::printf("{\"n\": %llu, \"m\": %d, \"graph_us_per_fit\": %.3f, \"direct_us_per_fit\": %.3f, "
                        "\"graph_nodes\": %zu, \"pts_per_s\": %.4e, \"GB_per_s\": %.1f, \"status\": %d}\n",
                        (unsigned long long)n, m, gu, direct[direct.size() / 2], nodes, n / (gu * 1e-6),
                        16.0 * n / (gu * 1e3), h.status);
            cudaGraphExecDestroy(ge);
            cudaGraphDestroy(g);
        }
    }
    lsqfit_cuda_destroy(ctx);
    return 0;
}

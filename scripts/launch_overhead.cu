// Host-side cost of one C-ABI call (validation + dispatch + cudaLaunchKernelEx)
// without Python, and the per-launch floor of a serial CUDA graph:
//   1. N back-to-back be_edge_packed_u64 calls on a 256x256 packed image vs N
//      bare launches of an empty kernel (enqueue cost per call);
//   2. graphs of N serial launches: empty kernel, empty kernel with PDL, and
//      be_pack_edge_u8 on the 256^2 uint8 image of config C1 (device time per
//      launch: the fixed cost a latency-bound config pays).
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -I include scripts/launch_overhead.cu \
//        -L paper_1401_5245_b200/lib -lbitedge_cuda -Xlinker -rpath \
//        -Xlinker '$ORIGIN/../paper_1401_5245_b200/lib' -o scripts/launch_overhead
#include <chrono>
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>
#include "bitedge.h"

__global__ void empty_kernel() {}
__global__ void empty_pdl_kernel() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
}

template <typename F>
float graph_us_per_launch(cudaStream_t s, int n, F body) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < n; ++i) body();
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    return ms * 1e3f / n;
}

int main() {
    const int64_t h = 256, w = 256, wp = 4;
    uint64_t *in, *out;
    cudaMalloc(&in, h * wp * 8);
    cudaMalloc(&out, h * wp * 8);
    cudaMemset(in, 0x5A, h * wp * 8);
    uint8_t *pix;
    uint32_t *pout;
    cudaMalloc(&pix, h * w);
    cudaMalloc(&pout, h * (w / 32) * 4);
    cudaMemset(pix, 1, h * w);
    cudaStream_t s;
    cudaStreamCreate(&s);
    const int N = 20000;
    for (int i = 0; i < 1000; ++i) be_edge_packed_u64(in, out, 1, h, w, wp, 1, 0, s);
    cudaStreamSynchronize(s);
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < N; ++i) be_edge_packed_u64(in, out, 1, h, w, wp, 1, 0, s);
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(s);
    auto t2 = std::chrono::steady_clock::now();
    for (int i = 0; i < N; ++i) empty_kernel<<<1, 32, 0, s>>>();
    auto t3 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(s);
    auto t4 = std::chrono::steady_clock::now();
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    printf("be_edge_packed_u64: %.2f us/call enqueue, %.2f us/call incl. drain\n", us(t0, t1) / N, us(t0, t2) / N);
    printf("empty <<<>>> launch: %.2f us/call enqueue, %.2f us/call incl. drain\n", us(t2, t3) / N, us(t2, t4) / N);

    const int G = 2000;
    float e = graph_us_per_launch(s, G, [&] { empty_kernel<<<2, 256, 0, s>>>(); });
    float ep = graph_us_per_launch(s, G, [&] {
        cudaLaunchConfig_t cfg;
        memset(&cfg, 0, sizeof(cfg));
        cfg.gridDim = dim3(2);
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, empty_pdl_kernel);
    });
    float c1 = graph_us_per_launch(s, G, [&] {
        be_pack_edge_u8(pix, pout, 1, h, w, w, w / 32, 1, nullptr, s);
    });
    printf("serial graph, device time per launch: empty %.2f us, empty+PDL %.2f us, "
           "C1 be_pack_edge_u8 %.2f us\n", e, ep, c1);
    printf("last error: %s\n", be_last_error());
    return 0;
}

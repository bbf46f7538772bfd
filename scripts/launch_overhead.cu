// Host-side cost of one C-ABI call (validation + dispatch + cudaLaunchKernelEx)
// without Python: N back-to-back be_edge_packed_u64 calls on a 256x256 image,
// wall clock / N, against N bare launches of an empty kernel.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -I include scripts/launch_overhead.cu \
//        -L paper_1401_5245_b200/lib -lbitedge_cuda -o scripts/launch_overhead
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
#include "bitedge.h"

__global__ void empty_kernel() {}

int main() {
    const int64_t h = 256, w = 256, wp = 4;
    uint64_t *in, *out;
    cudaMalloc(&in, h * wp * 8);
    cudaMalloc(&out, h * wp * 8);
    cudaMemset(in, 0x5A, h * wp * 8);
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
    printf("last error: %s\n", be_last_error());
    return 0;
}

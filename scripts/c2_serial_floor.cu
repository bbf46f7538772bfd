// Serial (one stream, graph-replayed) time per C2 step against two floors with
// the same launch shape (512 CTAs x 256 threads, PDL) over the same rotating
// buffer pool (22 x (16 MiB in + 2 MiB out) > 3x L2):
//   empty   -- griddepcontrol only: launch + grid fixed cost;
//   stream  -- each warp loads its 4 KB with four 256-bit loads and stores 4 words
//              per lane (K2w's traffic and access pattern, no pack / edge math);
//   K2w     -- be_pack_edge_u8 on the C2 batch (the real kernel).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I include scripts/c2_serial_floor.cu \
//        -L paper_1401_5245_b200/lib -lbitedge_cuda -Xlinker -rpath \
//        -Xlinker '$ORIGIN/../paper_1401_5245_b200/lib' -o scripts/c2_serial_floor
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "bitedge.h"

__global__ void empty_pdl() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
}

__global__ void stream_pdl(const uint8_t *in, uint32_t *out) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const uint8_t *src = in + warp * 4096 + 32 * lane;
    uint32_t acc[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        uint32_t v[8];
        asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                       "=r"(v[6]), "=r"(v[7])
                     : "l"(src + 1024 * k));
        acc[k] = v[0] ^ v[1] ^ v[2] ^ v[3] ^ v[4] ^ v[5] ^ v[6] ^ v[7];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) __stcs(out + warp * 128 + 32 * k + lane, acc[k]);
}

static void launch_pdl(void (*k)(), int grid, cudaStream_t s) {
    cudaLaunchConfig_t c = {};
    c.gridDim = dim3(grid); c.blockDim = dim3(256); c.stream = s;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a[0].val.programmaticStreamSerializationAllowed = 1;
    c.attrs = a; c.numAttrs = 1;
    cudaLaunchKernelEx(&c, k);
}
static void launch_stream(const uint8_t *in, uint32_t *out, int grid, cudaStream_t s) {
    cudaLaunchConfig_t c = {};
    c.gridDim = dim3(grid); c.blockDim = dim3(256); c.stream = s;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a[0].val.programmaticStreamSerializationAllowed = 1;
    c.attrs = a; c.numAttrs = 1;
    cudaLaunchKernelEx(&c, stream_pdl, in, out);
}

template <typename F>
static float serial_us(cudaStream_t s, int n, F body) {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < n; ++i) body(i);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e3f / n;
}

int main() {
    const int nimg = 4096, pool = 22, n = 2200;
    const size_t in_b = (size_t)nimg * 4096, out_b = (size_t)nimg * 64 * 2 * 4;
    std::vector<uint8_t *> ins(pool);
    std::vector<uint32_t *> outs(pool);
    std::vector<uint8_t> h(in_b);
    for (size_t i = 0; i < in_b; ++i) h[i] = (uint8_t)((i * 2654435761u) >> 31 & 1);
    for (int p = 0; p < pool; ++p) {
        cudaMalloc(&ins[p], in_b);
        cudaMalloc(&outs[p], out_b);
        cudaMemcpy(ins[p], h.data(), in_b, cudaMemcpyHostToDevice);
    }
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    const int grid = nimg * 32 / 256;
    float e = serial_us(s, n, [&](int) { launch_pdl(empty_pdl, grid, s); });
    float st = serial_us(s, n, [&](int i) { launch_stream(ins[i % pool], outs[i % pool], grid, s); });
    float k = serial_us(s, n, [&](int i) {
        be_pack_edge_u8(ins[i % pool], outs[i % pool], nimg, 64, 64, 64, 2, 1, nullptr, s);
    });
    const double alg = (double)nimg * 4096 * 1.125;
    printf("serial us/step: empty %.3f  stream (K2w traffic) %.3f  K2w %.3f\n", e, st, k);
    printf("alg GB/s: stream %.0f  K2w %.0f\n", alg / st / 1e3, alg / k / 1e3);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

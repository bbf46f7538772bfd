// capi_internal.cuh -- host-side helpers shared by the C-ABI translation units
// (capi_edges.cu, capi_words.cu, capi_p4.cu, capi_host.cu): argument
// validation with the reference's error semantics (bitimage.py:87-97, 188-193),
// launch helpers (programmatic dependent launch), raster geometry.
#pragma once

#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/bitedge.h"
#include "edge_tile.cuh"

namespace bitedge {
namespace capi {

// the only state: this thread's error text and launch counter (capi_host.cu)
extern thread_local char g_err[512];
extern thread_local int64_t g_launches;

// Dispatch knobs: BITEDGE_<name> environment variables
// for A/B measurements and the variant tests, read once per process on first
// use (be_reload_knobs re-reads them) -- a getenv per knob per call cost ~1.4 us
// of host time per launch with a typical environment.
enum Knob : int {
    KN_KERNEL,
    KN_K1_GENERIC,
    KN_UNAL_BYTES,
    KN_NO_UNAL,
    KN_NO_TMA,
    KN_CW4,
    KN_UNAL_CHUNKS,
    KN_CW8,
    KN_NO_WARPIMG,
    KN_WARPIMG_G4,
    KN_PDL_LATE,
    KN_TMA1,
    KN_FORCE_TMA,
    KN_U64_TMA,
    KN_TMA2_RSL8,
    KN_TMA2_RSL32,
    KN_NO_ROLL,
    KN_RS,
    KN_PRS,
    KN_UNAL_RS4,
    KN_P4_UNFUSED,
    KN_P4_BYTES,
    KN_PDL,
    KN_NO_FLAT,
    KN_K2P,
    KN_SYNC_BLOCK,
    KN_NO_H16,
    KN_RING,
    KN_NO_TMA_UNAL,
    KN_P4_NO_FLAT,
    KN_P4_FLAT16,
    KN_P4_FLAT_MAX,
    KN_P4_FLAT32,
    KN_TMA2_MIN,
    KN_TMA2_RSL,
    KN_TMA2_MINW,
    KN_ROLL_MIN,
    KN_COUNT
};
extern const char *const kKnobNames[KN_COUNT];
// the knob's value, or nullptr when unset
const char *knob(Knob k);

inline int fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

// "this kernel does not apply, try the next one" from the kernel-selection
// helpers: distinct from BE_OK, the negative BE_E* codes and every (positive)
// cudaError_t, so a CUDA error is never mistaken for a fallback.
constexpr int kNoKernel = -1000;

inline int cuda_check(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
        return (int)e;
    }
    ++g_launches;
    return BE_OK;
}

inline cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }

struct Geometry {
    int64_t n, h, w;
    int word_bits;
    int wp;          // storage words per row in uint32 units
    int pl;
    uint32_t lastbit, padmask, fillword;
    int swap;
};

inline int make_geometry(Geometry &G, int word_bits, int64_t n, int64_t h, int64_t w, int fill_bit) {
    if (word_bits != 32 && word_bits != 64)
        return fail(BE_EINVAL, "word_bits must be 32 or 64, got %d", word_bits);
    if (n < 0) return fail(BE_EINVAL, "batch size must be >= 0, got %lld", (long long)n);
    if (w < 1 || h < 1)
        return fail(BE_EINVAL, "image dimensions must be at least 1x1, got %lldx%lld",
                    (long long)w, (long long)h);
    if (fill_bit != 0 && fill_bit != 1)
        return fail(BE_EINVAL, "fill_bit must be 0 or 1, got %d", fill_bit);
    if (w > (int64_t)1 << 36 || h > ((int64_t)1 << 40) || (n > 0 && h > ((int64_t)1 << 40) / n))
        return fail(BE_EINVAL, "raster too large");
    G.n = n; G.h = h; G.w = w; G.word_bits = word_bits;
    const int64_t wp = word_bits == 64 ? 2 * ((w + 63) / 64) : (w + 31) / 32;
    if (wp > (1 << 30)) return fail(BE_EINVAL, "row too wide");
    G.wp = (int)wp;
    G.pl = (int)((w - 1) / 32);
    G.lastbit = 1u << (31 - (int)((w - 1) % 32));
    G.padmask = G.lastbit - 1u;
    G.fillword = fill_bit ? 0xFFFFFFFFu : 0u;
    G.swap = word_bits == 64 ? 1 : 0;
    return BE_OK;
}

inline int check_stride(const Geometry &G, int64_t stride_words, const char *what) {
    const int64_t need = G.word_bits == 64 ? (G.w + 63) / 64 : (G.w + 31) / 32;
    if (stride_words < need)
        return fail(BE_EINVAL, "%s row stride %lld words < %lld words per row", what,
                    (long long)stride_words, (long long)need);
    return BE_OK;
}

inline int check_ptr(const void *p, int word_bits, const char *what) {
    if (p == nullptr) return fail(BE_EINVAL, "%s is NULL", what);
    if (((uintptr_t)p) % (word_bits / 8) != 0)
        return fail(BE_EALIGN, "%s is not %d-byte aligned", what, word_bits / 8);
    return BE_OK;
}

// Launch with programmatic dependent launch enabled (BITEDGE_PDL=0 disables): the
// kernel's CTAs may be scheduled while the previous kernel on the stream drains;
// they block in griddepcontrol.wait until its results are visible.
inline bool pdl_enabled() {
    const char *e = knob(KN_PDL);
    return !(e && e[0] == '0');
}

template <typename... KArgs, typename... Args>
void launch_kb(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
               Args... args) {
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, args...);
}

template <typename... KArgs, typename... Args>
void launch_k(void (*kern)(KArgs...), unsigned grid, size_t smem, cudaStream_t st, Args... args) {
    launch_kb(kern, grid, (unsigned)bitedge::kThreads, smem, st, args...);
}

inline int ilog2(int v) { int l = 0; while ((1 << (l + 1)) <= v) ++l; return l; }
inline int next_pow2(int64_t v) { int p = 1; while (p < v && p < (1 << 30)) p <<= 1; return p; }

inline int sm_count() {
    thread_local int dev_cached = -1, sms_cached = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != dev_cached) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        sms_cached = v > 0 ? v : 148;
        dev_cached = dev;
    }
    return sms_cached;
}

// ---------------------------------------------------------------- word-kernel geometry

struct WordGeom {
    int64_t nrows, stride;  // uint32 units
    int wp, pl, swap;
    uint32_t lastbit, padmask, fillword;
    int64_t h;
};

inline WordGeom word_geom(const Geometry &G, int64_t stride_words) {
    WordGeom g;
    g.nrows = G.n * G.h;
    g.stride = G.word_bits == 64 ? 2 * stride_words : stride_words;
    g.wp = G.wp; g.pl = G.pl; g.swap = G.swap;
    g.lastbit = G.lastbit; g.padmask = G.padmask; g.fillword = G.fillword;
    g.h = G.h;
    return g;
}

__device__ __forceinline__ uint32_t force_pad(const WordGeom &g, int pw, uint32_t v) {
    if (pw == g.pl) return v | g.padmask;
    if (pw > g.pl) return 0xFFFFFFFFu;
    return v;
}

inline unsigned grid_for(int64_t total) {
    int64_t blocks = (total + 255) / 256;
    const int64_t cap = 148 * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return (unsigned)blocks;
}

inline int prep_words(Geometry &G, int word_bits, int64_t n, int64_t h, int64_t w, int64_t stride,
               int fill_bit, const void *a, const char *aname, const void *out) {
    int rc = make_geometry(G, word_bits, n, h, w, fill_bit);
    if (rc) return rc;
    if ((rc = check_stride(G, stride, "row"))) return rc;
    if (n == 0) return BE_OK;
    if ((rc = check_ptr(a, word_bits, aname))) return rc;
    if ((rc = check_ptr(out, word_bits, "output"))) return rc;
    return BE_OK;
}

// The fused-edge driver shared by every edge entry point (capi_edges.cu).
int edges_impl(const void *in, int input_kind, int64_t in_stride, const void *above,
               const void *below, uint32_t *o_edges, uint32_t *o_eset, uint32_t *const o_side[4],
               uint32_t *o_packed, int word_bits, int64_t out_stride_words, int64_t n, int64_t h,
               int64_t w, int fill_bit, int64_t row_lo, int64_t row_hi, void *stream, int thr = 1);

}  // namespace capi
}  // namespace bitedge

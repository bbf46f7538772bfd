// bitedge_capi.cu -- C ABI (include/bitedge.h) over the sm_100a kernels.
//
// Host side: argument validation with the reference's error semantics
// (bitimage.py:87-97, 188-193), tile-shape selection for the fused edge
// kernel (edge_tile.cuh), and the small word-parallel kernels behind the
// BitImage primitives (bitimage.py:149-249).  No allocation, no global state
// beyond thread-local error text and launch counter.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/bitedge.h"
#include "edge_tile.cuh"
#include "edge_stream.cuh"
#include "edge_reg.cuh"

using namespace bitedge;

namespace {

thread_local char g_err[512];
thread_local int64_t g_launches = 0;

int fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int cuda_check(const char *what) {
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

int make_geometry(Geometry &G, int word_bits, int64_t n, int64_t h, int64_t w, int fill_bit) {
    if (word_bits != 32 && word_bits != 64)
        return fail(BE_EINVAL, "word_bits must be 32 or 64, got %d", word_bits);
    if (n < 0) return fail(BE_EINVAL, "batch size must be >= 0, got %lld", (long long)n);
    if (w < 1 || h < 1)
        return fail(BE_EINVAL, "image dimensions must be at least 1x1, got %lldx%lld",
                    (long long)w, (long long)h);
    if (fill_bit != 0 && fill_bit != 1)
        return fail(BE_EINVAL, "fill_bit must be 0 or 1, got %d", fill_bit);
    if (w > (int64_t)1 << 36 || n * h > ((int64_t)1 << 40))
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

int check_stride(const Geometry &G, int64_t stride_words, const char *what) {
    const int64_t need = G.word_bits == 64 ? (G.w + 63) / 64 : (G.w + 31) / 32;
    if (stride_words < need)
        return fail(BE_EINVAL, "%s row stride %lld words < %lld words per row", what,
                    (long long)stride_words, (long long)need);
    return BE_OK;
}

int check_ptr(const void *p, int word_bits, const char *what) {
    if (p == nullptr) return fail(BE_EINVAL, "%s is NULL", what);
    if (((uintptr_t)p) % (word_bits / 8) != 0)
        return fail(BE_EALIGN, "%s is not %d-byte aligned", what, word_bits / 8);
    return BE_OK;
}

// Launch with programmatic dependent launch enabled (BITEDGE_PDL=0 disables): the
// kernel's CTAs may be scheduled while the previous kernel on the stream drains;
// they block in griddepcontrol.wait until its results are visible.
bool pdl_enabled() {
    const char *e = getenv("BITEDGE_PDL");
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

template <int KIND>
int launch_tile(TileParams &tp, int64_t rows, cudaStream_t st) {
    const int TQ = 1 << tp.log_tq, R = 1 << tp.log_r;
    const size_t smem = (size_t)(R + 2) * (TQ + 8) * 4 + R;
    const int64_t tiles_y = (rows + R - 1) / R;
    const int64_t grid = tiles_y * tp.tiles_x;
    if (grid <= 0) return BE_OK;
    if (grid > 0x7FFFFFFFLL) return fail(BE_EINVAL, "raster too large for one launch");
    const bool others = tp.o_side[0] || tp.o_side[1] || tp.o_side[2] || tp.o_side[3] || tp.o_packed;
    if (!others && tp.o_edges && !tp.o_eset)
        edge_tile_kernel<KIND, kOutEdges><<<(unsigned)grid, kThreads, smem, st>>>(tp);
    else if (!others && tp.o_eset && !tp.o_edges)
        edge_tile_kernel<KIND, kOutEset><<<(unsigned)grid, kThreads, smem, st>>>(tp);
    else
        edge_tile_kernel<KIND, kOutAny><<<(unsigned)grid, kThreads, smem, st>>>(tp);
    return cuda_check("edge_tile_kernel");
}

// ---------------------------------------------------------------- streaming kernel

int sm_count() {
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

// Kernel selection knob for A/B measurements: BITEDGE_KERNEL=tile forces the
// one-shot tile kernel, =stream forbids nothing (default: stream when eligible).
bool stream_allowed() {
    const char *e = getenv("BITEDGE_KERNEL");
    return !(e && strcmp(e, "tile") == 0);
}

template <int KIND, int OUT>
int launch_stream_out(StreamParams &sp, size_t smem, cudaStream_t st) {
    if (smem > 48 * 1024) {   // per launch: the attribute is per device
        cudaError_t e = cudaFuncSetAttribute(edge_stream_kernel<KIND, OUT>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return fail((int)e, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, edge_stream_kernel<KIND, OUT>, kThreads,
                                                  smem);
    if (per_sm < 1) per_sm = 1;
    int64_t grid = (int64_t)sm_count() * per_sm;
    if (grid > sp.ntiles) grid = sp.ntiles;
    edge_stream_kernel<KIND, OUT><<<(unsigned)grid, kThreads, smem, st>>>(sp);
    return cuda_check("edge_stream_kernel");
}

template <int KIND>
int launch_stream_kind(StreamParams &sp, size_t smem, cudaStream_t st) {
    if (sp.o_edges && sp.o_eset) return launch_stream_out<KIND, kOutAny>(sp, smem, st);
    if (sp.o_eset) return launch_stream_out<KIND, kOutEset>(sp, smem, st);
    return launch_stream_out<KIND, kOutEdges>(sp, smem, st);
}

// ---------------------------------------------------------------- register-direct kernel

// Launch helpers: dispatch the runtime choices onto template parameters.
template <int OUT, bool HALO>
int launch_reg_packed(RegParams &rp, int swap, int cw, int rs, unsigned grid, cudaStream_t st) {
    if constexpr (OUT == kOutAll) {   // up to 7 outputs: 4-word items keep it in registers
        if (swap) launch_k(edge_reg_packed_kernel<1, 4, 4, OUT, HALO>, grid, 0, st, rp);
        else if (rs == 2) launch_k(edge_reg_packed_kernel<0, 2, 4, OUT, HALO>, grid, 0, st, rp);
        else launch_k(edge_reg_packed_kernel<0, 4, 4, OUT, HALO>, grid, 0, st, rp);
        (void)cw;
    } else {
        if (!swap && rs == 2) {
            // (128-thread CTAs for C3's single wave: +2 % overlapped, -1 % serial; not taken)
            if (cw == 8) launch_k(edge_reg_packed_kernel<0, 2, 8, OUT, HALO>, grid, 0, st, rp);
            else launch_k(edge_reg_packed_kernel<0, 2, 4, OUT, HALO>, grid, 0, st, rp);
        } else if (!swap && rs == 8) {
            if (cw == 8) launch_k(edge_reg_packed_kernel<0, 8, 8, OUT, HALO>, grid, 0, st, rp);
            else launch_k(edge_reg_packed_kernel<0, 8, 4, OUT, HALO>, grid, 0, st, rp);
        } else if (swap) {
            if (cw == 8) launch_k(edge_reg_packed_kernel<1, 4, 8, OUT, HALO>, grid, 0, st, rp);
            else launch_k(edge_reg_packed_kernel<1, 4, 4, OUT, HALO>, grid, 0, st, rp);
        } else {
            if (cw == 8) launch_k(edge_reg_packed_kernel<0, 4, 8, OUT, HALO>, grid, 0, st, rp);
            else launch_k(edge_reg_packed_kernel<0, 4, 4, OUT, HALO>, grid, 0, st, rp);
        }
    }
    return cuda_check("edge_reg_packed_kernel");
}

template <int OUT, bool HALO>
int launch_reg_u8(RegParams &rp, int rs, unsigned grid, cudaStream_t st) {
    if (rp.v8) {
        if (rs == 8) launch_k(edge_reg_u8_kernel<8, OUT, HALO, true>, grid, 0, st, rp);
        else launch_k(edge_reg_u8_kernel<4, OUT, HALO, true>, grid, 0, st, rp);
    } else {
        if (rs == 8) launch_k(edge_reg_u8_kernel<8, OUT, HALO, false>, grid, 0, st, rp);
        else launch_k(edge_reg_u8_kernel<4, OUT, HALO, false>, grid, 0, st, rp);
    }
    return cuda_check("edge_reg_u8_kernel");
}

inline bool multi_out(const RegParams &rp) {
    return rp.o_side[0] || rp.o_side[1] || rp.o_side[2] || rp.o_side[3] || rp.o_packed;
}

template <bool HALO>
int launch_reg_halo(RegParams &rp, int input_kind, int swap, int cw, int rs, unsigned grid,
                    cudaStream_t st) {
    if (multi_out(rp)) {          // packed input only (uint8 multi-output goes to K2t2 or tile)
        if (input_kind == 1) return 1;
        return launch_reg_packed<kOutAll, HALO>(rp, swap, cw, rs, grid, st);
    }
    if (input_kind == 1) {
        if (rp.o_edges && rp.o_eset) return launch_reg_u8<kOutAny, HALO>(rp, rs, grid, st);
        if (rp.o_eset) return launch_reg_u8<kOutEset, HALO>(rp, rs, grid, st);
        return launch_reg_u8<kOutEdges, HALO>(rp, rs, grid, st);
    }
    if (rp.o_edges && rp.o_eset) return launch_reg_packed<kOutAny, HALO>(rp, swap, cw, rs, grid, st);
    if (rp.o_eset) return launch_reg_packed<kOutEset, HALO>(rp, swap, cw, rs, grid, st);
    return launch_reg_packed<kOutEdges, HALO>(rp, swap, cw, rs, grid, st);
}

// Returns 1 when the register-direct kernel does not apply (caller falls back).
inline int64_t rows_total(int64_t lo, int64_t hi) { return hi - lo; }

// K2t2 launch for strip height RSL (4-slot rings, 8 warps per CTA).
template <int RSL>
int launch_tma2(RegParams &rp, bool multi, bool halo, int64_t nseg, cudaStream_t st) {
    constexpr int kD = 4;
    const int64_t nstrips = (rows_total(rp.row_lo, rp.row_hi) + RSL - 1) / RSL;
    const int64_t nwarps = nstrips * nseg;
    const unsigned grid = (unsigned)((nwarps + 7) / 8);
    const size_t smem = (size_t)8 * kD * 2080 + (size_t)8 * kD * 8;
    rp.nstrips = nstrips;
#define BE_TMA2(OUTK, H)                                                                        \
    do {                                                                                        \
        auto kern = edge_tma2_u8_kernel<RSL, kD, OUTK, H>;                                      \
        /* per launch: the attribute is per device, and these launches are long */             \
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
        launch_k(kern, grid, smem, st, rp, nseg, nwarps);                                       \
    } while (0)
    if (multi) {
        if (halo) BE_TMA2(kOutAll, true); else BE_TMA2(kOutAll, false);
    } else if (rp.o_edges && rp.o_eset) {
        if (halo) BE_TMA2(kOutAny, true); else BE_TMA2(kOutAny, false);
    } else if (rp.o_eset) {
        if (halo) BE_TMA2(kOutEset, true); else BE_TMA2(kOutEset, false);
    } else {
        if (halo) BE_TMA2(kOutEdges, true); else BE_TMA2(kOutEdges, false);
    }
#undef BE_TMA2
    return cuda_check("edge_tma2_u8_kernel");
}

int try_reg(const void *in, int input_kind, int64_t in_row_bytes, const void *above,
            const void *below, uint32_t *o_edges, uint32_t *o_eset, uint32_t *const o_side[4],
            uint32_t *o_packed, int64_t out_stride_u32, const Geometry &G, int64_t nrows,
            int64_t row_lo, int64_t row_hi, cudaStream_t st, int thr) {
    const char *e = getenv("BITEDGE_KERNEL");
    if (e && (strcmp(e, "tile") == 0 || strcmp(e, "stream") == 0)) return 1;
    auto al16 = [](const void *p) { return p == nullptr || ((uintptr_t)p % 16) == 0; };
    if (!al16(in) || !al16(above) || !al16(below) || in_row_bytes % 16 != 0) return 1;
    if (G.h >= ((int64_t)1 << 31)) return 1;
    RegParams rp;
    memset(&rp, 0, sizeof(rp));
    rp.in = (const char *)in; rp.above = (const char *)above; rp.below = (const char *)below;
    rp.in_row_bytes = in_row_bytes;
    rp.o_edges = o_edges; rp.o_eset = o_eset; rp.out_stride = out_stride_u32;
    for (int k = 0; k < 4; ++k) rp.o_side[k] = o_side[k];
    rp.o_packed = o_packed;
    const bool multi = multi_out(rp);
    // uint8 -> uint64 words (the drop-in BitImage layout): only K2t2 stores
    // swapped halves; it takes every such shape >= 1024 px wide, the tile kernel
    // the rest
    const bool u64_out = input_kind == 1 && G.swap;
    if (u64_out && (G.w < 1024 || getenv("BITEDGE_NO_TMA"))) return 1;
    rp.oswap = u64_out ? 1 : 0;
    rp.nrows = nrows; rp.row_lo = row_lo; rp.row_hi = row_hi;
    rp.h = (uint32_t)G.h; rp.w = G.w; rp.wp = G.wp; rp.pl = G.pl;
    rp.lastbit = G.lastbit; rp.padmask = G.padmask; rp.fillword = G.fillword;
    auto al = [](const void *p, int a) { return p == nullptr || ((uintptr_t)p % a) == 0; };
    const bool in32 = al(in, 32) && in_row_bytes % 32 == 0 && al(above, 32) && al(below, 32);
    // packed items are 8 words (256-bit loads) when rows are 32-byte aligned, else 4
    // Packed items are 8 words (256-bit loads) when rows are 32-byte aligned, else 4.
    // Small rasters (< 4 waves of 4-row strips) use 2-row strips instead, which
    // doubles the threads in flight (C3: 5.1 us serial / 88 % overlapped vs
    // 5.3 / 79 % for 4-word x 4-row items; scripts/c3sweep.sh).
    const int64_t strips4 = (row_hi - row_lo + 3) / 4;
    const bool big = strips4 * ((G.wp + 7) / 8) >= (int64_t)sm_count() * 4096;
    int cw = (input_kind == 0 && in32 && !multi && !getenv("BITEDGE_CW4")) ? 8 : 4;
    const int packed_rs = (input_kind == 0 && !G.swap && !big) ? 2 : 4;
    if (input_kind == 0 && in32 && !multi && getenv("BITEDGE_CW8")) cw = 8;
    rp.items = input_kind == 1 ? G.wp : (G.wp + cw - 1) / cw;
    rp.v8 = input_kind == 1 && in32 && G.w % 32 == 0;
    rp.thr = thr;
    const int ocw = input_kind == 1 ? 1 : cw;
    rp.vst = (out_stride_u32 % ocw == 0) && al(o_edges, 4 * ocw) && al(o_eset, 4 * ocw);
    for (int k = 0; k < 4; ++k) rp.vst = rp.vst && al(o_side[k], 4 * ocw);
    rp.vst = rp.vst && al(o_packed, 4 * ocw);
    if (input_kind == 1 && !multi && !u64_out && !above && !below && row_lo == 0 && row_hi == nrows &&
        in_row_bytes == G.w && ((uintptr_t)in % 32) == 0 && G.w % 32 == 0 && G.wp <= 32 &&
        (G.wp & (G.wp - 1)) == 0 && out_stride_u32 == G.wp && !getenv("BITEDGE_NO_WARPIMG")) {
        const int lwpr = ilog2(G.wp), rpi = 32 >> lwpr;
        if (G.h % rpi == 0 && G.h / rpi <= 8) {
            const int groups = (int)(G.h / rpi);
            const int64_t nimg = G.n;
            const int64_t grid = (nimg * 32 + kThreads - 1) / kThreads;
            if (grid <= 0x7FFFFFFFLL) {
#define BE_WARPIMG_G(L, GM)                                                                    \
    do {                                                                                       \
        if (o_edges && o_eset)                                                                 \
            launch_kb(edge_warp_img_kernel<L, kOutAny, GM>, wgrid, wblock, wsmem, st, rp,      \
                      groups, nimg);                                                           \
        else if (o_eset)                                                                       \
            launch_kb(edge_warp_img_kernel<L, kOutEset, GM>, wgrid, wblock, wsmem, st, rp,     \
                      groups, nimg);                                                           \
        else                                                                                   \
            launch_kb(edge_warp_img_kernel<L, kOutEdges, GM>, wgrid, wblock, wsmem, st, rp,    \
                      groups, nimg);                                                           \
    } while (0)
#define BE_WARPIMG(L)                                                                          \
    case L:                                                                                    \
        if (groups <= 4 && !g8) BE_WARPIMG_G(L, 4); else BE_WARPIMG_G(L, 8);                   \
        return cuda_check("edge_warp_img_kernel");
                // GMAX = 4 (48 regs, one wave of 4096 C2 images) is 1.5 % faster with
                // overlapped batches but 9 % slower serially under PDL than GMAX = 8
                // (77 regs, 1.15 waves): opt-in knob.
                const bool g8 = getenv("BITEDGE_WARPIMG_G4") == nullptr;
                // (Capping residency at one wave with 128-thread CTAs + 32 KB of
                // dummy smem -- 28 warps/SM, 4144 slots for 4096 images -- was
                // 20 % slower overlapped and serially: not taken.)
                const unsigned wblock = (unsigned)kThreads;
                const unsigned wgrid = (unsigned)grid;
                const size_t wsmem = 0;
                rp.pdl_late = getenv("BITEDGE_PDL_LATE") != nullptr;
                switch (lwpr) {
                    BE_WARPIMG(0)
                    BE_WARPIMG(1)
                    BE_WARPIMG(2)
                    BE_WARPIMG(3)
                    BE_WARPIMG(4)
                    BE_WARPIMG(5)
                    default: break;
                }
#undef BE_WARPIMG
#undef BE_WARPIMG_G
            }
        }
    }
    const int64_t rows = row_hi - row_lo;
    // uint8 rows >= 1024 px with enough work: per-warp TMA ring (K2t)
    if (input_kind == 1 && (G.w >= 2048 || u64_out) && !getenv("BITEDGE_NO_TMA") &&
        (!getenv("BITEDGE_TMA1") || u64_out)) {
        const int64_t nseg = (G.w + 2047) / 2048;
        const int64_t nwarps32 = (rows_total(row_lo, row_hi) + 31) / 32 * nseg;
        const bool force = getenv("BITEDGE_FORCE_TMA") != nullptr || u64_out;
        if ((force || nwarps32 >= (int64_t)sm_count() * 24) && (nwarps32 * 4 + 7) / 8 <= 0x7FFFFFFFLL) {
            // Strip height: 8 rows for the 0/1 fast pack (4x the warps of 32-row
            // strips, so the last wave's tail is a quarter as long: C5 737 ->
            // 676 us); 32 rows when the pack is ALU-bound (threshold compare),
            // where the 25 % extra staged halo rows of 8-row strips cost more
            // than the tail (F2 on C5: 800 vs 921 us).  Sweep in DESIGN.md.
            const bool short_strips = (thr == 1 || getenv("BITEDGE_TMA2_RSL8")) &&
                                      !getenv("BITEDGE_TMA2_RSL32");
            const bool halo = above || below;
            return short_strips ? launch_tma2<8>(rp, multi, halo, nseg, st)
                                : launch_tma2<32>(rp, multi, halo, nseg, st);
        }
    }
    if ((multi || u64_out) && input_kind == 1) return 1;   // other uint8 shapes: tile kernel
    if (input_kind == 1 && G.w >= 1024 && !getenv("BITEDGE_NO_TMA")) {
        constexpr int kRSLT = 32, kD = 6;
        const int64_t nseg = (G.w + 1023) / 1024;
        const int64_t nstrips = (rows_total(row_lo, row_hi) + kRSLT - 1) / kRSLT;
        const int64_t nwarps = nstrips * nseg;
        const bool force = getenv("BITEDGE_FORCE_TMA") != nullptr;   // tests: any size
        if ((force || nwarps >= (int64_t)sm_count() * 32) && (nwarps + 7) / 8 <= 0x7FFFFFFFLL) {
            const unsigned grid = (unsigned)((nwarps + 7) / 8);
            const size_t smem = (size_t)8 * kD * 1056 + (size_t)8 * kD * 8;
            const bool halo = above || below;
            rp.nstrips = nstrips;
#define BE_TMA(OUTK, H)                                                                         \
    do {                                                                                        \
        auto kern = edge_tma_u8_kernel<kRSLT, kD, OUTK, H>;                                     \
        /* per launch: the attribute is per device, and these launches are long */             \
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
        launch_k(kern, grid, smem, st, rp, nseg, nwarps);                                       \
    } while (0)
            if (rp.o_edges && rp.o_eset) {
                if (halo) BE_TMA(kOutAny, true); else BE_TMA(kOutAny, false);
            } else if (rp.o_eset) {
                if (halo) BE_TMA(kOutEset, true); else BE_TMA(kOutEset, false);
            } else {
                if (halo) BE_TMA(kOutEdges, true); else BE_TMA(kOutEdges, false);
            }
#undef BE_TMA
            return cuda_check("edge_tma_u8_kernel");
        }
    }
    // uint8 with 32-byte rows and enough strips to fill the GPU: long rolling strips
    constexpr int kRSL = 32, kQ = 4;
    if (input_kind == 1 && rp.v8 && !getenv("BITEDGE_NO_ROLL") &&
        (rows + kRSL - 1) / kRSL * rp.items >= (int64_t)sm_count() * 2048) {
        rp.nstrips = (rows + kRSL - 1) / kRSL;
        const int64_t g = (rp.nstrips * rp.items + kThreads - 1) / kThreads;
        if (g <= 0x7FFFFFFFLL) {
            const unsigned grid = (unsigned)g;
            const bool halo = above || below;
            if (rp.o_edges && rp.o_eset) {
                if (halo) launch_k(edge_roll_u8_kernel<kRSL, kQ, kOutAny, true>, grid, 0, st, rp);
                else launch_k(edge_roll_u8_kernel<kRSL, kQ, kOutAny, false>, grid, 0, st, rp);
            } else if (rp.o_eset) {
                if (halo) launch_k(edge_roll_u8_kernel<kRSL, kQ, kOutEset, true>, grid, 0, st, rp);
                else launch_k(edge_roll_u8_kernel<kRSL, kQ, kOutEset, false>, grid, 0, st, rp);
            } else {
                if (halo) launch_k(edge_roll_u8_kernel<kRSL, kQ, kOutEdges, true>, grid, 0, st, rp);
                else launch_k(edge_roll_u8_kernel<kRSL, kQ, kOutEdges, false>, grid, 0, st, rp);
            }
            return cuda_check("edge_roll_u8_kernel");
        }
    }
    // strip height: 4 rows (the one-shot kernels keep every row of the strip in flight)
    int rs = input_kind == 0 ? packed_rs : 4;
    if (input_kind == 1) {
        const char *rse = getenv("BITEDGE_RS");
        if (rse) rs = atoi(rse) == 8 ? 8 : 4;
    } else if (!G.swap) {
        const char *rse = getenv("BITEDGE_PRS");      // packed strip height experiments: 2/4/8
        if (rse) rs = atoi(rse) == 2 ? 2 : (atoi(rse) == 8 ? 8 : 4);
    }
    if (multi && rs == 8) rs = 4;                    // kOutAll has 2- and 4-row strips
    rp.nstrips = (rows + rs - 1) / rs;
    const int64_t threads = rp.nstrips * rp.items;
    const int64_t grid = (threads + kThreads - 1) / kThreads;
    if (grid > 0x7FFFFFFFLL) return 1;
    if (above || below)
        return launch_reg_halo<true>(rp, input_kind, G.swap, cw, rs, (unsigned)grid, st);
    return launch_reg_halo<false>(rp, input_kind, G.swap, cw, rs, (unsigned)grid, st);
}

// Returns 1 when the streaming kernel does not apply (caller falls back).
int try_stream(const void *in, int input_kind, int64_t in_row_bytes, const void *above,
               const void *below, uint32_t *o_edges, uint32_t *o_eset, int word_bits,
               int64_t out_stride_u32, const Geometry &G, int64_t nrows, int64_t row_lo,
               int64_t row_hi, cudaStream_t st, int thr) {
    if (!stream_allowed()) return 1;
    auto al16 = [](const void *p) { return p == nullptr || ((uintptr_t)p % 16) == 0; };
    if (!al16(in) || !al16(above) || !al16(below) || in_row_bytes % 16 != 0) return 1;
    if (nrows >= ((int64_t)1 << 31)) return 1;                     // 32-bit row arithmetic
    StreamParams sp;
    memset(&sp, 0, sizeof(sp));
    sp.in = (const char *)in; sp.above = (const char *)above; sp.below = (const char *)below;
    sp.in_row_bytes = in_row_bytes;
    sp.o_edges = o_edges; sp.o_eset = o_eset; sp.out_stride = out_stride_u32;
    sp.nrows = nrows; sp.h = G.h; sp.w = G.w; sp.row_lo = row_lo; sp.row_hi = row_hi;
    sp.wp = G.wp; sp.pl = G.pl; sp.lastbit = G.lastbit; sp.padmask = G.padmask;
    sp.fillword = G.fillword;
    sp.thr = thr;
    sp.vst = (out_stride_u32 % 4 == 0) && al16(o_edges) && al16(o_eset);
    int TQ, stage_target = 24 * 1024;
    if (input_kind == 0) {
        const int64_t wpr = (G.wp + 3) / 4 * 4;                 // words readable per row
        TQ = wpr >= 256 ? 256 : next_pow2(wpr);
        sp.tiles_x = (G.wp + TQ - 1) / TQ;
        sp.contiguous = sp.tiles_x == 1 && in_row_bytes <= 8 * wpr;
        sp.raw_pitch = sp.contiguous ? (int)in_row_bytes : 4 * TQ + 32;
        sp.col0 = sp.contiguous ? 0 : 16;
        sp.row_bytes_alloc = sp.contiguous ? in_row_bytes : 4 * wpr;
    } else {
        TQ = G.wp >= 64 ? 64 : next_pow2(G.wp);
        sp.tiles_x = (G.wp + TQ - 1) / TQ;
        const int64_t wr = (G.w + 15) / 16 * 16;
        sp.contiguous = sp.tiles_x == 1 && in_row_bytes <= 2 * wr;
        sp.raw_pitch = sp.contiguous ? (int)in_row_bytes : 32 * TQ + 32;
        sp.col0 = sp.contiguous ? 0 : 16;
        sp.row_bytes_alloc = sp.contiguous ? in_row_bytes : wr;
        const int room = (sp.raw_pitch - sp.col0) / 16;
        sp.pieces = room < 2 * TQ ? room : 2 * TQ;
    }
    if (sp.raw_pitch > stage_target / 3) return 1;                 // rows too wide to stage
    sp.log_tq = ilog2(TQ);
    int R = stage_target / sp.raw_pitch - 2;
    const int64_t rows = row_hi - row_lo;
    if (R > rows) R = (int)rows;
    if (R < 1) R = 1;
    sp.R = R;
    sp.ntiles = ((rows + R - 1) / R) * sp.tiles_x;
    sp.stage_bytes = ((R + 2) * sp.raw_pitch + 127) / 128 * 128;
    sp.stages = 4;
    size_t smem = (size_t)sp.stages * sp.stage_bytes + 8 * sp.stages;
    if (input_kind == 1) smem += (size_t)(R + 2) * (TQ + 8) * 4;
    if (smem > 110 * 1024) return 1;
    if (input_kind == 1) return launch_stream_kind<kSU8>(sp, smem, st);
    return word_bits == 64 ? launch_stream_kind<kSP64>(sp, smem, st)
                           : launch_stream_kind<kSP32>(sp, smem, st);
}

// Shared driver of every fused-edge entry point.
int edges_impl(const void *in, int input_kind, int64_t in_stride, const void *above,
               const void *below, uint32_t *o_edges, uint32_t *o_eset, uint32_t *const o_side[4],
               uint32_t *o_packed, int word_bits, int64_t out_stride_words, int64_t n, int64_t h,
               int64_t w, int fill_bit, int64_t row_lo, int64_t row_hi, void *stream, int thr = 1) {
    Geometry G;
    int rc = make_geometry(G, word_bits, n, h, w, fill_bit);
    if (rc) return rc;
    if (n == 0) return BE_OK;
    if (in == nullptr) return fail(BE_EINVAL, "input is NULL");
    if (input_kind != 0 && input_kind != 1)
        return fail(BE_EINVAL, "input_kind must be 0 (packed) or 1 (uint8)");
    if ((rc = check_stride(G, out_stride_words, "output"))) return rc;
    uint32_t *outs[7] = {o_edges, o_eset, o_side[0], o_side[1], o_side[2], o_side[3], o_packed};
    int any = 0;
    for (int i = 0; i < 7; ++i) {
        if (outs[i] == nullptr) continue;
        any = 1;
        if ((rc = check_ptr(outs[i], word_bits, "output"))) return rc;
        if ((const void *)outs[i] == in) return fail(BE_EINVAL, "output aliases the input");
    }
    if (!any) return fail(BE_EINVAL, "no output requested");
    if ((above || below) && n != 1)
        return fail(BE_EINVAL, "halo rows require a single slab (n == 1)");
    const int64_t nrows = n * h;
    if (row_lo < 0 || row_hi > nrows || row_lo > row_hi)
        return fail(BE_EINVAL, "row range [%lld, %lld) outside [0, %lld)", (long long)row_lo,
                    (long long)row_hi, (long long)nrows);
    if (row_lo == row_hi) return BE_OK;

    TileParams tp;
    memset(&tp, 0, sizeof(tp));
    tp.in = in; tp.above = above; tp.below = below;
    tp.o_edges = o_edges; tp.o_eset = o_eset;
    for (int s = 0; s < 4; ++s) tp.o_side[s] = o_side[s];
    tp.o_packed = o_packed;
    // strides in uint32 units for packed data
    tp.out_stride = word_bits == 64 ? 2 * out_stride_words : out_stride_words;
    tp.nrows = nrows; tp.h = h; tp.w = w; tp.row_lo = row_lo; tp.row_hi = row_hi;
    tp.wp = G.wp; tp.pl = G.pl; tp.lastbit = G.lastbit; tp.padmask = G.padmask;
    tp.fillword = G.fillword; tp.swap = G.swap;
    if (thr < 0 || thr > 255) return fail(BE_EINVAL, "threshold must be 0..255, got %d", thr);
    tp.thr = thr;

    // tile shape: TQ pixel words (power of two <= 64) x R rows, ~16 KB of
    // packed input or ~32 KB of uint8 input per CTA, smem <= 48 KB.
    const int TQ = G.wp <= 64 ? next_pow2(G.wp) : 64;
    const int64_t words_per_tile = input_kind == 1 ? 1024 : 4096;
    int64_t R = words_per_tile / TQ;
    const int64_t smem_cap_rows = (48 * 1024) / ((TQ + 8) * 4 + 1) - 2;
    while (R > smem_cap_rows) R >>= 1;
    const int64_t rows = row_hi - row_lo;
    while (R > 1 && R / 2 >= rows) R >>= 1;
    if (R < 1) R = 1;
    tp.log_tq = ilog2(TQ);
    tp.log_r = ilog2((int)R);
    tp.tiles_x = (G.wp + TQ - 1) / TQ;

    cudaStream_t st = S(stream);
    const bool only_edges = !o_side[0] && !o_side[1] && !o_side[2] && !o_side[3] && !o_packed;
    if (input_kind == 0) {
        if ((rc = check_ptr(in, word_bits, "input"))) return rc;
        if ((rc = check_stride(G, in_stride, "input"))) return rc;
        if (above && (rc = check_ptr(above, word_bits, "above halo"))) return rc;
        if (below && (rc = check_ptr(below, word_bits, "below halo"))) return rc;
        tp.in_stride = word_bits == 64 ? 2 * in_stride : in_stride;
        rc = try_reg(in, 0, in_stride * (word_bits / 8), above, below, o_edges, o_eset, o_side,
                     o_packed, tp.out_stride, G, nrows, row_lo, row_hi, st, thr);
        if (rc != 1) return rc;
        if (only_edges) {
            rc = try_stream(in, 0, in_stride * (word_bits / 8), above, below, o_edges, o_eset,
                            word_bits, tp.out_stride, G, nrows, row_lo, row_hi, st, thr);
            if (rc != 1) return rc;
        }
        bool vec = TQ >= 4 && (tp.in_stride % 4) == 0 && ((uintptr_t)in % 16) == 0 &&
                   (!above || ((uintptr_t)above % 16) == 0) &&
                   (!below || ((uintptr_t)below % 16) == 0);
        if (!vec) return launch_tile<kPScalar>(tp, rows, st);
        return word_bits == 64 ? launch_tile<kP64Vec>(tp, rows, st)
                               : launch_tile<kP32Vec>(tp, rows, st);
    }
    if (in_stride < w) return fail(BE_EINVAL, "input row stride %lld bytes < width %lld",
                                   (long long)in_stride, (long long)w);
    tp.in_stride = in_stride;
    rc = try_reg(in, 1, in_stride, above, below, o_edges, o_eset, o_side, o_packed,
                 tp.out_stride, G, nrows, row_lo, row_hi, st, thr);
    if (rc != 1) return rc;
    if (only_edges && word_bits == 32) {
        rc = try_stream(in, 1, in_stride, above, below, o_edges, o_eset, word_bits, tp.out_stride,
                        G, nrows, row_lo, row_hi, st, thr);
        if (rc != 1) return rc;
    }
    bool vec = (in_stride % 16) == 0 && ((uintptr_t)in % 16) == 0 &&
               (!above || ((uintptr_t)above % 16) == 0) && (!below || ((uintptr_t)below % 16) == 0);
    return vec ? launch_tile<kU8Vec>(tp, rows, st) : launch_tile<kU8Byte>(tp, rows, st);
}

// ---------------------------------------------------------------- small kernels

struct WordGeom {
    int64_t nrows, stride;  // uint32 units
    int wp, pl, swap;
    uint32_t lastbit, padmask, fillword;
    int64_t h;
};

WordGeom word_geom(const Geometry &G, int64_t stride_words) {
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

// invert / AND / OR (bitimage.py:181-205), padding re-forced to 1.
__global__ void bitop_kernel(int op, const uint32_t *__restrict__ a, const uint32_t *__restrict__ b,
                             uint32_t *__restrict__ out, WordGeom g) {
    const int64_t total = g.nrows * g.wp;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = t / g.wp;
        const int m = (int)(t - row * g.wp);
        const int64_t o = row * g.stride + m;
        uint32_t v = a[o];
        if (op == BE_OP_NOT) v = ~v;
        else if (op == BE_OP_AND) v &= b[o];
        else v |= b[o];
        out[o] = force_pad(g, m ^ g.swap, v);
    }
}

// Word of the shifted raster (bitimage.py:207-240); pw = pixel word, row = global row.
__device__ __forceinline__ uint32_t shifted_word(const uint32_t *__restrict__ in, const WordGeom &g,
                                                 int64_t row, int pw, int dir) {
    const uint32_t *r = in + row * g.stride;
    const int64_t y = row % g.h;
    switch (dir) {
        case BE_DOWN:   // out(y) = in(y-1): row 0 <- fill
            return y == 0 ? g.fillword : r[-g.stride + (pw ^ g.swap)];
        case BE_UP:     // out(y) = in(y+1): last row <- fill
            return y == g.h - 1 ? g.fillword : r[g.stride + (pw ^ g.swap)];
        case BE_RIGHT: {  // out(x) = in(x-1): pixel 0 <- fill
            const uint32_t c = r[pw ^ g.swap];
            const uint32_t l = pw == 0 ? g.fillword : r[(pw - 1) ^ g.swap];
            return __funnelshift_r(c, l, 1);
        }
        default: {      // BE_LEFT, out(x) = in(x+1): pixel w-1 <- fill
            if (pw > g.pl) return 0xFFFFFFFFu;
            const uint32_t c = r[pw ^ g.swap];
            const uint32_t rr = pw + 1 < g.wp ? r[(pw + 1) ^ g.swap] : 0u;
            uint32_t v = __funnelshift_l(rr, c, 1);
            if (pw == g.pl) v = (v & ~g.lastbit) | (g.fillword & g.lastbit);
            return v;
        }
    }
}

__global__ void shift_kernel(const uint32_t *__restrict__ in, const uint32_t *__restrict__ mask,
                             uint32_t *__restrict__ out, WordGeom g, int dir) {
    const int64_t total = g.nrows * g.wp;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = t / g.wp;
        const int pw = (int)(t - row * g.wp);
        uint32_t v = shifted_word(in, g, row, pw, dir);
        const int64_t o = row * g.stride + (pw ^ g.swap);
        if (mask) v &= mask[o];
        out[o] = force_pad(g, pw, v);
    }
}

__global__ void count_black_kernel(const uint32_t *__restrict__ in, unsigned long long *counts,
                                   WordGeom g) {
    const int64_t total = g.nrows * g.wp;
    unsigned long long acc = 0;
    int64_t cur_img = -1;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = t / g.wp;
        const int pw = (int)(t - row * g.wp);
        if (pw > g.pl) continue;
        uint32_t black = ~in[row * g.stride + (pw ^ g.swap)];
        if (pw == g.pl) black &= ~g.padmask;
        const int64_t img = row / g.h;
        if (img != cur_img) {
            if (cur_img >= 0 && acc) atomicAdd(counts + cur_img, acc);
            cur_img = img;
            acc = 0;
        }
        acc += __popc(black);
    }
    if (cur_img >= 0 && acc) atomicAdd(counts + cur_img, acc);
}

// to_array (bitimage.py:149-153): one thread per pixel word -> 32 bytes.
__global__ void unpack_kernel(const uint32_t *__restrict__ in, uint8_t *__restrict__ out,
                              WordGeom g, int64_t w, int64_t out_stride) {
    const int64_t total = g.nrows * (int64_t)(g.pl + 1);
    const int wpix = g.pl + 1;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = t / wpix;
        const int pw = (int)(t - row * wpix);
        const uint32_t v = in[row * g.stride + (pw ^ g.swap)];
        uint8_t *o = out + row * out_stride + (int64_t)pw * 32;
        const int64_t x0 = (int64_t)pw * 32;
        if (x0 + 32 <= w && ((uintptr_t)o % 16) == 0) {
            uint32_t q[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t nib = (v >> (28 - 4 * k)) & 0xFu;   // pixels 4k..4k+3
                q[k] = ((nib >> 3) & 1u) | (((nib >> 2) & 1u) << 8) | (((nib >> 1) & 1u) << 16) |
                       ((nib & 1u) << 24);
            }
            reinterpret_cast<uint4 *>(o)[0] = make_uint4(q[0], q[1], q[2], q[3]);
            reinterpret_cast<uint4 *>(o)[1] = make_uint4(q[4], q[5], q[6], q[7]);
        } else {
            for (int b = 0; b < 32 && x0 + b < w; ++b) o[b] = (v >> (31 - b)) & 1u;
        }
    }
}

// detect_edges_scan: the paper's "traditional scanning",
// Edge(p) = p' AND (n2 OR n4 OR n6 OR n8) evaluated pixel by pixel -- an
// algorithm independent of the mask kernels (no word-wide shifts or ORs), used
// as the full-size GPU cross-check.  A thread owns one
// 32-pixel word: it loads the five words its pixels' neighbours can live in
// (centre, above, below, left, right; the border fill where they fall outside)
// once, then walks its 32 pixels one at a time.
__device__ __forceinline__ uint32_t scan_word_at(const uint32_t *__restrict__ in, const WordGeom &g,
                                                 int64_t row, int pw) {
    return in[row * g.stride + (pw ^ g.swap)];
}

__global__ void scan_kernel(const uint32_t *__restrict__ in, uint32_t *__restrict__ out, WordGeom g,
                            int64_t w) {
    const int64_t total = g.nrows * g.wp;
    const uint32_t fill = g.fillword & 1u;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = t / g.wp;
        const int pw = (int)(t - row * g.wp);
        const int64_t y = row % g.h;
        const uint32_t c = scan_word_at(in, g, row, pw);
        const uint32_t up = y > 0 ? scan_word_at(in, g, row - 1, pw) : 0u;
        const uint32_t dn = y + 1 < g.h ? scan_word_at(in, g, row + 1, pw) : 0u;
        const uint32_t lw = pw > 0 ? scan_word_at(in, g, row, pw - 1) : 0u;
        const uint32_t rw = pw + 1 < g.wp ? scan_word_at(in, g, row, pw + 1) : 0u;
        uint32_t word = 0;
        for (int b = 0; b < 32; ++b) {
            const int64_t x = (int64_t)pw * 32 + b;
            uint32_t bit = 1u;
            if (x < w) {
                const uint32_t p = (c >> (31 - b)) & 1u;
                // n2 (above) and n6 (below): same column, rows y-1 / y+1
                const uint32_t n2 = y > 0 ? (up >> (31 - b)) & 1u : fill;
                const uint32_t n6 = y + 1 < g.h ? (dn >> (31 - b)) & 1u : fill;
                // n4 (left): pixel x-1, in the previous word when b == 0
                const uint32_t n4 = x == 0 ? fill : (b == 0 ? lw & 1u : (c >> (32 - b)) & 1u);
                // n8 (right): pixel x+1, in the next word when b == 31
                const uint32_t n8 = x + 1 >= w ? fill : (b == 31 ? rw >> 31 : (c >> (30 - b)) & 1u);
                bit = !(!p && (n2 | n4 | n6 | n8));
            }
            word = (word << 1) | bit;
        }
        out[row * g.stride + (pw ^ g.swap)] = word;
    }
}

unsigned grid_for(int64_t total) {
    int64_t blocks = (total + 255) / 256;
    const int64_t cap = 148 * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return (unsigned)blocks;
}

int prep_words(Geometry &G, int word_bits, int64_t n, int64_t h, int64_t w, int64_t stride,
               int fill_bit, const void *a, const char *aname, const void *out) {
    int rc = make_geometry(G, word_bits, n, h, w, fill_bit);
    if (rc) return rc;
    if ((rc = check_stride(G, stride, "row"))) return rc;
    if (n == 0) return BE_OK;
    if ((rc = check_ptr(a, word_bits, aname))) return rc;
    if ((rc = check_ptr(out, word_bits, "output"))) return rc;
    return BE_OK;
}

// ---------------------------------------------------------------- PBM P4 codec (F1)
// P4 payload rows are ceil(w/8) bytes, MSB-first, 1 = black;
// the rasters here are MSB-first words with 1 = white and padding 1.

__global__ void p4_decode_kernel(const uint8_t *__restrict__ p4, uint32_t *__restrict__ out,
                                 WordGeom g, int64_t rb, int64_t out_stride) {
    const int64_t total = g.nrows * g.wp;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = t / g.wp;
        const int pw = (int)(t - row * g.wp);
        const uint8_t *r = p4 + row * rb;
        uint32_t v = 0u;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t j = (int64_t)pw * 4 + k;
            v = (v << 8) | (j < rb ? r[j] : 0u);
        }
        out[row * out_stride + (pw ^ g.swap)] = force_pad(g, pw, ~v);
    }
}

__global__ void p4_encode_kernel(const uint32_t *__restrict__ in, uint8_t *__restrict__ p4,
                                 WordGeom g, int64_t rb, int64_t in_stride) {
    const int64_t total = g.nrows * rb;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = t / rb;
        const int64_t j = t - row * rb;
        const int pw = (int)(j >> 2);
        uint32_t v = in[row * in_stride + (pw ^ g.swap)];
        if (pw == g.pl) v |= g.padmask;            // padding -> 0 on disk
        p4[t] = (uint8_t)(~(v >> (24 - 8 * (j & 3))));
    }
}

}  // namespace

// ================================================================ C ABI

extern "C" int be_p4_decode(const uint8_t *p4, void *out, int word_bits, int64_t n, int64_t h,
                            int64_t w, int64_t out_row_stride_words, void *stream) {
    Geometry G;
    int rc = make_geometry(G, word_bits, n, h, w, 1);
    if (rc) return rc;
    if ((rc = check_stride(G, out_row_stride_words, "output"))) return rc;
    if (n == 0) return BE_OK;
    if (p4 == nullptr) return fail(BE_EINVAL, "P4 payload is NULL");
    if ((rc = check_ptr(out, word_bits, "output"))) return rc;
    WordGeom g = word_geom(G, out_row_stride_words);
    const int64_t rb = (w + 7) / 8;
    p4_decode_kernel<<<grid_for(g.nrows * g.wp), 256, 0, S(stream)>>>(p4, (uint32_t *)out, g, rb,
                                                                       g.stride);
    return cuda_check("p4_decode_kernel");
}

extern "C" int be_p4_encode(const void *in, uint8_t *p4, int word_bits, int64_t n, int64_t h,
                            int64_t w, int64_t in_row_stride_words, void *stream) {
    Geometry G;
    int rc = make_geometry(G, word_bits, n, h, w, 1);
    if (rc) return rc;
    if ((rc = check_stride(G, in_row_stride_words, "input"))) return rc;
    if (n == 0) return BE_OK;
    if (p4 == nullptr) return fail(BE_EINVAL, "P4 payload is NULL");
    if ((rc = check_ptr(in, word_bits, "input"))) return rc;
    WordGeom g = word_geom(G, in_row_stride_words);
    const int64_t rb = (w + 7) / 8;
    p4_encode_kernel<<<grid_for(g.nrows * rb), 256, 0, S(stream)>>>((const uint32_t *)in, p4, g,
                                                                     rb, g.stride);
    return cuda_check("p4_encode_kernel");
}

extern "C" int be_p4_edges(const uint8_t *p4_in, uint8_t *p4_out, int64_t n, int64_t h, int64_t w,
                           int fill_bit, uint32_t *scratch_or_null, void *stream) {
    Geometry G;
    int rc = make_geometry(G, 32, n, h, w, fill_bit);
    if (rc) return rc;
    if (n == 0) return BE_OK;
    if (p4_in == nullptr || p4_out == nullptr) return fail(BE_EINVAL, "P4 buffers must not be NULL");
    if ((const void *)p4_in == (const void *)p4_out) return fail(BE_EINVAL, "output aliases the input");
    const int64_t rb = (w + 7) / 8;
    cudaStream_t st = S(stream);
    auto al = [](const void *p, int a) { return ((uintptr_t)p % a) == 0; };
    // fused path: P4 rows are whole 16-byte chunks -> K1 reads and writes P4 directly
    if (rb % 16 == 0 && al(p4_in, 16) && al(p4_out, 16) && !getenv("BITEDGE_P4_UNFUSED") &&
        n * h < ((int64_t)1 << 31)) {
        RegParams rp;
        memset(&rp, 0, sizeof(rp));
        rp.in = (const char *)p4_in; rp.in_row_bytes = rb;
        rp.o_edges = (uint32_t *)p4_out; rp.out_stride = rb / 4;
        rp.nrows = n * h; rp.row_lo = 0; rp.row_hi = n * h;
        rp.h = (uint32_t)h; rp.w = w; rp.wp = G.wp; rp.pl = G.pl;
        rp.lastbit = G.lastbit; rp.padmask = G.padmask; rp.fillword = G.fillword;
        rp.thr = 1;
        const bool v8 = rb % 32 == 0 && al(p4_in, 32) && al(p4_out, 32);
        const int cw = v8 ? 8 : 4;
        rp.items = (G.wp + cw - 1) / cw;
        rp.vst = 1;
        // 2-row strips for small rasters (twice the threads in flight), as try_reg does
        const bool big = ((n * h + 3) / 4) * ((G.wp + 7) / 8) >= (int64_t)sm_count() * 4096;
        const int rs = big ? 4 : 2;
        rp.nstrips = (n * h + rs - 1) / rs;
        const int64_t grid = (rp.nstrips * rp.items + kThreads - 1) / kThreads;
        if (grid <= 0x7FFFFFFFLL) {
            if (cw == 8 && rs == 4)
                launch_k(edge_reg_packed_kernel<0, 4, 8, kOutEdges, false, true>, (unsigned)grid, 0,
                         st, rp);
            else if (cw == 8)
                launch_k(edge_reg_packed_kernel<0, 2, 8, kOutEdges, false, true>, (unsigned)grid, 0,
                         st, rp);
            else if (rs == 4)
                launch_k(edge_reg_packed_kernel<0, 4, 4, kOutEdges, false, true>, (unsigned)grid, 0,
                         st, rp);
            else
                launch_k(edge_reg_packed_kernel<0, 2, 4, kOutEdges, false, true>, (unsigned)grid, 0,
                         st, rp);
            return cuda_check("edge_reg_packed_kernel<P4>");
        }
    }
    // general path: decode -> K1 -> encode through caller scratch (2 word rasters)
    if (scratch_or_null == nullptr)
        return fail(BE_EINVAL, "unaligned P4 rows (ceil(w/8) %% 16 != 0) need a scratch buffer of "
                               "2 * n * h * ceil(w/32) words");
    const int64_t words = n * h * G.wp;
    uint32_t *dec = scratch_or_null, *edg = scratch_or_null + words;
    if ((rc = be_p4_decode(p4_in, dec, 32, n, h, w, G.wp, stream))) return rc;
    if ((rc = be_edge_packed_u32(dec, edg, n, h, w, G.wp, fill_bit, 0, stream))) return rc;
    return be_p4_encode(edg, p4_out, 32, n, h, w, G.wp, stream);
}

extern "C" {

const char *be_last_error(void) { return g_err; }
int be_abi_version(void) { return BE_ABI_VERSION; }
int64_t be_launch_count(void) { return g_launches; }

int be_edges_general(const void *in, int input_kind, int64_t in_row_stride,
                     const void *above_or_null, const void *below_or_null, const be_outputs *outs,
                     int word_bits, int64_t out_row_stride_words, int64_t n, int64_t h, int64_t w,
                     int fill_bit, int64_t row_lo, int64_t row_hi, void *stream) {
    if (outs == nullptr) return fail(BE_EINVAL, "outputs is NULL");
    uint32_t *side[4] = {(uint32_t *)outs->side[0], (uint32_t *)outs->side[1],
                         (uint32_t *)outs->side[2], (uint32_t *)outs->side[3]};
    return edges_impl(in, input_kind, in_row_stride, above_or_null, below_or_null,
                      (uint32_t *)outs->edges, (uint32_t *)outs->edgeset, side,
                      (uint32_t *)outs->packed, word_bits, out_row_stride_words, n, h, w, fill_bit,
                      row_lo, row_hi, stream);
}

static int edge_packed(const void *in, void *out, int word_bits, int64_t n, int64_t h, int64_t w,
                       int64_t stride, int fill_bit, int emit_edgeset, void *stream) {
    uint32_t *side[4] = {nullptr, nullptr, nullptr, nullptr};
    uint32_t *o = (uint32_t *)out;
    return edges_impl(in, 0, stride, nullptr, nullptr, emit_edgeset ? nullptr : o,
                      emit_edgeset ? o : nullptr, side, nullptr, word_bits, stride, n, h, w,
                      fill_bit, 0, n * h, stream);
}

int be_edge_packed_u32(const uint32_t *in, uint32_t *out, int64_t n, int64_t h, int64_t w,
                       int64_t row_stride_words, int fill_bit, int emit_edgeset, void *stream) {
    return edge_packed(in, out, 32, n, h, w, row_stride_words, fill_bit, emit_edgeset, stream);
}

int be_edge_packed_u64(const uint64_t *in, uint64_t *out, int64_t n, int64_t h, int64_t w,
                       int64_t row_stride_words, int fill_bit, int emit_edgeset, void *stream) {
    return edge_packed(in, out, 64, n, h, w, row_stride_words, fill_bit, emit_edgeset, stream);
}

int be_pack_edge_u8(const uint8_t *in, uint32_t *out, int64_t n, int64_t h, int64_t w,
                    int64_t in_row_stride, int64_t out_row_stride_words, int fill_bit,
                    uint32_t *packed_in_or_null, void *stream) {
    uint32_t *side[4] = {nullptr, nullptr, nullptr, nullptr};
    if (out == nullptr && n != 0) return fail(BE_EINVAL, "output is NULL");
    return edges_impl(in, 1, in_row_stride, nullptr, nullptr, out, nullptr, side, packed_in_or_null,
                      32, out_row_stride_words, n, h, w, fill_bit, 0, n * h, stream);
}

int be_edge_packed_halo_u32(const uint32_t *slab, const uint32_t *above_or_null,
                            const uint32_t *below_or_null, uint32_t *out, int64_t rows, int64_t w,
                            int64_t row_stride_words, int fill_bit, int64_t row_lo, int64_t row_hi,
                            void *stream) {
    uint32_t *side[4] = {nullptr, nullptr, nullptr, nullptr};
    if (out == nullptr) return fail(BE_EINVAL, "output is NULL");
    return edges_impl(slab, 0, row_stride_words, above_or_null, below_or_null, out, nullptr, side,
                      nullptr, 32, row_stride_words, 1, rows, w, fill_bit, row_lo, row_hi, stream);
}

int be_pack_u8(const uint8_t *in, void *out, int word_bits, int64_t n, int64_t h, int64_t w,
               int64_t in_row_stride, int64_t out_row_stride_words, void *stream) {
    uint32_t *side[4] = {nullptr, nullptr, nullptr, nullptr};
    if (out == nullptr && n != 0) return fail(BE_EINVAL, "output is NULL");
    return edges_impl(in, 1, in_row_stride, nullptr, nullptr, nullptr, nullptr, side,
                      (uint32_t *)out, word_bits, out_row_stride_words, n, h, w, 1, 0, n * h,
                      stream);
}

int be_unpack_u8(const void *in, uint8_t *out, int word_bits, int64_t n, int64_t h, int64_t w,
                 int64_t in_row_stride_words, int64_t out_row_stride, void *stream) {
    Geometry G;
    int rc = make_geometry(G, word_bits, n, h, w, 1);
    if (rc) return rc;
    if ((rc = check_stride(G, in_row_stride_words, "input"))) return rc;
    if (out_row_stride < w) return fail(BE_EINVAL, "output row stride < width");
    if (n == 0) return BE_OK;
    if ((rc = check_ptr(in, word_bits, "input"))) return rc;
    if (out == nullptr && n != 0) return fail(BE_EINVAL, "output is NULL");
    WordGeom g = word_geom(G, in_row_stride_words);
    unpack_kernel<<<grid_for(g.nrows * (g.pl + 1)), 256, 0, S(stream)>>>(
        (const uint32_t *)in, out, g, w, out_row_stride);
    return cuda_check("unpack_kernel");
}

int be_bitop(int op, const void *a, const void *b, void *out, int word_bits, int64_t n, int64_t h,
             int64_t w, int64_t row_stride_words, void *stream) {
    Geometry G;
    if (op != BE_OP_NOT && op != BE_OP_AND && op != BE_OP_OR)
        return fail(BE_EINVAL, "unknown op %d", op);
    int rc = prep_words(G, word_bits, n, h, w, row_stride_words, 1, a, "operand a", out);
    if (rc || n == 0) return rc;
    if (op != BE_OP_NOT && (rc = check_ptr(b, word_bits, "operand b"))) return rc;
    WordGeom g = word_geom(G, row_stride_words);
    bitop_kernel<<<grid_for(g.nrows * g.wp), 256, 0, S(stream)>>>(
        op, (const uint32_t *)a, (const uint32_t *)b, (uint32_t *)out, g);
    return cuda_check("bitop_kernel");
}

int be_shift(const void *in, void *out, int word_bits, int64_t n, int64_t h, int64_t w,
             int64_t row_stride_words, int direction, int fill_bit, void *stream) {
    Geometry G;
    if (direction < BE_LEFT || direction > BE_DOWN)
        return fail(BE_EINVAL, "unknown direction %d", direction);
    int rc = prep_words(G, word_bits, n, h, w, row_stride_words, fill_bit, in, "input", out);
    if (rc || n == 0) return rc;
    if (in == out) return fail(BE_EINVAL, "output aliases the input");
    WordGeom g = word_geom(G, row_stride_words);
    shift_kernel<<<grid_for(g.nrows * g.wp), 256, 0, S(stream)>>>(
        (const uint32_t *)in, nullptr, (uint32_t *)out, g, direction);
    return cuda_check("shift_kernel");
}

int be_shift_and(const void *img, const void *mask, void *out, int word_bits, int64_t n,
                 int64_t h, int64_t w, int64_t row_stride_words, int side, int fill_bit,
                 void *stream) {
    Geometry G;
    if (side < BE_LEFT || side > BE_DOWN) return fail(BE_EINVAL, "unknown side %d", side);
    int rc = prep_words(G, word_bits, n, h, w, row_stride_words, fill_bit, img, "image", out);
    if (rc || n == 0) return rc;
    if ((rc = check_ptr(mask, word_bits, "mask"))) return rc;
    if (img == out) return fail(BE_EINVAL, "output aliases the input");
    static const int opposite[4] = {BE_RIGHT, BE_LEFT, BE_DOWN, BE_UP};
    WordGeom g = word_geom(G, row_stride_words);
    shift_kernel<<<grid_for(g.nrows * g.wp), 256, 0, S(stream)>>>(
        (const uint32_t *)img, (const uint32_t *)mask, (uint32_t *)out, g, opposite[side]);
    return cuda_check("shift_kernel");
}

int be_count_black(const void *in, int64_t *counts, int word_bits, int64_t n, int64_t h,
                   int64_t w, int64_t row_stride_words, void *stream) {
    Geometry G;
    int rc = make_geometry(G, word_bits, n, h, w, 1);
    if (rc) return rc;
    if ((rc = check_stride(G, row_stride_words, "row"))) return rc;
    if (n == 0) return BE_OK;
    if ((rc = check_ptr(in, word_bits, "input"))) return rc;
    if (counts == nullptr || ((uintptr_t)counts % 8)) return fail(BE_EINVAL, "bad counts pointer");
    cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(int64_t) * n, S(stream));
    if (e != cudaSuccess) return fail((int)e, "cudaMemsetAsync: %s", cudaGetErrorString(e));
    WordGeom g = word_geom(G, row_stride_words);
    count_black_kernel<<<grid_for(g.nrows * g.wp), 256, 0, S(stream)>>>(
        (const uint32_t *)in, (unsigned long long *)counts, g);
    return cuda_check("count_black_kernel");
}

int be_scan_edges(const void *in, void *out, int word_bits, int64_t n, int64_t h, int64_t w,
                  int64_t row_stride_words, int fill_bit, void *stream) {
    Geometry G;
    int rc = prep_words(G, word_bits, n, h, w, row_stride_words, fill_bit, in, "input", out);
    if (rc || n == 0) return rc;
    if (in == out) return fail(BE_EINVAL, "output aliases the input");
    WordGeom g = word_geom(G, row_stride_words);
    scan_kernel<<<grid_for(g.nrows * g.wp), 256, 0, S(stream)>>>(
        (const uint32_t *)in, (uint32_t *)out, g, w);
    return cuda_check("scan_kernel");
}

int be_threshold_edge_u8(const uint8_t *in, uint32_t *out, int64_t n, int64_t h, int64_t w,
                         int64_t in_row_stride, int64_t out_row_stride_words, int threshold,
                         int fill_bit, uint32_t *binary_or_null, void *stream) {
    uint32_t *side[4] = {nullptr, nullptr, nullptr, nullptr};
    if (out == nullptr && n != 0) return fail(BE_EINVAL, "output is NULL");
    return edges_impl(in, 1, in_row_stride, nullptr, nullptr, out, nullptr, side, binary_or_null,
                      32, out_row_stride_words, n, h, w, fill_bit, 0, n * h, stream, threshold);
}

int be_threshold_u8(const uint8_t *in, void *out, int word_bits, int64_t n, int64_t h, int64_t w,
                    int64_t in_row_stride, int64_t out_row_stride_words, int threshold,
                    void *stream) {
    uint32_t *side[4] = {nullptr, nullptr, nullptr, nullptr};
    if (out == nullptr && n != 0) return fail(BE_EINVAL, "output is NULL");
    return edges_impl(in, 1, in_row_stride, nullptr, nullptr, nullptr, nullptr, side,
                      (uint32_t *)out, word_bits, out_row_stride_words, n, h, w, 1, 0, n * h,
                      stream, threshold);
}

// ---- peer-memory halos: CUDA IPC export / import of a device buffer --------

typedef int (*cuMemGetAddressRange_t)(unsigned long long *, size_t *, unsigned long long);

int be_ipc_export(const void *dev_ptr, void *handle_out, int64_t *offset_out) {
    if (dev_ptr == nullptr || handle_out == nullptr || offset_out == nullptr)
        return fail(BE_EINVAL, "NULL argument");
    // the IPC handle names the whole allocation: find its base through the driver
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || fn == nullptr)
        return fail(e != cudaSuccess ? (int)e : BE_EINVAL, "cuMemGetAddressRange unavailable");
    unsigned long long base = 0;
    size_t size = 0;
    if (((cuMemGetAddressRange_t)fn)(&base, &size, (unsigned long long)(uintptr_t)dev_ptr) != 0)
        return fail(BE_EINVAL, "pointer is not a device allocation");
    cudaIpcMemHandle_t h;
    e = cudaIpcGetMemHandle(&h, (void *)(uintptr_t)base);
    if (e != cudaSuccess) return fail((int)e, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    memcpy(handle_out, &h, sizeof(h));
    *offset_out = (int64_t)((uintptr_t)dev_ptr - base);
    return BE_OK;
}

int be_ipc_open(const void *handle, int64_t offset, void **dev_ptr_out) {
    if (handle == nullptr || dev_ptr_out == nullptr) return fail(BE_EINVAL, "NULL argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void *base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail((int)e, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    *dev_ptr_out = (char *)base + offset;
    return BE_OK;
}

int be_ipc_close(void *dev_ptr, int64_t offset) {
    if (dev_ptr == nullptr) return fail(BE_EINVAL, "NULL argument");
    cudaError_t e = cudaIpcCloseMemHandle((char *)dev_ptr - offset);
    if (e != cudaSuccess) return fail((int)e, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
    return BE_OK;
}

int be_host_edges(const void *host_in, int input_kind, uint32_t *host_out, int64_t n, int64_t h,
                  int64_t w, int fill_bit, void *const dev_in[2], uint32_t *const dev_out[2],
                  int64_t chunk_images, void *stream0, void *stream1, int blocking) {
    Geometry G;
    int rc = make_geometry(G, 32, n, h, w, fill_bit);
    if (rc) return rc;
    if (n == 0) return BE_OK;
    if (!host_in || !host_out || !dev_in || !dev_out || !dev_in[0] || !dev_in[1] || !dev_out[0] ||
        !dev_out[1])
        return fail(BE_EINVAL, "host / device buffers must not be NULL");
    if (input_kind != 0 && input_kind != 1)
        return fail(BE_EINVAL, "input_kind must be 0 (packed u32) or 1 (uint8)");
    if (chunk_images < 1) return fail(BE_EINVAL, "chunk_images must be >= 1");
    const int64_t wp = G.wp;
    const size_t in_img = (size_t)h * (input_kind == 1 ? (size_t)w : (size_t)wp * 4);
    const size_t out_img = (size_t)h * wp * 4;
    cudaStream_t ss[2] = {S(stream0), S(stream1)};
    uint32_t *side[4] = {nullptr, nullptr, nullptr, nullptr};
    // chunk c runs entirely on stream c % 2: H2D -> kernel -> D2H.  In-stream
    // order protects the reuse of buffer c % 2 by chunk c + 2, and the two
    // streams let one chunk's H2D overlap the other's kernel and D2H.
    for (int64_t c = 0, lo = 0; lo < n; ++c, lo += chunk_images) {
        const int64_t k = (n - lo) < chunk_images ? (n - lo) : chunk_images;
        const int b = (int)(c & 1);
        cudaError_t e = cudaMemcpyAsync(dev_in[b], (const char *)host_in + lo * in_img, k * in_img,
                                        cudaMemcpyHostToDevice, ss[b]);
        if (e != cudaSuccess) return fail((int)e, "H2D: %s", cudaGetErrorString(e));
        rc = edges_impl(dev_in[b], input_kind, input_kind == 1 ? w : wp, nullptr, nullptr,
                        dev_out[b], nullptr, side, nullptr, 32, wp, k, h, w, fill_bit, 0, k * h,
                        ss[b]);
        if (rc) return rc;
        e = cudaMemcpyAsync((char *)host_out + lo * out_img, dev_out[b], k * out_img,
                            cudaMemcpyDeviceToHost, ss[b]);
        if (e != cudaSuccess) return fail((int)e, "D2H: %s", cudaGetErrorString(e));
    }
    if (blocking) {
        for (int b = 0; b < 2; ++b) {
            cudaError_t e = cudaStreamSynchronize(ss[b]);
            if (e != cudaSuccess) return fail((int)e, "sync: %s", cudaGetErrorString(e));
        }
    }
    return BE_OK;
}

int be_host_edges_rows(const void *host_in, int input_kind, uint32_t *host_out, int64_t h,
                       int64_t w, int fill_bit, int halo_flags, void *const dev_in[2],
                       uint32_t *const dev_out[2], int64_t chunk_rows, void *stream0,
                       void *stream1, int blocking) {
    Geometry G;
    int rc = make_geometry(G, 32, 1, h, w, fill_bit);
    if (rc) return rc;
    if (!host_in || !host_out || !dev_in || !dev_out || !dev_in[0] || !dev_in[1] || !dev_out[0] ||
        !dev_out[1])
        return fail(BE_EINVAL, "host / device buffers must not be NULL");
    if (input_kind != 0 && input_kind != 1)
        return fail(BE_EINVAL, "input_kind must be 0 (packed u32) or 1 (uint8)");
    if (chunk_rows < 1) return fail(BE_EINVAL, "chunk_rows must be >= 1");
    if (halo_flags & ~3) return fail(BE_EINVAL, "halo_flags must be a combination of 1 and 2");
    const int64_t wp = G.wp;
    const size_t in_row = input_kind == 1 ? (size_t)w : (size_t)wp * 4;
    const size_t out_row = (size_t)wp * 4;
    const bool has_above = halo_flags & 1, has_below = halo_flags & 2;
    // row r of the image is host row r + has_above; rows -1 / h exist iff flagged
    const char *hin = (const char *)host_in + (has_above ? in_row : 0);
    cudaStream_t ss[2] = {S(stream0), S(stream1)};
    uint32_t *side[4] = {nullptr, nullptr, nullptr, nullptr};
    // chunk c on stream c % 2: H2D of rows [r0-1, r1+1) -> halo kernel on rows
    // [r0, r1) -> D2H; in-stream order protects buffer c % 2 for chunk c + 2
    for (int64_t c = 0, r0 = 0; r0 < h; ++c, r0 += chunk_rows) {
        const int64_t r1 = (h - r0) < chunk_rows ? h : r0 + chunk_rows;
        const bool up = r0 > 0 || has_above, dn = r1 < h || has_below;
        const int64_t lo = up ? r0 - 1 : r0, hi = dn ? r1 + 1 : r1;
        const int b = (int)(c & 1);
        char *din = (char *)dev_in[b];
        cudaError_t e = cudaMemcpyAsync(din, hin + lo * (int64_t)in_row, (hi - lo) * in_row,
                                        cudaMemcpyHostToDevice, ss[b]);
        if (e != cudaSuccess) return fail((int)e, "H2D: %s", cudaGetErrorString(e));
        const char *slab = din + (r0 - lo) * in_row;
        const void *above = up ? (const void *)din : nullptr;
        const void *below = dn ? (const void *)(slab + (r1 - r0) * in_row) : nullptr;
        rc = edges_impl(slab, input_kind, input_kind == 1 ? w : wp, above, below, dev_out[b],
                        nullptr, side, nullptr, 32, wp, 1, r1 - r0, w, fill_bit, 0, r1 - r0, ss[b]);
        if (rc) return rc;
        e = cudaMemcpyAsync((char *)host_out + r0 * out_row, dev_out[b], (r1 - r0) * out_row,
                            cudaMemcpyDeviceToHost, ss[b]);
        if (e != cudaSuccess) return fail((int)e, "D2H: %s", cudaGetErrorString(e));
    }
    if (blocking) {
        for (int b = 0; b < 2; ++b) {
            cudaError_t e = cudaStreamSynchronize(ss[b]);
            if (e != cudaSuccess) return fail((int)e, "sync: %s", cudaGetErrorString(e));
        }
    }
    return BE_OK;
}

}  // extern "C"

// capi_edges.cu -- the fused edge kernels' host side: kernel selection (tile /
// TMA-stream / register-direct K1, K2, K2w, K2r, K2t, K2t2, halos, multi-output)
// and the C-ABI entry points that compute edges (include/bitedge.h).
#include "capi_internal.cuh"
#include "edge_flat.cuh"
#include "edge_reg.cuh"
#include "edge_stream.cuh"

using namespace bitedge;
using namespace bitedge::capi;

namespace bitedge {
namespace capi {

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

// Kernel selection knob for A/B measurements: BITEDGE_KERNEL=tile forces the
// one-shot tile kernel, =stream forbids nothing (default: stream when eligible).
bool stream_allowed() {
    const char *e = knob(KN_KERNEL);
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

// K1's tail-free (ALIGNED) instantiations apply: edges and / or EdgeSet (not the
// kOutAll multi-output), 8-word items, whole items with no padding bits
// (BITEDGE_K1_GENERIC turns them off).
inline bool k1_aligned(bool single, int cw, int64_t w) {
    return single && cw == 8 && w % 256 == 0 && !knob(KN_K1_GENERIC);
}

// Launch helpers: dispatch the runtime choices onto template parameters.
template <int OUT, bool HALO>
int launch_reg_packed(RegParams &rp, int swap, int cw, int rs, unsigned grid, cudaStream_t st) {
    K1Div dv;
    if (!k1_setup(rp, dv)) return kNoKernel;   // > 2^32 threads or rows: tile kernel
    if (rp.in_end != nullptr) {                // UNAL: 4-byte aligned rows, 4-word items
        if constexpr (OUT == kOutAll || HALO) {
            return kNoKernel;
        } else {
            if (swap && rs == 2) launch_k(edge_reg_packed_kernel<1, 2, 4, OUT, false, false, false, true>, grid, 0, st, rp, dv);
            else if (swap) launch_k(edge_reg_packed_kernel<1, 4, 4, OUT, false, false, false, true>, grid, 0, st, rp, dv);
            else if (rs == 2) launch_k(edge_reg_packed_kernel<0, 2, 4, OUT, false, false, false, true>, grid, 0, st, rp, dv);
            else launch_k(edge_reg_packed_kernel<0, 4, 4, OUT, false, false, false, true>, grid, 0, st, rp, dv);
            return cuda_check("edge_reg_packed_kernel<UNAL>");
        }
    }
    if constexpr (OUT != kOutAll) {
        if (rp.h16) {                                      // 16-byte rows, 8-word items
            if (cw != 8 || (rs != 2 && rs != 4)) return kNoKernel;
            if (swap && rs == 2) launch_k(edge_reg_packed_kernel<1, 2, 8, OUT, HALO, false, false, false, true>, grid, 0, st, rp, dv);
            else if (swap) launch_k(edge_reg_packed_kernel<1, 4, 8, OUT, HALO, false, false, false, true>, grid, 0, st, rp, dv);
            else if (rs == 2) launch_k(edge_reg_packed_kernel<0, 2, 8, OUT, HALO, false, false, false, true>, grid, 0, st, rp, dv);
            else launch_k(edge_reg_packed_kernel<0, 4, 8, OUT, HALO, false, false, false, true>, grid, 0, st, rp, dv);
            return cuda_check("edge_reg_packed_kernel<H16>");
        }
    }
    if constexpr (OUT == kOutAll) {   // up to 7 outputs: 4-word items keep it in registers
        if (swap) launch_k(edge_reg_packed_kernel<1, 4, 4, OUT, HALO>, grid, 0, st, rp, dv);
        else if (rs == 2) launch_k(edge_reg_packed_kernel<0, 2, 4, OUT, HALO>, grid, 0, st, rp, dv);
        else launch_k(edge_reg_packed_kernel<0, 4, 4, OUT, HALO>, grid, 0, st, rp, dv);
        (void)cw;
    } else {
        // whole 8-word items with no padding (w % 256 == 0: C3, C4, and the drop-in's
        // uint64 BitImage words at those widths): the tail-free kernels
        const bool aligned = k1_aligned(OUT != kOutAll, cw, rp.w);
        if (aligned && swap && rs == 2) {
            launch_k(edge_reg_packed_kernel<1, 2, 8, OUT, HALO, false, true>, grid, 0, st, rp, dv);
        } else if (aligned && swap && rs == 4) {
            launch_k(edge_reg_packed_kernel<1, 4, 8, OUT, HALO, false, true>, grid, 0, st, rp, dv);
        } else if (aligned && rs == 2) {
            launch_k(edge_reg_packed_kernel<0, 2, 8, OUT, HALO, false, true>, grid, 0, st, rp, dv);
        } else if (aligned && rs == 4) {
            launch_k(edge_reg_packed_kernel<0, 4, 8, OUT, HALO, false, true>, grid, 0, st, rp, dv);
        } else if (!swap && rs == 2) {
            // (128-thread CTAs for C3's single wave: +2 % overlapped, -1 % serial; not taken)
            if (cw == 8) launch_k(edge_reg_packed_kernel<0, 2, 8, OUT, HALO>, grid, 0, st, rp, dv);
            else launch_k(edge_reg_packed_kernel<0, 2, 4, OUT, HALO>, grid, 0, st, rp, dv);
        } else if (!swap && rs == 8) {
            if (cw == 8) launch_k(edge_reg_packed_kernel<0, 8, 8, OUT, HALO>, grid, 0, st, rp, dv);
            else launch_k(edge_reg_packed_kernel<0, 8, 4, OUT, HALO>, grid, 0, st, rp, dv);
        } else if (swap) {
            if (cw == 8) launch_k(edge_reg_packed_kernel<1, 4, 8, OUT, HALO>, grid, 0, st, rp, dv);
            else launch_k(edge_reg_packed_kernel<1, 4, 4, OUT, HALO>, grid, 0, st, rp, dv);
        } else {
            if (cw == 8) launch_k(edge_reg_packed_kernel<0, 4, 8, OUT, HALO>, grid, 0, st, rp, dv);
            else launch_k(edge_reg_packed_kernel<0, 4, 4, OUT, HALO>, grid, 0, st, rp, dv);
        }
    }
    return cuda_check("edge_reg_packed_kernel");
}

template <int OUT, bool HALO>
int launch_reg_u8(RegParams &rp, int rs, unsigned grid, cudaStream_t st) {
    if (rp.in_end != nullptr) {                  // UNAL: rows at any byte, no halos
        if constexpr (HALO) {
            return kNoKernel;
        } else {
            // widest alignment every row start has (rp.v8 carries it: 8, 4 or 1);
            // 2-row strips for small rasters (twice the threads in flight)
            if (rs == 2) {
                if (rp.v8 == 8) launch_k(edge_reg_u8_kernel<2, OUT, false, false, 8>, grid, 0, st, rp);
                else if (rp.v8 == 4) launch_k(edge_reg_u8_kernel<2, OUT, false, false, 4>, grid, 0, st, rp);
                else launch_k(edge_reg_u8_kernel<2, OUT, false, false, 1>, grid, 0, st, rp);
            } else {
                if (rp.v8 == 8) launch_k(edge_reg_u8_kernel<4, OUT, false, false, 8>, grid, 0, st, rp);
                else if (rp.v8 == 4) launch_k(edge_reg_u8_kernel<4, OUT, false, false, 4>, grid, 0, st, rp);
                else launch_k(edge_reg_u8_kernel<4, OUT, false, false, 1>, grid, 0, st, rp);
            }
            return cuda_check("edge_reg_u8_kernel<UNAL>");
        }
    }
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
    const bool sides = rp.o_side[0] || rp.o_side[1] || rp.o_side[2] || rp.o_side[3];
    if (input_kind == 1 && rp.o_packed && !sides) {
        // uint8: the packed words, with or without edges / EdgeSet -- K2 stores all
    } else if (multi_out(rp)) {   // packed input only (other uint8 multi-output: K2t2 or tile)
        if (input_kind == 1) return kNoKernel;
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

// Returns kNoKernel when the register-direct kernel does not apply (caller falls back).
inline int64_t rows_total(int64_t lo, int64_t hi) { return hi - lo; }
// aligned uint8 rasters take K2t2 from this many row segments (rows x 2048-px segments)
constexpr int64_t kTma2MinSegs = 12000;
// thresholded pack (ALU-heavier: halo rows cost more, so longer strips): K2t2 from 24 000
// row segments with 12-row strips until 32-row strips make 24 warps per SM (8192^2, t = 128:
// 16.9 -> 12.3 us, 0.68 -> 0.94 of the copy peak; 12288^2 37.6 -> 27.1 us; a batch of 64
// 1920x1080 frames 33.5 -> 25.4 us; 5000x5008 stays with K2: 7.1 us against 8.6)
constexpr int kThrMidRows = 12;
constexpr int64_t kTma2MinSegsThr = 24000;
// ... and from this row width: a 2048-px segment that is >= 69 % full beats the one-shot
// K2 (batches of 1920x1080 frames: 35.6 -> 21.7 us, 0.64 -> 1.05 of the copy peak;
// 1600x1200: 16.7 -> 14.1 us).  K2 runs 32-byte rows of 768 .. 1536 px at a flat 0.79
// since its neighbour-byte fix and K2t2 at about its segment fill, so they cross at
// ~1400 px (1344: 14.4 us both; 1408: 15.0 vs 14.5; 1280: 13.6 vs 14.5).
// Rows that are not 32-byte multiples (K2 then loads 128 bits at a time, or word by
// word) move over from 1040 px: batches of 1200-px rows 89.8 -> 58.5 us (0.44 -> 0.68),
// 1250-px rows 40.4 -> 22.8 us, 1100-px rows 19.7 -> 16.7 us; 32-byte rows of 1056 px
// are faster in K2 (15.1 vs 20.1 us).  BITEDGE_TMA2_MINW overrides both.
inline int64_t tma2_min_width(bool rows32) {
    if (const char *v = knob(KN_TMA2_MINW)) return atoll(v);
    return rows32 ? 1408 : 1040;
}

// K2r (32-row rolling strips) from this many threads (BITEDGE_ROLL_MIN overrides)
inline int64_t roll_min_threads() {
    if (const char *v = knob(KN_ROLL_MIN)) return atoll(v);
    return (int64_t)sm_count() * 2048;
}

// K2t2 strip height for the 0/1 pack, from the launch's row segments T = rows x
// 2048-px segments (= warps x strip height).  Many waves of resident warps (24 per
// SM): 8 rows, the tail is short.  A few waves: the rows are cut into strips that
// fill a whole number of waves (8192^2: 4096 warps of 8-row strips are 1.15 waves of
// 3552 -- 11.3 us, 19.5 serial; 820 strips of 10 rows x 4 segments are 0.92 -- 10.9
// / 17.8 us).  Less than a wave of 8-row strips: shorter strips keep more copies in
// flight (5000x5008: 5 rows 5.7 / 11.6 us, 8 rows 8.5 / 18.1, K2 8.7 / 12.1;
// 6000x8000: 6 rows 11.9 / 15.8, 8 rows 11.5 / 18.3) -- `short_ok`: aligned rows of
// whole 2048-px segments only (4096x4100 through the UNAL ring: 5.4 us at 5 rows,
// 4.7 at 8).  scripts/u8_mid_sweep.py; BITEDGE_TMA2_RSL forces a height.
inline int tma2_strip_rows(int64_t rows, int64_t nseg, bool short_ok) {
    if (const char *v = knob(KN_TMA2_RSL)) {
        const int r = atoi(v);
        if (r >= 2 && r <= 4096) return r;
    }
    const int64_t cap = (int64_t)sm_count() * 24;
    const int64_t T = rows * nseg, w8 = (rows + 7) / 8 * nseg;
    if (w8 >= 8 * cap) return 8;
    if (w8 <= cap) return (!short_ok || T < kTma2MinSegs) ? 8 : (T < 20000 ? 5 : 6);
    const int64_t nw = w8 / cap;                         // whole waves at >= 8 rows per strip
    const int64_t max_strips = nw * cap / nseg;
    if (max_strips < 1) return 8;
    const int64_t r = (rows + max_strips - 1) / max_strips;
    return r < 8 ? 8 : (r > 64 ? 64 : (int)r);
}

// K2t2 launch for strip height RSL (4-slot rings, 8 warps per CTA); RSL = 0: the
// run-time strip height rp.rsl.
template <int RSL, bool UNAL = false>
int launch_tma2(RegParams &rp, bool multi, bool halo, int64_t nseg, cudaStream_t st) {
    constexpr int kD = 4;
    const int rsl = RSL > 0 ? RSL : rp.rsl;
    const int64_t nstrips = (rows_total(rp.row_lo, rp.row_hi) + rsl - 1) / rsl;
    const int64_t nwarps = nstrips * nseg;
    const unsigned grid = (unsigned)((nwarps + 7) / 8);
    // ring slot: 16 + 2048 + 16 bytes (+32 for UNAL: granule-aligned copies)
    const size_t smem = (size_t)8 * kD * (UNAL ? 2112 : 2080) + (size_t)8 * kD * 8;
    rp.nstrips = nstrips;
    if (UNAL && halo) return kNoKernel;
#define BE_TMA2(OUTK, H)                                                                        \
    do {                                                                                        \
        auto kern = edge_tma2_u8_kernel<RSL, kD, OUTK, H && !UNAL, UNAL>;                      \
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

// K2 UNAL: uint8 rows at any byte offset (see edge_reg_u8_kernel), 4-row strips,
// edges and / or EdgeSet, uint32 or (oswap) uint64 output words.
int try_reg_u8_unal(const void *in, int64_t in_row_bytes, uint32_t *o_edges, uint32_t *o_eset,
                    uint32_t *o_packed, int64_t out_stride_u32, const Geometry &G, int64_t nrows, int64_t row_lo,
                    int64_t row_hi, cudaStream_t st, int thr) {
    if (G.h >= ((int64_t)1 << 31)) return kNoKernel;
    RegParams rp;
    memset(&rp, 0, sizeof(rp));
    rp.in = (const char *)in; rp.in_row_bytes = in_row_bytes;
    rp.in_end = (const char *)in + (nrows - 1) * in_row_bytes + G.w;
    rp.o_edges = o_edges; rp.o_eset = o_eset; rp.out_stride = out_stride_u32;
    rp.o_packed = o_packed;
    rp.oswap = G.swap;
    rp.nrows = nrows; rp.row_lo = row_lo; rp.row_hi = row_hi;
    rp.h = (uint32_t)G.h; rp.w = G.w; rp.wp = G.wp; rp.pl = G.pl;
    rp.lastbit = G.lastbit; rp.padmask = G.padmask; rp.fillword = G.fillword;
    rp.items = G.wp;
    rp.thr = thr;
    // rows >= 2048 px: the TMA ring (K2t2) with granule-aligned copies and a
    // per-row realignment of the packed words (16384 x 16100: 45 -> 95 % of the
    // copy peak); K2 UNAL below otherwise
    if (G.w >= tma2_min_width(false) && !knob(KN_NO_TMA) && !knob(KN_NO_TMA_UNAL)) {
        const int64_t nseg = (G.w + 2047) / 2048;
        const int64_t nwarps32 = (row_hi - row_lo + 31) / 32 * nseg;
        // (no minimum work from 2048 px, unlike aligned rows: at 4096 x 4100 the ring is
        // 4.74 us against K2 UNAL's 6.46 us; narrower rows half-fill their segment and
        // need the aligned rows' minimum: 8000 x 1500 is 5.45 us here, 5.01 in K2 UNAL,
        // a batch of 64 1900 x 1080 frames 24.6 against 49.4 us)
        const bool enough = G.w >= 2048 || (row_hi - row_lo) * nseg >= kTma2MinSegs ||
                            knob(KN_FORCE_TMA);
        if (enough && (nwarps32 * 4 + 7) / 8 <= 0x7FFFFFFFLL) {
            const bool short_strips = (thr == 1 || knob(KN_TMA2_RSL8)) && !knob(KN_TMA2_RSL32);
            const bool multi = o_packed != nullptr;
            if (!short_strips) return launch_tma2<32, true>(rp, multi, false, nseg, st);
            rp.rsl = tma2_strip_rows(row_hi - row_lo, nseg, false);
            return rp.rsl == 8 ? launch_tma2<8, true>(rp, multi, false, nseg, st)
                               : launch_tma2<0, true>(rp, multi, false, nseg, st);
        }
    }
    {   // alignment of every row start (base and row stride)
        const uintptr_t a = (uintptr_t)in | (uintptr_t)in_row_bytes;
        rp.v8 = (a % 8 == 0 && !knob(KN_UNAL_BYTES)) ? 8
              : (a % 4 == 0 && !knob(KN_UNAL_BYTES)) ? 4 : 1;
    }
    // 4-row strips; 2-row strips when that leaves fewer than 2 CTAs per SM
    // (64 x 256 x 250: 128 CTAs of 4-row strips on 148 SMs)
    int rs = 4;
    if (((row_hi - row_lo + 3) / 4) * rp.items < (int64_t)sm_count() * 2 * kThreads &&
        !knob(KN_UNAL_RS4))
        rs = 2;
    rp.nstrips = (row_hi - row_lo + rs - 1) / rs;
    const int64_t grid = (rp.nstrips * rp.items + kThreads - 1) / kThreads;
    if (grid > 0x7FFFFFFFLL) return kNoKernel;
    if (o_edges && o_eset) return launch_reg_u8<kOutAny, false>(rp, rs, (unsigned)grid, st);
    if (o_eset) return launch_reg_u8<kOutEset, false>(rp, rs, (unsigned)grid, st);
    return launch_reg_u8<kOutEdges, false>(rp, rs, (unsigned)grid, st);
}

// K1f (edge_flat.cuh): packed rows with row stride == words per row that is not a
// multiple of the vector width, edges and / or EdgeSet, no halos.
template <int CW, int SWAP, int OUT>
int launch_flat_cw(const FlatParams &fp, int ru, unsigned grid, cudaStream_t st) {
#define BE_FLAT(R)                                                                    \
    if constexpr (R < CW && (!SWAP || R % 2 == 0))                                    \
        if (ru == R) {                                                                \
            launch_k(edge_flat_kernel<CW, SWAP, (R < CW ? R : 1), OUT>, grid, 0, st, fp); \
            return cuda_check("edge_flat_kernel");                                    \
        }
    BE_FLAT(1) BE_FLAT(2) BE_FLAT(3) BE_FLAT(4) BE_FLAT(5) BE_FLAT(6) BE_FLAT(7)
#undef BE_FLAT
    return kNoKernel;
}

// K1s (edge_flat.cuh): contiguous ragged packed rows staged through a per-warp
// shared-memory ring.  LR = log2(ring words per warp): 2^11 (8 KB, 3 CTAs/SM)
// while one step's window of pieces leaves >= 2 slots for prefetch, else 2^12.
template <int SWAP, int OUT, int LR>
int launch_flat_ring(const FlatRingParams &fr, unsigned grid, size_t smem, cudaStream_t st) {
    auto kern = edge_flat_ring_kernel<SWAP, OUT, LR>;
    static bool attr = false;                         // (per instantiation)
    if (!attr) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    launch_k(kern, grid, smem, st, fr);
    return cuda_check("edge_flat_ring_kernel");
}

int try_flat_ring(const void *in, uint32_t *o_edges, uint32_t *o_eset, const Geometry &G,
                  int64_t nrows, int64_t row_lo, int64_t row_hi, cudaStream_t st) {
    // opt-in (BITEDGE_RING): as fast as K1f on large ragged rasters (both at the
    // copy peak), slower on small ones (per-warp ring start-up)
    if (!knob(KN_RING) || knob(KN_NO_FLAT)) return kNoKernel;
    const int64_t S = G.wp;
    const int64_t nwords = nrows * S;
    if (row_lo != 0 || row_hi != nrows || nwords >= ((int64_t)1 << 31) - 4096 || S < 64 ||
        nwords % 4 != 0 || G.h >= ((int64_t)1 << 31))
        return kNoKernel;
    auto al = [](const void *p, int a) { return p == nullptr || ((uintptr_t)p % a) == 0; };
    if (!al(in, 16) || !al(o_edges, 8) || !al(o_eset, 8)) return kNoKernel;
    // pieces one 256-word step reads: <= ceil((2S + 259) / 256) + 1; keep >= 2
    // slots for prefetch
    const int64_t window = (2 * S + 259 + kRingSegW - 1) / kRingSegW + 1;
    int lr;
    if (window + 2 <= (1 << 11) / kRingSegW) lr = 11;
    else if (window + 2 <= (1 << 12) / kRingSegW) lr = 12;
    else return kNoKernel;
    const int warps_per_sm = lr == 11 ? 24 : 8;       // smem: 3 / 1 CTAs of 8 warps per SM
    const int64_t maxw = (int64_t)sm_count() * warps_per_sm;
    int64_t minspan = 4 * S > 1024 ? 4 * S : 1024;    // halo reads <= 2S per span
    int64_t nwarps = (nwords + minspan - 1) / minspan;
    if (nwarps > maxw) nwarps = maxw;
    if (nwarps < 1) nwarps = 1;
    int64_t span = (nwords + nwarps - 1) / nwarps;
    span = (span + 255) / 256 * 256;
    nwarps = (nwords + span - 1) / span;
    FlatRingParams fr;
    memset(&fr, 0, sizeof(fr));
    fr.in = (const uint32_t *)in;
    fr.o_edges = o_edges; fr.o_eset = o_eset;
    fr.nwords = (uint32_t)nwords; fr.S = (uint32_t)S; fr.h = (uint32_t)G.h;
    fr.pl = G.pl; fr.lastbit = G.lastbit; fr.padmask = G.padmask; fr.fillword = G.fillword;
    fr.span = (uint32_t)span; fr.nwarps = (uint32_t)nwarps;
    fr.div_s = make_fastdiv((uint32_t)S);
    fr.div_h = make_fastdiv((uint32_t)G.h);
    const int rw = 1 << lr;
    const size_t smem = (size_t)8 * rw * 4 + (size_t)8 * (rw / kRingSegW) * 8;
    const unsigned grid = (unsigned)((nwarps + 7) / 8);
    const int out = (o_edges && o_eset) ? kOutAny : o_eset ? kOutEset : kOutEdges;
#define BE_RING(SW, LRV)                                                                  \
    return out == kOutAny ? launch_flat_ring<SW, kOutAny, LRV>(fr, grid, smem, st)        \
         : out == kOutEset ? launch_flat_ring<SW, kOutEset, LRV>(fr, grid, smem, st)      \
                           : launch_flat_ring<SW, kOutEdges, LRV>(fr, grid, smem, st);
    if (G.swap) {
        if (lr == 11) { BE_RING(1, 11) } else { BE_RING(1, 12) }
    } else {
        if (lr == 11) { BE_RING(0, 11) } else { BE_RING(0, 12) }
    }
#undef BE_RING
}

int try_flat(const void *in, uint32_t *o_edges, uint32_t *o_eset, const Geometry &G,
             int64_t nrows, int64_t row_lo, int64_t row_hi, cudaStream_t st) {
    if (knob(KN_NO_FLAT)) return kNoKernel;
    const int64_t S = G.wp;                                    // uint32 words per row
    const int64_t nwords = nrows * S;
    if (row_lo != 0 || row_hi != nrows || nwords > ((int64_t)1 << 30) || S < 16 ||
        G.h >= ((int64_t)1 << 31))
        return kNoKernel;
    auto al = [](const void *p, int a) { return p == nullptr || ((uintptr_t)p % a) == 0; };
    const int cw = (al(in, 32) && al(o_edges, 32) && al(o_eset, 32)) ? 8
                 : (al(in, 16) && al(o_edges, 16) && al(o_eset, 16)) ? 4 : 0;
    if (cw == 0 || S % cw == 0) return kNoKernel;
    FlatParams fp;
    memset(&fp, 0, sizeof(fp));
    fp.in = (const uint32_t *)in;
    fp.o_edges = o_edges; fp.o_eset = o_eset;
    fp.nwords = (uint32_t)nwords; fp.S = (uint32_t)S; fp.h = (uint32_t)G.h;
    fp.nrows = (uint32_t)nrows;
    fp.pl = G.pl; fp.lastbit = G.lastbit; fp.padmask = G.padmask; fp.fillword = G.fillword;
    fp.nchunks = (uint32_t)((nwords + cw - 1) / cw);
    fp.div_s = make_fastdiv((uint32_t)S);
    fp.div_h = make_fastdiv((uint32_t)G.h);
    const int ru = (int)((cw - S % cw) % cw);
    constexpr unsigned per_cta = (kThreads / 32) * 31;        // a warp owns 31 chunks
    const unsigned grid = (fp.nchunks + per_cta - 1) / per_cta;
    const int out = (o_edges && o_eset) ? kOutAny : o_eset ? kOutEset : kOutEdges;
#define BE_FLAT_OUT(CWV, SW)                                                               \
    return out == kOutAny ? launch_flat_cw<CWV, SW, kOutAny>(fp, ru, grid, st)             \
         : out == kOutEset ? launch_flat_cw<CWV, SW, kOutEset>(fp, ru, grid, st)           \
                           : launch_flat_cw<CWV, SW, kOutEdges>(fp, ru, grid, st);
    if (cw == 8) {
        if (G.swap) { BE_FLAT_OUT(8, 1) } else { BE_FLAT_OUT(8, 0) }
    } else {
        if (G.swap) { BE_FLAT_OUT(4, 1) } else { BE_FLAT_OUT(4, 0) }
    }
#undef BE_FLAT_OUT
}

int try_reg(const void *in, int input_kind, int64_t in_row_bytes, const void *above,
            const void *below, uint32_t *o_edges, uint32_t *o_eset, uint32_t *const o_side[4],
            uint32_t *o_packed, int64_t out_stride_u32, const Geometry &G, int64_t nrows,
            int64_t row_lo, int64_t row_hi, cudaStream_t st, int thr) {
    const char *e = knob(KN_KERNEL);
    if (e && (strcmp(e, "tile") == 0 || strcmp(e, "stream") == 0)) return kNoKernel;
    auto al16 = [](const void *p) { return p == nullptr || ((uintptr_t)p % 16) == 0; };
    // packed rows that are only 4-byte aligned (not 16-byte multiples, or a
    // strided view): K1's UNAL items, without halos
    const bool unal = input_kind == 0 && (!al16(in) || in_row_bytes % 16 != 0) && !above &&
                      !below && ((uintptr_t)in % 4) == 0 && in_row_bytes % 4 == 0 &&
                      !knob(KN_NO_UNAL);
    // uint8 rows at any byte (row lengths that are not 16-byte multiples): K2's
    // UNAL strips, single-output, without halos
    const bool sides0 = o_side[0] || o_side[1] || o_side[2] || o_side[3];
    const bool u8unal = input_kind == 1 && (!al16(in) || in_row_bytes % 16 != 0) && !above &&
                        !below && !sides0 && (o_edges || o_eset || o_packed) &&
                        !knob(KN_NO_UNAL);
    if (u8unal) return try_reg_u8_unal(in, in_row_bytes, o_edges, o_eset, o_packed, out_stride_u32, G, nrows,
                                       row_lo, row_hi, st, thr);
    if (!unal && (!al16(in) || !al16(above) || !al16(below) || in_row_bytes % 16 != 0))
        return kNoKernel;
    if (G.h >= ((int64_t)1 << 31)) return kNoKernel;
    RegParams rp;
    memset(&rp, 0, sizeof(rp));
    rp.in = (const char *)in; rp.above = (const char *)above; rp.below = (const char *)below;
    rp.in_row_bytes = in_row_bytes;
    rp.o_edges = o_edges; rp.o_eset = o_eset; rp.out_stride = out_stride_u32;
    for (int k = 0; k < 4; ++k) rp.o_side[k] = o_side[k];
    rp.o_packed = o_packed;
    const bool multi = multi_out(rp);
    // uint8 -> uint64 words (the drop-in BitImage layout): K2t2 (large rasters
    // >= 1024 px wide) and K2 store the swapped halves (oswap); K2w / K2r / K2t do
    // not, and the four side outputs go to the tile kernel
    const bool u64_out = input_kind == 1 && G.swap;
    const bool u64_k2 = u64_out && (G.w < 1024 || knob(KN_NO_TMA));
    // K2 writes edges / EdgeSet plus, optionally, the packed words; nothing else
    const bool k2_outs = !sides0 && (o_edges || o_eset || o_packed);
    if (u64_k2 && !k2_outs) return kNoKernel;
    rp.oswap = u64_out ? 1 : 0;
    rp.nrows = nrows; rp.row_lo = row_lo; rp.row_hi = row_hi;
    rp.h = (uint32_t)G.h; rp.w = G.w; rp.wp = G.wp; rp.pl = G.pl;
    rp.lastbit = G.lastbit; rp.padmask = G.padmask; rp.fillword = G.fillword;
    auto al = [](const void *p, int a) { return p == nullptr || ((uintptr_t)p % a) == 0; };
    const bool in32 = al(in, 32) && in_row_bytes % 32 == 0 && al(above, 32) && al(below, 32);
    // Packed items are 8 words (256-bit loads) when rows are 32-byte aligned, else 4.
    // Small rasters (< 4 waves of 4-row strips) use 2-row strips instead, which
    // doubles the threads in flight (C3: 5.1 us serial / 88 % overlapped vs
    // 5.3 / 79 % for 4-word x 4-row items; scripts/c3sweep.sh).
    const int64_t strips4 = (row_hi - row_lo + 3) / 4;
    const bool big = strips4 * ((G.wp + 7) / 8) >= (int64_t)sm_count() * 4096;
    int cw = (input_kind == 0 && in32 && !multi && !knob(KN_CW4)) ? 8 : 4;
    // rows that are 16-byte but not 32-byte multiples: 8-word items as two 128-bit
    // loads / stores (H16) instead of 4-word items (8192 x 8000 uint64 words:
    // the per-item work over 8 words, not 4)
    const bool in16 = al16(in) && in_row_bytes % 16 == 0 && al16(above) && al16(below);
    if (input_kind == 0 && !in32 && in16 && !unal && !multi && !knob(KN_CW4) &&
        !knob(KN_NO_H16)) {
        cw = 8;
        rp.h16 = 1;
    }
    if (unal) {
        if (multi) return kNoKernel;
        // contiguous rows (stride == row length): the flat kernel's aligned vector
        // accesses instead of K1's word-by-word items
        if (in_row_bytes == (int64_t)G.wp * 4 && out_stride_u32 == G.wp) {
            int rc = try_flat_ring(in, o_edges, o_eset, G, nrows, row_lo, row_hi, st);
            if (rc != kNoKernel) return rc;
            rc = try_flat(in, o_edges, o_eset, G, nrows, row_lo, row_hi, st);
            if (rc != kNoKernel) return rc;
        }
        rp.in_end = (const char *)in + (nrows - 1) * in_row_bytes + (int64_t)G.wp * 4;
        rp.unal_words = knob(KN_UNAL_CHUNKS) == nullptr;   // words: measured faster
    }
    // (uint64 words take 2-row strips only in the tail-free and UNAL kernels)
    const bool swap2 = !G.swap || unal || rp.h16 || k1_aligned(!multi, cw, G.w);
    const int packed_rs = (input_kind == 0 && swap2 && !big) ? 2 : 4;
    if (input_kind == 0 && in32 && !multi && knob(KN_CW8)) cw = 8;
    rp.items = input_kind == 1 ? G.wp : (G.wp + cw - 1) / cw;
    rp.v8 = input_kind == 1 && in32 && G.w % 32 == 0;
    rp.thr = thr;
    const int ocw = input_kind == 1 ? 1 : rp.h16 ? 4 : cw;
    rp.vst = (out_stride_u32 % ocw == 0) && al(o_edges, 4 * ocw) && al(o_eset, 4 * ocw);
    for (int k = 0; k < 4; ++k) rp.vst = rp.vst && al(o_side[k], 4 * ocw);
    rp.vst = rp.vst && al(o_packed, 4 * ocw);
    if (input_kind == 1 && !multi && !u64_out && !above && !below && row_lo == 0 && row_hi == nrows &&
        in_row_bytes == G.w && ((uintptr_t)in % 32) == 0 && G.w % 32 == 0 && G.wp <= 32 &&
        (G.wp & (G.wp - 1)) == 0 && out_stride_u32 == G.wp && !knob(KN_NO_WARPIMG)) {
        const int lwpr = ilog2(G.wp), rpi = 32 >> lwpr;
        if (G.h % rpi == 0 && G.h / rpi <= 8) {
            const int groups = (int)(G.h / rpi);
            const int64_t nimg = G.n;
            const int64_t grid = (nimg * 32 + kThreads - 1) / kThreads;
            // K2p: the whole batch requested by TMA at kernel start, one CTA per SM
            // (up to IPW images of <= 8 KB per warp); K2w otherwise
            constexpr int kIPW = 4;
            const int64_t img_bytes = (int64_t)groups * 1024;
            const int64_t warps_needed = (nimg + kIPW - 1) / kIPW;
            const int64_t cta = (warps_needed + 7) / 8;
            const int64_t ctas = cta < sm_count() ? sm_count() : cta;
            const int64_t nwarps = ctas * 8 < nimg ? ctas * 8 : nimg;
            // barrier header (8 warps x kIPW mbarriers, 128-byte rounded) + buffers;
            // must match edge_warp_img_tma_kernel's HDR
            const size_t psmem = (size_t)((8 * kIPW * 8 + 127) / 128 * 128) +
                                 (size_t)8 * kIPW * img_bytes;
            if (knob(KN_K2P) && nimg >= 8 && psmem <= 227 * 1024 &&
                ((uintptr_t)in % 16) == 0 && nimg < ((int64_t)1 << 40)) {
                const unsigned pgrid = (unsigned)((nwarps + 7) / 8);
#define BE_K2P(L)                                                                              \
    case L: {                                                                                  \
        auto kern = o_edges && o_eset ? edge_warp_img_tma_kernel<L, kOutAny, kIPW>              \
                  : o_eset ? edge_warp_img_tma_kernel<L, kOutEset, kIPW>                       \
                           : edge_warp_img_tma_kernel<L, kOutEdges, kIPW>;                     \
        static bool attr_set = false;                                                          \
        if (!attr_set) {                                                                       \
            cudaFuncSetAttribute(edge_warp_img_tma_kernel<L, kOutAny, kIPW>,                    \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);      \
            cudaFuncSetAttribute(edge_warp_img_tma_kernel<L, kOutEset, kIPW>,                   \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);      \
            cudaFuncSetAttribute(edge_warp_img_tma_kernel<L, kOutEdges, kIPW>,                  \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);      \
            attr_set = true;                                                                   \
        }                                                                                      \
        launch_kb(kern, pgrid, (unsigned)kThreads, psmem, st, rp, groups, nimg, nwarps);       \
        return cuda_check("edge_warp_img_tma_kernel");                                         \
    }
                switch (lwpr) {
                    BE_K2P(0)
                    BE_K2P(1)
                    BE_K2P(2)
                    BE_K2P(3)
                    BE_K2P(4)
                    BE_K2P(5)
                    default: break;
                }
#undef BE_K2P
            }
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
                const bool g8 = knob(KN_WARPIMG_G4) == nullptr;
                // (Capping residency at one wave with 128-thread CTAs + 32 KB of
                // dummy smem -- 28 warps/SM, 4144 slots for 4096 images -- was
                // 20 % slower overlapped and serially: not taken.)
                const unsigned wblock = (unsigned)kThreads;
                const unsigned wgrid = (unsigned)grid;
                const size_t wsmem = 0;
                rp.pdl_late = knob(KN_PDL_LATE) != nullptr;
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
    const int64_t tma2_minw = tma2_min_width(rp.v8 != 0);
    if (input_kind == 1 && (G.w >= tma2_minw || (u64_out && !u64_k2)) && !knob(KN_NO_TMA) &&
        (!knob(KN_TMA1) || u64_out)) {
        const int64_t nseg = (G.w + 2047) / 2048;
        const int64_t nwarps32 = (rows_total(row_lo, row_hi) + 31) / 32 * nseg;
        const bool force = knob(KN_FORCE_TMA) != nullptr || (u64_out && knob(KN_U64_TMA));
        // Strip height: 8 rows for the 0/1 fast pack (4x the warps of 32-row
        // strips, so the last wave's tail is a quarter as long: C5 737 ->
        // 676 us); 32 rows when the pack is ALU-bound (threshold compare),
        // where the 25 % extra staged halo rows of 8-row strips cost more
        // than the tail (F2 on C5: 800 vs 921 us).  Sweep in DESIGN.md.
        const bool short_strips = (thr == 1 || knob(KN_TMA2_RSL8)) && !knob(KN_TMA2_RSL32);
        // Enough work to keep the ring kernels' copies in flight on every SM: 24 warps
        // per SM of 32-row strips; with the 0/1 pack's short strips, 12 000 row
        // segments (a 5000x5008 raster: 5.7 us against K2's 8.7; 8192^2: 10.9 vs 18.9 us,
        // 1.06 vs 0.61 of the copy peak; 4096^2 stays with K2: 4.8 us either way)
        int64_t min_segs = kTma2MinSegs;
        if (const char *v = knob(KN_TMA2_MIN)) min_segs = atoll(v);
        // (rows under 2048 px -- uint64 words from 1024 px -- half-fill their segments:
        // 16x1024^2 is 6.8 us here against K2's 3.6)
        const bool big32 = nwarps32 >= (int64_t)sm_count() * 24;
        if (!short_strips && !knob(KN_TMA2_MIN)) min_segs = kTma2MinSegsThr;
        const bool enough = G.w >= tma2_minw ? rows_total(row_lo, row_hi) * nseg >= min_segs
                                             : big32;
        if ((force || enough) && (nwarps32 * 4 + 7) / 8 <= 0x7FFFFFFFLL) {
            const bool halo = above || below;
            if (!short_strips) {
                // thresholded pack: 32-row strips for many waves; fewer warps than that
                // take BITEDGE_TMA2_RSL / kThrMidRows-row strips at run time
                const char *rv = knob(KN_TMA2_RSL);
                if (big32 && !rv) return launch_tma2<32>(rp, multi, halo, nseg, st);
                rp.rsl = rv ? atoi(rv) : kThrMidRows;
                if (rp.rsl < 2 || rp.rsl > 4096) rp.rsl = kThrMidRows;
                return launch_tma2<0>(rp, multi, halo, nseg, st);
            }
            rp.rsl = tma2_strip_rows(rows_total(row_lo, row_hi), nseg, G.w >= tma2_minw);
            return rp.rsl == 8 ? launch_tma2<8>(rp, multi, halo, nseg, st)
                               : launch_tma2<0>(rp, multi, halo, nseg, st);
        }
    }
    if (!k2_outs && input_kind == 1) return kNoKernel;   // other uint8 multi-output: tile kernel
    if (input_kind == 1 && !u64_out && !o_packed && G.w >= 1024 && !knob(KN_NO_TMA)) {
        // (8-row strips, as in K2t2, measured slower here at every size: 4096^2 8.3 us
        // against K2's 4.8, 8192^2 24.1 against K2t2's 11.1)
        constexpr int kRSLT = 32, kD = 6;
        const int64_t nseg = (G.w + 1023) / 1024;
        const int64_t nstrips = (rows_total(row_lo, row_hi) + kRSLT - 1) / kRSLT;
        const int64_t nwarps = nstrips * nseg;
        // Opt-in since K2 / K2r stopped stalling on their neighbour bytes (BITEDGE_TMA1
        // with enough work, or BITEDGE_FORCE_TMA at any size -- the variant tests): large
        // batches of 1024-px rows run K2r at 0.89 of the copy peak against K2t's 0.78, and
        // rows just over 1024 px half-fill K2t's second segment (128 x 1024 x 1152: 61.7
        // against K2's 32.5 us)
        const bool force = knob(KN_FORCE_TMA) != nullptr;   // tests: any size
        const bool opt_in = knob(KN_TMA1) && nwarps >= (int64_t)sm_count() * 32;
        if ((force || opt_in) && (nwarps + 7) / 8 <= 0x7FFFFFFFLL) {
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
    if (input_kind == 1 && rp.v8 && !u64_out && !o_packed && !knob(KN_NO_ROLL) &&
        (rows + kRSL - 1) / kRSL * rp.items >= roll_min_threads()) {
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
        const char *rse = knob(KN_RS);
        if (rse) rs = atoi(rse) == 8 ? 8 : 4;
    } else if (!G.swap) {
        const char *rse = knob(KN_PRS);      // packed strip height experiments: 2/4/8
        if (rse) rs = atoi(rse) == 2 ? 2 : (atoi(rse) == 8 ? 8 : 4);
    }
    if ((multi || rp.in_end || rp.h16) && rs == 8) rs = 4;   // kOutAll / UNAL / H16: 2- and 4-row strips
    if (rp.in_end && knob(KN_UNAL_RS4)) rs = 4;
    rp.nstrips = (rows + rs - 1) / rs;
    const int64_t threads = rp.nstrips * rp.items;
    const int64_t grid = (threads + kThreads - 1) / kThreads;
    if (grid > 0x7FFFFFFFLL) return kNoKernel;
    if (above || below)
        return launch_reg_halo<true>(rp, input_kind, G.swap, cw, rs, (unsigned)grid, st);
    return launch_reg_halo<false>(rp, input_kind, G.swap, cw, rs, (unsigned)grid, st);
}

// Returns kNoKernel when the streaming kernel does not apply (caller falls back).
int try_stream(const void *in, int input_kind, int64_t in_row_bytes, const void *above,
               const void *below, uint32_t *o_edges, uint32_t *o_eset, int word_bits,
               int64_t out_stride_u32, const Geometry &G, int64_t nrows, int64_t row_lo,
               int64_t row_hi, cudaStream_t st, int thr) {
    if (!stream_allowed()) return kNoKernel;
    auto al16 = [](const void *p) { return p == nullptr || ((uintptr_t)p % 16) == 0; };
    if (!al16(in) || !al16(above) || !al16(below) || in_row_bytes % 16 != 0) return kNoKernel;
    if (nrows >= ((int64_t)1 << 31)) return kNoKernel;                     // 32-bit row arithmetic
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
    if (sp.raw_pitch > stage_target / 3) return kNoKernel;                 // rows too wide to stage
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
    if (smem > 110 * 1024) return kNoKernel;
    if (input_kind == 1) return launch_stream_kind<kSU8>(sp, smem, st);
    return word_bits == 64 ? launch_stream_kind<kSP64>(sp, smem, st)
                           : launch_stream_kind<kSP32>(sp, smem, st);
}

// Shared driver of every fused-edge entry point.
int edges_impl(const void *in, int input_kind, int64_t in_stride, const void *above,
               const void *below, uint32_t *o_edges, uint32_t *o_eset, uint32_t *const o_side[4],
               uint32_t *o_packed, int word_bits, int64_t out_stride_words, int64_t n, int64_t h,
               int64_t w, int fill_bit, int64_t row_lo, int64_t row_hi, void *stream, int thr) {
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
        if (rc != kNoKernel) return rc;
        if (only_edges) {
            rc = try_stream(in, 0, in_stride * (word_bits / 8), above, below, o_edges, o_eset,
                            word_bits, tp.out_stride, G, nrows, row_lo, row_hi, st, thr);
            if (rc != kNoKernel) return rc;
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
    if (rc != kNoKernel) return rc;
    if (only_edges && word_bits == 32) {
        rc = try_stream(in, 1, in_stride, above, below, o_edges, o_eset, word_bits, tp.out_stride,
                        G, nrows, row_lo, row_hi, st, thr);
        if (rc != kNoKernel) return rc;
    }
    bool vec = (in_stride % 16) == 0 && ((uintptr_t)in % 16) == 0 &&
               (!above || ((uintptr_t)above % 16) == 0) && (!below || ((uintptr_t)below % 16) == 0);
    return vec ? launch_tile<kU8Vec>(tp, rows, st) : launch_tile<kU8Byte>(tp, rows, st);
}


// K3e: output rows 0 and rows-1 of a row slab -- the only two rows that read a
// halo -- in ONE launch (row-sharded C4: the interior rows
// [1, rows-1) run in K1 while the halo rows are in flight, then this kernel
// finishes the slab).  Thread = one uint32 word of one of the two rows; the
// up / down rows come from the slab or the halo row (NULL: the border fill,
// bitimage.py:216-223), the left / right neighbour words straight from the row
// (pixel w-1's right neighbour is the fill, bitimage.py:235-239); padding = 1.
__global__ void __launch_bounds__(256)
edge_halo_ends_kernel(const uint32_t *__restrict__ slab, const uint32_t *__restrict__ above,
                      const uint32_t *__restrict__ below, uint32_t *__restrict__ out,
                      int64_t rows, int64_t stride, int wp, int pl, uint32_t lastbit,
                      uint32_t padmask, uint32_t fw) {
    pdl_wait();
    pdl_trigger();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int nends = rows > 1 ? 2 : 1;
    if (t >= (int64_t)nends * wp) return;
    const int which = (int)(t / wp);
    const int j = (int)(t - (int64_t)which * wp);
    const int64_t r = which == 0 ? 0 : rows - 1;
    const uint32_t *row = slab + r * stride;
    const uint32_t c = row[j];
    const uint32_t lw = j > 0 ? row[j - 1] : fw;
    const uint32_t rw = j + 1 < wp ? row[j + 1] : fw;
    const uint32_t u = r > 0 ? row[j - stride] : (above ? above[j] : fw);
    const uint32_t d = r + 1 < rows ? row[j + stride] : (below ? below[j] : fw);
    const uint32_t ln = __funnelshift_r(c, lw, 1);
    uint32_t rn = __funnelshift_l(rw, c, 1);
    uint32_t f = 0u;
    if (j == pl) {
        rn = (rn & ~lastbit) | (fw & lastbit);
        f = padmask;
    }
    out[r * stride + j] = c | ~(ln | rn | u | d) | f;
}

}  // namespace capi
}  // namespace bitedge

extern "C" {

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

int be_edge_packed_halo_ends_u32(const uint32_t *slab, const uint32_t *above_or_null,
                                 const uint32_t *below_or_null, uint32_t *out, int64_t rows,
                                 int64_t w, int64_t row_stride_words, int fill_bit, void *stream) {
    Geometry G;
    int rc = make_geometry(G, 32, 1, rows, w, fill_bit);
    if (rc) return rc;
    if ((rc = check_stride(G, row_stride_words, "row"))) return rc;
    if ((rc = check_ptr(slab, 32, "slab"))) return rc;
    if ((rc = check_ptr(out, 32, "output"))) return rc;
    if ((above_or_null && ((uintptr_t)above_or_null & 3)) || (below_or_null && ((uintptr_t)below_or_null & 3)))
        return fail(BE_EALIGN, "halo rows must be 4-byte aligned");
    const int64_t total = (rows > 1 ? 2 : 1) * (int64_t)G.wp;
    launch_kb(edge_halo_ends_kernel, (unsigned)((total + 255) / 256), 256u, 0, S(stream), slab,
              above_or_null, below_or_null, out, rows, row_stride_words, G.wp, G.pl, G.lastbit,
              G.padmask, G.fillword);
    return cuda_check("edge_halo_ends_kernel");
}

int be_pack_u8(const uint8_t *in, void *out, int word_bits, int64_t n, int64_t h, int64_t w,
               int64_t in_row_stride, int64_t out_row_stride_words, void *stream) {
    uint32_t *side[4] = {nullptr, nullptr, nullptr, nullptr};
    if (out == nullptr && n != 0) return fail(BE_EINVAL, "output is NULL");
    return edges_impl(in, 1, in_row_stride, nullptr, nullptr, nullptr, nullptr, side,
                      (uint32_t *)out, word_bits, out_row_stride_words, n, h, w, 1, 0, n * h,
                      stream);
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

}  // extern "C"

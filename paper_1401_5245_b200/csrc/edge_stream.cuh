// edge_stream.cuh -- persistent, TMA-pipelined form of the fused edge kernel.
//
// Same arithmetic as edge_tile.cuh (SPEC.md:147-173 fused into one pass), but
// built for streaming at HBM speed on sm_100a:
//
//  * a persistent grid (a few CTAs per SM) walks the tiles round-robin;
//  * every tile -- rows g0-1 .. g0+R (1-row halo above and below) of a column
//    range, plus a 16-byte column halo either side -- is fetched by the Tensor
//    Memory Accelerator with `cp.async.bulk` (one instruction per staged row,
//    or one per tile when the staged rows are contiguous in HBM) into an
//    S-stage shared-memory ring whose completion is tracked by mbarrier
//    transaction counts, so the loads for tiles k+1 .. k+S-1 are in flight
//    while tile k is computed;
//  * uint8 tiles are packed 16 bytes -> 16 bits (BitImage.from_array,
//    bitimage.py:122-136) from shared memory into a packed tile first;
//  * the compute pass is the word formula of edge_tile.cuh with the border
//    fill at pixel 0 / pixel w-1 / first and last row of every image, and all
//    padding bits of the output forced to 1 (bitimage.py:101-104).
//
// Requirements (checked on the host; otherwise the tile kernel runs): input
// base and row pitch 16-byte aligned.  Like every 128-bit-vectorised path,
// the kernel may read up to the 16-byte boundary after a row's last word.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "edge_tile.cuh"

namespace bitedge {

enum StreamKind : int { kSP32 = 0, kSP64 = 1, kSU8 = 2 };

struct StreamParams {
    const char *in;          // packed words or uint8 pixels (16-B aligned)
    const char *above;       // halo row -1 (or nullptr)
    const char *below;       // halo row `nrows` (or nullptr)
    int64_t in_row_bytes;    // row pitch of `in` in bytes (multiple of 16)
    int64_t row_bytes_alloc; // bytes of a row that may be read (16-B rounded)
    uint32_t *o_edges;
    uint32_t *o_eset;
    int64_t out_stride;      // uint32 units
    int64_t nrows, h, w, row_lo, row_hi;
    int wp;                  // storage uint32 words per row
    int pl;
    uint32_t lastbit, padmask, fillword;
    int log_tq;              // tile width TQ = 1 << log_tq pixel words
    int R;                   // compute rows per tile
    int tiles_x;
    int64_t ntiles;
    int contiguous;          // staged rows copied with one bulk copy per tile
    int raw_pitch;           // bytes per staged row in shared memory (multiple of 16)
    int col0;                // byte offset of word/pixel q0 inside a staged row
    int stage_bytes;         // raw bytes per stage (multiple of 16)
    int stages;
    int pieces;              // uint8: 16-byte pieces of a staged row that lie in the row
    int thr;                 // uint8 pack threshold (1 = nonzero is white)
    int vst;                 // outputs allow 128-bit stores (16-B aligned rows)
};

// ---- PTX wrappers -----------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// TMA bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0).
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// ---- producer: stage tile t into ring slot `slot` ----------------------------

template <int KIND>
__device__ __forceinline__ void issue_tile(const StreamParams &p, int64_t t, char *stage,
                                           uint64_t *bar) {
    const int tx = (int)(t % p.tiles_x);
    const int64_t g0 = p.row_lo + (t / p.tiles_x) * (int64_t)p.R;
    const int TQ = 1 << p.log_tq;
    // staged row i <-> global row g0 - 1 + i, i in [0, R+2)
    const int64_t ga = g0 - 1 < 0 ? 0 : g0 - 1;
    const int64_t gb = g0 + p.R + 1 > p.nrows ? p.nrows : g0 + p.R + 1;     // exclusive
    // byte range of each staged row to copy, and where it lands in shared memory
    int64_t b_lo, b_hi;
    if (p.contiguous) {
        b_lo = 0;
        b_hi = p.in_row_bytes;
    } else if (KIND == kSU8) {
        b_lo = (int64_t)tx * TQ * 32 - 16;
        b_hi = (int64_t)(tx + 1) * TQ * 32 + 16;
    } else {
        b_lo = ((int64_t)tx * TQ - 4) * 4;
        b_hi = ((int64_t)(tx + 1) * TQ + 4) * 4;
    }
    const int64_t dst_off = p.col0 - (KIND == kSU8 ? (int64_t)tx * TQ * 32 : (int64_t)tx * TQ * 4);
    if (b_lo < 0) b_lo = 0;
    if (b_hi > p.row_bytes_alloc) b_hi = p.row_bytes_alloc;
    const uint32_t seg = (uint32_t)(b_hi - b_lo);
    uint32_t total = 0;
    const bool has_above = (g0 == 0 && p.above != nullptr);
    const bool has_below = (g0 + p.R >= p.nrows && p.below != nullptr);
    if (p.contiguous) total += (uint32_t)((gb - ga) * p.in_row_bytes);
    else total += (uint32_t)(gb - ga) * seg;
    if (has_above) total += seg;
    if (has_below) total += seg;
    mbar_expect_tx(bar, total);
    if (p.contiguous) {
        tma_load_1d(stage + (ga - (g0 - 1)) * p.raw_pitch, p.in + ga * p.in_row_bytes,
                    (uint32_t)((gb - ga) * p.in_row_bytes), bar);
    } else {
        for (int64_t g = ga; g < gb; ++g)
            tma_load_1d(stage + (g - (g0 - 1)) * p.raw_pitch + dst_off + b_lo,
                        p.in + g * p.in_row_bytes + b_lo, seg, bar);
    }
    if (has_above) tma_load_1d(stage + dst_off + b_lo, p.above + b_lo, seg, bar);
    if (has_below) {
        // global row nrows lands at staged row nrows - (g0 - 1) (R+1 for a full tile)
        const int64_t bi = p.nrows - (g0 - 1);
        tma_load_1d(stage + bi * p.raw_pitch + dst_off + b_lo, p.below + b_lo, seg, bar);
    }
}

// ---- consumer ----------------------------------------------------------------

// Row-position tracker: y = global row mod h, advanced without divisions.
struct RowPos {
    uint32_t y, h, step;       // step = row increment mod h
    __device__ __forceinline__ void advance() {
        y += step;
        if (y >= h) y -= h;
    }
};

template <int SWAP>
__device__ __forceinline__ uint4 to_pixel_order(uint4 v) {
    return SWAP ? make_uint4(v.y, v.x, v.w, v.z) : v;
}

__device__ __forceinline__ void tail_fix(int pw, const StreamParams &p, uint32_t fw, uint32_t &rn,
                                         uint32_t &force) {
    if (pw == p.pl) {
        rn = (rn & ~p.lastbit) | (fw & p.lastbit);
        force = p.padmask;
    } else if (pw > p.pl) {
        force = 0xFFFFFFFFu;
    }
}

template <int OUT>
__device__ __forceinline__ void emit(uint32_t *e, uint32_t *s, int64_t o, uint32_t v_edges,
                                     uint32_t v_eset) {
    if (OUT == kOutEdges) __stcs(e + o, v_edges);
    else if (OUT == kOutEset) __stcs(s + o, v_eset);
    else {
        __stcs(e + o, v_edges);
        __stcs(s + o, v_eset);
    }
}

template <int KIND, int OUT>
__global__ void __launch_bounds__(kThreads, 2)
edge_stream_kernel(const StreamParams p) {
    extern __shared__ __align__(128) char sm[];
    constexpr bool U8 = (KIND == kSU8);
    constexpr int SWAP = (KIND == kSP64) ? 1 : 0;
    const int S = p.stages;
    const int log_tq = p.log_tq;
    const int TQ = 1 << log_tq;
    const int R = p.R;
    char *ring = sm;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + (size_t)S * p.stage_bytes);
    // packed tile for uint8 input: (R+2) rows x (TQ+8) words, interior at column 4
    uint32_t *pk = reinterpret_cast<uint32_t *>(bars + S);
    const int PP = TQ + 8;
    const int tid = threadIdx.x;
    const Thr T = make_thr(p.thr);

    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_barrier_init();
    }
    __syncthreads();

    const int64_t first = blockIdx.x, step = gridDim.x;
    if (tid == 0) {
        for (int s = 0; s < S - 1; ++s) {
            const int64_t t = first + s * step;
            if (t < p.ntiles) issue_tile<KIND>(p, t, ring + (size_t)s * p.stage_bytes, &bars[s]);
        }
    }

    const uint32_t fw = p.fillword;
    const uint32_t h32 = (uint32_t)p.h;
    // Rows of a tile are processed as 4-word chunks (TQ >= 16) or single words.
    const bool vec = TQ >= 16;
    const int log_c = vec ? log_tq - 2 : log_tq;     // column items per tile row
    const int citem = tid & ((1 << log_c) - 1);
    const int rg = tid >> log_c;                     // row group
    const int NG = kThreads >> log_c;
    // blocked rows for chunks (vertical reuse), interleaved rows for words (coalescing)
    const int rr = vec ? (R + NG - 1) / NG : 1;
    const int r_begin = vec ? rg * rr : rg;
    const int r_stride = vec ? 1 : NG;
    const uint32_t step_mod = (uint32_t)((int64_t)r_stride % p.h);

    int k = 0;
    for (int64_t t = first; t < p.ntiles; t += step, ++k) {
        const int slot = k % S;
        if (tid == 0) {
            const int64_t tn = t + (int64_t)(S - 1) * step;
            const int sn = (k + S - 1) % S;
            if (tn < p.ntiles) issue_tile<KIND>(p, tn, ring + (size_t)sn * p.stage_bytes, &bars[sn]);
        }
        const int tx = (int)(t % p.tiles_x);
        const int64_t g0 = p.row_lo + (t / p.tiles_x) * (int64_t)R;
        const int q0 = tx * TQ;
        mbar_wait(&bars[slot], (uint32_t)((k / S) & 1));
        const char *st = ring + (size_t)slot * p.stage_bytes;

        if (U8) {
            // pack staged rows 0..R+1: one 32-pixel word per item (2 x 16-byte smem reads)
            const int total = (R + 2) << log_tq;
            for (int idx = tid; idx < total; idx += kThreads) {
                const int i = idx >> log_tq, jw = idx & (TQ - 1);
                uint32_t word = 0xFFFFFFFFu;               // words past the staged row
                if (2 * jw < p.pieces) {
                    const char *src = st + i * p.raw_pitch + p.col0 + 32 * jw;
                    const uint32_t hi = pack16(*reinterpret_cast<const uint4 *>(src), T);
                    const uint32_t lo = 2 * jw + 1 < p.pieces
                                            ? pack16(*reinterpret_cast<const uint4 *>(src + 16), T)
                                            : 0xFFFFu;
                    word = (hi << 16) | lo;
                }
                pk[i * PP + 4 + jw] = word;
            }
            if (p.tiles_x > 1) {   // column halo pieces (the pixels next to the tile)
                for (int idx = tid; idx < 2 * (R + 2); idx += kThreads) {
                    const int i = idx >> 1, right = idx & 1;
                    const uint32_t half = pack16(*reinterpret_cast<const uint4 *>(
                        st + i * p.raw_pitch + p.col0 + (right ? 32 * TQ : -16)), T);
                    pk[i * PP + (right ? TQ + 4 : 3)] = right ? (half << 16) : half;
                }
            }
            __syncthreads();
        }

        // word source: w(i, jj) = wb[i * pitch + jj] (memory order), i = staged row
        const uint32_t *wb;
        int pitch;
        if (U8) {
            wb = pk + 4;
            pitch = PP;
        } else {
            wb = reinterpret_cast<const uint32_t *>(st + p.col0);
            pitch = p.raw_pitch >> 2;
        }
        const int rmax = (int)min((int64_t)R, p.row_hi - g0);
        const int r1 = vec ? min(rmax, r_begin + rr) : rmax;
        const bool no_top_fill = p.above != nullptr, no_bot_fill = p.below != nullptr;
        if (vec) {
            const int j4 = 4 * citem;
            const int pw4 = q0 + j4;
            if (pw4 < p.wp && r_begin < r1) {
                const bool first_chunk = (pw4 == 0);
                const bool tail = (pw4 + 3 >= p.pl);
                const int nst = min(4, p.wp - pw4);          // words of the chunk in the row
                RowPos rp{(uint32_t)(g0 + r_begin) % h32, h32, step_mod};
                const uint32_t *s = wb + (r_begin + 1) * pitch + j4;
                uint4 up = to_pixel_order<SWAP>(*reinterpret_cast<const uint4 *>(s - pitch));
                uint4 cur = to_pixel_order<SWAP>(*reinterpret_cast<const uint4 *>(s));
                int64_t o = (g0 + r_begin) * p.out_stride + pw4;
                for (int r = r_begin; r < r1; ++r, s += pitch, o += p.out_stride) {
                    uint4 dn = to_pixel_order<SWAP>(*reinterpret_cast<const uint4 *>(s + pitch));
                    const uint32_t lw = first_chunk ? fw : s[SWAP ? -2 : -1];
                    const uint32_t rw = s[SWAP ? 5 : 4];
                    uint4 u = up, d = dn;
                    if (rp.y == 0 && !no_top_fill) u = make_uint4(fw, fw, fw, fw);
                    if (rp.y == h32 - 1 && !no_bot_fill) d = make_uint4(fw, fw, fw, fw);
                    uint32_t rn0 = __funnelshift_l(cur.y, cur.x, 1);
                    uint32_t rn1 = __funnelshift_l(cur.z, cur.y, 1);
                    uint32_t rn2 = __funnelshift_l(cur.w, cur.z, 1);
                    uint32_t rn3 = __funnelshift_l(rw, cur.w, 1);
                    const uint32_t ln0 = __funnelshift_r(cur.x, lw, 1);
                    const uint32_t ln1 = __funnelshift_r(cur.y, cur.x, 1);
                    const uint32_t ln2 = __funnelshift_r(cur.z, cur.y, 1);
                    const uint32_t ln3 = __funnelshift_r(cur.w, cur.z, 1);
                    uint32_t f0 = 0, f1 = 0, f2 = 0, f3 = 0;
                    if (tail) {
                        // pixel w-1 reads the fill (bitimage.py:234-239); padding forced to 1
                        tail_fix(pw4 + 0, p, fw, rn0, f0);
                        tail_fix(pw4 + 1, p, fw, rn1, f1);
                        tail_fix(pw4 + 2, p, fw, rn2, f2);
                        tail_fix(pw4 + 3, p, fw, rn3, f3);
                    }
                    const uint32_t a0 = ln0 | rn0 | u.x | d.x, a1 = ln1 | rn1 | u.y | d.y;
                    const uint32_t a2 = ln2 | rn2 | u.z | d.z, a3 = ln3 | rn3 | u.w | d.w;
                    uint4 ve = make_uint4(cur.x | ~a0 | f0, cur.y | ~a1 | f1, cur.z | ~a2 | f2,
                                          cur.w | ~a3 | f3);
                    uint4 vs = make_uint4((~cur.x & a0) | f0, (~cur.y & a1) | f1,
                                          (~cur.z & a2) | f2, (~cur.w & a3) | f3);
                    ve = to_pixel_order<SWAP>(ve);
                    vs = to_pixel_order<SWAP>(vs);
                    if (nst == 4 && p.vst) {
                        if (OUT != kOutEset) __stcs(reinterpret_cast<uint4 *>(p.o_edges + o), ve);
                        if (OUT != kOutEdges) __stcs(reinterpret_cast<uint4 *>(p.o_eset + o), vs);
                    } else {
                        const uint32_t e4[4] = {ve.x, ve.y, ve.z, ve.w};
                        const uint32_t s4[4] = {vs.x, vs.y, vs.z, vs.w};
                        for (int q = 0; q < nst; ++q) {
                            if (OUT != kOutEset) p.o_edges[o + q] = e4[q];
                            if (OUT != kOutEdges) p.o_eset[o + q] = s4[q];
                        }
                    }
                    up = cur;
                    cur = dn;
                    rp.advance();
                }
            }
        } else {
            const int j = citem;
            const int pw = q0 + j;
            if (pw < p.wp && r_begin < rmax) {
                const bool first_col = (pw == 0);
                uint32_t keep = 0xFFFFFFFFu, fixb = 0u, force = 0u;
                if (pw == p.pl) {
                    keep = ~p.lastbit;
                    fixb = fw & p.lastbit;
                    force = p.padmask;
                } else if (pw > p.pl) {
                    force = 0xFFFFFFFFu;
                }
                const int jc = j ^ SWAP, jl = (j - 1) ^ SWAP, jr = (j + 1) ^ SWAP;
                RowPos rp{(uint32_t)(g0 + r_begin) % h32, h32, step_mod};
                const int64_t ostep = (int64_t)NG * p.out_stride;
                int64_t o = (g0 + r_begin) * p.out_stride + (pw ^ SWAP);
                const uint32_t *s = wb + (r_begin + 1) * pitch;
                for (int r = r_begin; r < rmax; r += NG, s += NG * pitch, o += ostep) {
                    const uint32_t cc = s[jc];
                    const uint32_t u = (rp.y == 0 && !no_top_fill) ? fw : s[-pitch + jc];
                    const uint32_t d = (rp.y == h32 - 1 && !no_bot_fill) ? fw : s[pitch + jc];
                    const uint32_t l = first_col ? fw : s[jl];
                    const uint32_t ln = __funnelshift_r(cc, l, 1);
                    const uint32_t rn = (__funnelshift_l(s[jr], cc, 1) & keep) | fixb;
                    const uint32_t any = ln | rn | u | d;
                    emit<OUT>(p.o_edges, p.o_eset, o, cc | ~any | force, (~cc & any) | force);
                    rp.advance();
                }
            }
        }
        __syncthreads();   // ring slot and packed tile are free again
    }
}

}  // namespace bitedge

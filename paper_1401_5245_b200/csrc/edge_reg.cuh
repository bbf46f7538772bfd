// edge_reg.cuh -- register-direct streaming form of the fused edge kernel
// (the default path for 16-byte-aligned rasters; K1 packed, K2 uint8).
//
// No shared memory and no barriers: every thread owns a column item of a
// strip of RS rows and
//   1. issues all RS+2 row loads of its item at once (the strip plus a 1-row
//      halo above and below; 128-bit loads, L1 no-allocate), so each thread
//      keeps (RS+2) x 16..32 bytes in flight;
//   2. walks the strip with up / centre / down already in registers; the
//      horizontal neighbour words come from the adjacent lanes by warp
//      shuffle (`shfl.up` / `shfl.down`), with one extra scalar load only for
//      a warp's first/last lane when its neighbour item lives in another warp;
//   3. writes each output word once (128-bit streaming stores for K1).
// The arithmetic per word is the single-pass form of SPEC.md:147-173:
//     edges = c | ~(Ln | Rn | Un | Dn),  Ln/Rn = funnel shifts by one pixel
// with the fill at pixel 0, at pixel w-1 (bitimage.py:234-239) and at the
// first/last row of every image (bitimage.py:216-223), padding forced to 1.
//
// K1 item = 4 pixel-order uint32 words (one 128-bit load per row);
// K2 item = 1 output word = 32 uint8 pixels (two 128-bit loads per row,
// packed in registers: BitImage.from_array, bitimage.py:122-136).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "edge_tile.cuh"

namespace bitedge {

struct RegParams {
    const char *in;          // 16-B aligned
    const char *above;       // halo row -1 (16-B aligned) or nullptr
    const char *below;       // halo row nrows or nullptr
    int64_t in_row_bytes;    // multiple of 16
    uint32_t *o_edges;
    uint32_t *o_eset;
    int64_t out_stride;      // uint32 units
    int64_t nrows, row_lo, row_hi;
    uint32_t h;              // rows per image (< 2^31)
    int64_t w;
    int wp;                  // storage uint32 words per row
    int pl;
    uint32_t lastbit, padmask, fillword;
    int items;               // column items per row (K1: ceil(wp/4) chunks; K2: words)
    int64_t nstrips;
    int vst;                 // 128-bit output stores allowed
    int v8;                  // uint8 rows are 32-B aligned: 256-bit loads
};

template <int SWAP>
__device__ __forceinline__ uint4 pix_order(uint4 v) {
    return SWAP ? make_uint4(v.y, v.x, v.w, v.z) : v;
}

__device__ __forceinline__ void fix_tail(int pw, const RegParams &p, uint32_t &rn, uint32_t &force) {
    if (pw == p.pl) {
        rn = (rn & ~p.lastbit) | (p.fillword & p.lastbit);
        force = p.padmask;
    } else if (pw > p.pl) {
        force = 0xFFFFFFFFu;
    }
}

// ---------------------------------------------------------------- K1: packed words

// Load CW (4 or 8) consecutive uint32 words with one 128/256-bit load.
template <int CW>
__device__ __forceinline__ void load_chunk(const char *p, uint32_t (&v)[CW]) {
    if (CW == 8) {
        asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                       "=r"(v[6]), "=r"(v[7])
                     : "l"(p));
    } else {
        uint4 q = ldg_stream_v4(p);
        v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    }
}

template <int CW>
__device__ __forceinline__ void store_chunk(uint32_t *p, const uint32_t (&v)[CW]) {
    if (CW == 8) {
        asm volatile("st.global.cs.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]),
                     "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                     : "memory");
    } else {
        __stcs(reinterpret_cast<uint4 *>(p), make_uint4(v[0], v[1], v[2], v[3]));
    }
}

// Item = CW pixel words of one row (memory order == pixel order for uint32 rows;
// uint64 rows swap the halves of each word pair).  RS rows per strip.
template <int SWAP, int RS, int CW, int OUT, bool HALO>
__global__ void __launch_bounds__(kThreads)
edge_reg_packed_kernel(const RegParams p) {
    pdl_wait();
    pdl_trigger();
    const int64_t t = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int64_t strip = t / p.items;
    const int c = (int)(t - strip * p.items);
    const bool live = strip < p.nstrips;
    const int64_t g0 = p.row_lo + strip * RS;
    const int pw0 = CW * c;
    const uint32_t fw = p.fillword;
    const int64_t rb = p.in_row_bytes;

    // ---- issue every load of the strip up front; staged row i = global row g0-1+i
    const char *base = p.in + (g0 - 1) * rb + 4 * pw0;
    const int i_lo = g0 == 0 ? 1 : 0;
    const int64_t lim = p.nrows - (g0 - 1);                 // rows i < lim exist
    const bool need_l = live && c > 0 && lane == 0;
    const bool need_r = live && c + 1 < p.items && lane == 31;
    uint32_t v[RS + 2][CW];
    uint32_t lwx[RS], rwx[RS];
#pragma unroll
    for (int i = 0; i < RS + 2; ++i) {
        const char *ptr = base + i * rb;
        bool ok = live && i >= i_lo && i < lim;
        if (HALO) {
            if (i == 0 && g0 == 0 && p.above) { ptr = p.above + 4 * pw0; ok = live; }
            if (i == lim && p.below) { ptr = p.below + 4 * pw0; ok = live; }
        }
        if (ok) {
            load_chunk<CW>(ptr, v[i]);
        } else {
#pragma unroll
            for (int q = 0; q < CW; ++q) v[i][q] = fw;
        }
        if (i >= 1 && i <= RS) {
            lwx[i - 1] = fw;
            rwx[i - 1] = 0u;
            if (ok && need_l) lwx[i - 1] = __ldg((const uint32_t *)ptr + (SWAP ? -2 : -1));
            if (ok && need_r) rwx[i - 1] = __ldg((const uint32_t *)ptr + (SWAP ? CW + 1 : CW));
        }
    }

    const bool tail = pw0 + CW - 1 >= p.pl;
    const int nst = min(CW, p.wp - pw0);
    uint32_t y = live ? (uint32_t)(g0 % p.h) : 0u;
    int64_t o = g0 * p.out_stride + pw0;
#pragma unroll
    for (int r = 0; r < RS; ++r) {
        // pixel-order views of up / centre / down
        uint32_t cu[CW], cc[CW], cd[CW];
#pragma unroll
        for (int q = 0; q < CW; ++q) {
            cu[q] = v[r][q ^ SWAP];
            cc[q] = v[r + 1][q ^ SWAP];
            cd[q] = v[r + 2][q ^ SWAP];
        }
        uint32_t lw = __shfl_up_sync(0xFFFFFFFFu, cc[CW - 1], 1);
        uint32_t rw = __shfl_down_sync(0xFFFFFFFFu, cc[0], 1);
        if (lane == 0) lw = lwx[r];
        if (lane == 31) rw = rwx[r];
        if (c == 0) lw = fw;
        const int64_t g = g0 + r;
        if (live && g < p.row_hi) {
            const bool top = (y == 0) && !(HALO && p.above);
            const bool bot = (y == p.h - 1) && !(HALO && p.below);
            uint32_t ve[CW], vs[CW];
#pragma unroll
            for (int q = 0; q < CW; ++q) {
                const uint32_t left = q == 0 ? lw : cc[q - 1];
                const uint32_t right = q == CW - 1 ? rw : cc[q + 1];
                const uint32_t ln = __funnelshift_r(cc[q], left, 1);
                uint32_t rn = __funnelshift_l(right, cc[q], 1);
                uint32_t f = 0u;
                if (tail) fix_tail(pw0 + q, p, rn, f);
                const uint32_t u = top ? fw : cu[q];
                const uint32_t d = bot ? fw : cd[q];
                const uint32_t a = ln | rn | u | d;
                ve[q ^ SWAP] = cc[q] | ~a | f;
                vs[q ^ SWAP] = (~cc[q] & a) | f;
            }
            if (nst == CW && p.vst) {
                if (OUT != kOutEset) store_chunk<CW>(p.o_edges + o, ve);
                if (OUT != kOutEdges) store_chunk<CW>(p.o_eset + o, vs);
            } else {
                for (int q = 0; q < nst; ++q) {
                    if (OUT != kOutEset) p.o_edges[o + q] = ve[q];
                    if (OUT != kOutEdges) p.o_eset[o + q] = vs[q];
                }
            }
        }
        o += p.out_stride;
        if (++y == p.h) y = 0;
    }
}

// ---------------------------------------------------------------- K2: uint8 pixels

// 32 bytes -> one MSB-first word (pixels x0 .. x0+31); bytes beyond the row are garbage
// and only ever land in padding bits.
__device__ __forceinline__ uint32_t pack32(uint4 a, uint4 b) {
    return (pack16(a) << 16) | pack16(b);
}

// One 256-bit load (sm_100: LDG.E.256), 32-byte aligned, L1 no-allocate.
__device__ __forceinline__ void ldg_stream_v8(const void *p, uint4 &a, uint4 &b) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z),
                   "=r"(b.w)
                 : "l"(p));
}

// K2w: small glyph-like images (BASELINE config C2: 64 x 64).  One warp per
// image: with 2^LWPR words (32 * 2^LWPR pixels) per row, one 256-bit load per
// lane covers RPI = 32 >> LWPR whole rows (1 KB per warp instruction, fully
// coalesced), lane L holding word L % WPR of row L / WPR of that row group.
// Up/down neighbours come from lane -/+ WPR (or the adjacent row group's
// register), left/right from lane -/+ 1; no halo rows are loaded because an
// image's outer neighbours are the border fill.  Requires w == 32 * WPR,
// contiguous rows, h == G * RPI with G <= 8.
template <int LWPR, int OUT>
__global__ void __launch_bounds__(kThreads)
edge_warp_img_kernel(const RegParams p, int G, int64_t nimg) {
    pdl_wait();
    pdl_trigger();
    constexpr int WPR = 1 << LWPR;
    constexpr int RPI = 32 >> LWPR;
    const int64_t img = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
    if (img >= nimg) return;                      // whole warps exit together
    const int lane = threadIdx.x & 31;
    const int rl = lane >> LWPR, wi = lane & (WPR - 1);
    const uint32_t fw = p.fillword;
    const char *src = p.in + img * (int64_t)G * 1024 + 32 * lane;
    uint4 a[8], b[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (k < G) ldg_stream_v8(src + 1024 * k, a[k], b[k]);
    uint32_t wd[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) wd[k] = k < G ? pack32(a[k], b[k]) : 0xFFFFFFFFu;

    uint32_t *oe = p.o_edges + img * (int64_t)G * 32 + lane;
    uint32_t *os = p.o_eset + img * (int64_t)G * 32 + lane;
    const bool last_word = (wi == WPR - 1);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        if (k >= G) break;
        const uint32_t cw = wd[k];
        // rows above / below inside this row group, and across the group boundary
        const uint32_t up_in = __shfl_up_sync(0xFFFFFFFFu, cw, WPR);
        const uint32_t dn_in = __shfl_down_sync(0xFFFFFFFFu, cw, WPR);
        const uint32_t up_x = __shfl_sync(0xFFFFFFFFu, k > 0 ? wd[k > 0 ? k - 1 : 0] : fw,
                                          (lane + 32 - WPR) & 31);
        const uint32_t dn_x = __shfl_sync(0xFFFFFFFFu, k + 1 < G ? wd[k + 1 < 8 ? k + 1 : 7] : fw,
                                          (lane + WPR) & 31);
        const uint32_t u = rl > 0 ? up_in : (k > 0 ? up_x : fw);
        const uint32_t d = rl < RPI - 1 ? dn_in : (k + 1 < G ? dn_x : fw);
        uint32_t lw = __shfl_up_sync(0xFFFFFFFFu, cw, 1);
        const uint32_t rw = __shfl_down_sync(0xFFFFFFFFu, cw, 1);
        if (wi == 0) lw = fw;
        const uint32_t ln = __funnelshift_r(cw, lw, 1);
        uint32_t rn = __funnelshift_l(rw, cw, 1);
        if (last_word) rn = (rn & ~1u) | (fw & 1u);   // pixel w-1 reads the fill
        const uint32_t any = ln | rn | u | d;
        if (OUT != kOutEset) __stcs(oe + 32 * k, cw | ~any);
        if (OUT != kOutEdges) __stcs(os + 32 * k, ~cw & any);
    }
}

template <int RS, int OUT, bool HALO, bool V8>
__global__ void __launch_bounds__(kThreads)
edge_reg_u8_kernel(const RegParams p) {
    pdl_wait();
    pdl_trigger();
    const int64_t t = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int64_t strip = t / p.items;
    const int c = (int)(t - strip * p.items);          // output word of the row
    const bool live = strip < p.nstrips;
    const int64_t g0 = p.row_lo + strip * RS;
    const uint32_t fw = p.fillword;
    const int64_t x0 = 32 * (int64_t)c;
    const int64_t rb = p.in_row_bytes;
    // second 16-byte piece inside the 16-B-rounded row?
    const bool has_hi = x0 + 16 < ((p.w + 15) & ~(int64_t)15);
    const bool need_l = live && c > 0 && lane == 0;
    const bool need_r = live && c + 1 < p.items && lane == 31;

    const char *base = p.in + (g0 - 1) * rb + x0;
    const int i_lo = g0 == 0 ? 1 : 0;
    const int64_t lim = p.nrows - (g0 - 1);
    uint32_t wd[RS + 2];
    uint32_t lbit[RS], rbit[RS];
    {
        uint4 ra[RS + 2], rb2[RS + 2];
#pragma unroll
        for (int i = 0; i < RS + 2; ++i) {
            const char *ptr = base + i * rb;
            bool ok = live && i >= i_lo && i < lim;
            if (HALO) {
                if (i == 0 && g0 == 0 && p.above) { ptr = p.above + x0; ok = live; }
                if (i == lim && p.below) { ptr = p.below + x0; ok = live; }
            }
            ra[i] = make_uint4(~0u, ~0u, ~0u, ~0u);
            rb2[i] = ra[i];
            if (ok) {
                if (V8) {
                    ldg_stream_v8(ptr, ra[i], rb2[i]);
                } else {
                    ra[i] = ldg_stream_v4(ptr);
                    if (has_hi) rb2[i] = ldg_stream_v4(ptr + 16);
                }
            }
            if (i >= 1 && i <= RS) {
                lbit[i - 1] = fw;
                rbit[i - 1] = 0u;
                if (ok && need_l) lbit[i - 1] = ptr[-1] != 0 ? 1u : 0u;
                if (ok && need_r) rbit[i - 1] = ptr[32] != 0 ? 0x80000000u : 0u;
            }
        }
#pragma unroll
        for (int i = 0; i < RS + 2; ++i) wd[i] = pack32(ra[i], rb2[i]);
    }

    uint32_t keep = 0xFFFFFFFFu, fixb = 0u, force = 0u;
    if (c == p.pl) {                 // pixel w-1 reads the fill; padding forced to 1
        keep = ~p.lastbit;
        fixb = fw & p.lastbit;
        force = p.padmask;
    } else if (c > p.pl) {
        force = 0xFFFFFFFFu;
    }
    uint32_t y = live ? (uint32_t)(g0 % p.h) : 0u;
    int64_t o = g0 * p.out_stride + c;
#pragma unroll
    for (int r = 0; r < RS; ++r) {
        const uint32_t cw = wd[r + 1];
        uint32_t lw = __shfl_up_sync(0xFFFFFFFFu, cw, 1);
        uint32_t rw = __shfl_down_sync(0xFFFFFFFFu, cw, 1);
        if (lane == 0) lw = lbit[r];
        if (lane == 31) rw = rbit[r];
        if (c == 0) lw = fw;
        const int64_t g = g0 + r;
        if (live && g < p.row_hi) {
            const uint32_t u = (y == 0 && !(HALO && p.above)) ? fw : wd[r];
            const uint32_t d = (y == p.h - 1 && !(HALO && p.below)) ? fw : wd[r + 2];
            const uint32_t ln = __funnelshift_r(cw, lw, 1);
            const uint32_t rn = (__funnelshift_l(rw, cw, 1) & keep) | fixb;
            const uint32_t any = ln | rn | u | d;
            if (OUT != kOutEset) __stcs(p.o_edges + o, cw | ~any | force);
            if (OUT != kOutEdges) __stcs(p.o_eset + o, (~cw & any) | force);
        }
        o += p.out_stride;
        if (++y == p.h) y = 0;
    }
}

// K2r: uint8 pixels, long strips with a rolling register window.  A thread
// owns one output word (32 pixels) of RSL consecutive rows and keeps the next
// 2-3 rows' 256-bit loads in flight while it packs and emits the current
// one, so the 2 halo rows cost 2/RSL instead of 2/RS (the one-shot K2's
// dominant overhead on big pages, BASELINE config C5).  Ring of Q = 4 raw
// slots; the loop is unrolled by Q so every slot index is static.
template <int RSL, int OUT, bool HALO>
__global__ void __launch_bounds__(kThreads)
edge_roll_u8_kernel(const RegParams p) {
    pdl_wait();
    pdl_trigger();
    constexpr int Q = 4;
    static_assert(RSL % Q == 0, "strip must be a multiple of the ring");
    const int64_t t = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int64_t strip = t / p.items;
    const int c = (int)(t - strip * p.items);
    const bool live = strip < p.nstrips;
    const int64_t g0 = p.row_lo + strip * RSL;
    const uint32_t fw = p.fillword;
    const int64_t x0 = 32 * (int64_t)c;
    const int64_t rb = p.in_row_bytes;
    const bool need_l = live && c > 0 && lane == 0;
    const bool need_r = live && c + 1 < p.items && lane == 31;
    const char *base = p.in + (g0 - 1) * rb + x0;
    const int i_lo = g0 == 0 ? 1 : 0;
    const int64_t lim = p.nrows - (g0 - 1);            // staged rows i < lim exist

    // staged row i (global g0-1+i), i in [0, RSL+2): raw 32 bytes + edge bits
    uint4 ra[Q], rb2[Q];
    uint32_t lb[Q], rbt[Q];
    auto issue = [&](int i, int slot) {
        const char *ptr = base + i * rb;
        bool ok = live && i >= i_lo && i < lim && i < RSL + 2;
        if (HALO) {
            if (i == 0 && g0 == 0 && p.above) { ptr = p.above + x0; ok = live; }
            if (i == lim && i < RSL + 2 && p.below) { ptr = p.below + x0; ok = live; }
        }
        ra[slot] = make_uint4(~0u, ~0u, ~0u, ~0u);
        rb2[slot] = ra[slot];
        lb[slot] = fw;
        rbt[slot] = 0u;
        if (ok) {
            ldg_stream_v8(ptr, ra[slot], rb2[slot]);
            if (need_l) lb[slot] = ptr[-1] != 0 ? 1u : 0u;
            if (need_r) rbt[slot] = ptr[32] != 0 ? 0x80000000u : 0u;
        }
    };

    uint32_t keep = 0xFFFFFFFFu, fixb = 0u, force = 0u;
    if (c == p.pl) {
        keep = ~p.lastbit;
        fixb = fw & p.lastbit;
        force = p.padmask;
    } else if (c > p.pl) {
        force = 0xFFFFFFFFu;
    }
    uint32_t y = live ? (uint32_t)(g0 % p.h) : 0u;
    int64_t o = g0 * p.out_stride + c;

    // prologue: staged rows 0 (halo above) .. 3 in flight; pack rows 0 and 1
    issue(0, 0);
    issue(1, 1);
    issue(2, 2);
    issue(3, 3);
    uint32_t w_up = pack32(ra[0], rb2[0]);
    uint32_t w_c = pack32(ra[1], rb2[1]);
    uint32_t lb_c = lb[1], rb_c = rbt[1];
    for (int r0 = 0; r0 < RSL; r0 += Q) {
#pragma unroll
        for (int k = 0; k < Q; ++k) {
            const int r = r0 + k;                      // output row; staged row r+1 is centre
            issue(r + 4, k);                           // rows r+2 .. r+4 stay in flight
            const int sd = (k + 2) % Q;                // staged row r+2 = down neighbour
            const uint32_t w_d = pack32(ra[sd], rb2[sd]);
            uint32_t lw = __shfl_up_sync(0xFFFFFFFFu, w_c, 1);
            uint32_t rw = __shfl_down_sync(0xFFFFFFFFu, w_c, 1);
            if (lane == 0) lw = lb_c;
            if (lane == 31) rw = rb_c;
            if (c == 0) lw = fw;
            const int64_t g = g0 + r;
            if (live && g < p.row_hi) {
                const uint32_t u = (y == 0 && !(HALO && p.above)) ? fw : w_up;
                const uint32_t d = (y == p.h - 1 && !(HALO && p.below)) ? fw : w_d;
                const uint32_t ln = __funnelshift_r(w_c, lw, 1);
                const uint32_t rn = (__funnelshift_l(rw, w_c, 1) & keep) | fixb;
                const uint32_t any = ln | rn | u | d;
                if (OUT != kOutEset) __stcs(p.o_edges + o, w_c | ~any | force);
                if (OUT != kOutEdges) __stcs(p.o_eset + o, (~w_c & any) | force);
            }
            w_up = w_c;
            w_c = w_d;
            lb_c = lb[sd];
            rb_c = rbt[sd];
            o += p.out_stride;
            if (++y == p.h) y = 0;
        }
    }
}

}  // namespace bitedge

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
    int thr;                 // uint8 pack threshold (1 = nonzero is white)
    uint32_t *o_side[4];     // kOutAll only: fundamental edges L, R, U, D (or nullptr)
    uint32_t *o_packed;      // kOutAll only: the packed input, padding 1 (or nullptr)
    int pdl_late;            // K2w: signal dependents after the stores, not at entry
    int oswap;               // K2t2: 1 = uint64 output words (pixel word p at uint32 index p ^ 1)
    const char *in_end;      // K1 UNAL: end of the input buffer (loads stop there)
    int unal_words;          // K1 UNAL: load the 4 words one by one instead of 2 chunks
    int h16;                 // K1: 8-word items from 16-byte (not 32-byte) aligned rows
    int rsl;                 // K2t2 with RSL = 0: rows per strip (>= 2)
};

// kOutAll: every requested output of one word from the values the edge formula
// already has (pixel-order, white polarity): centre c, the neighbour planes
// ln / rn / u / d (fill applied) and the padding force f.  Fundamental edge of
// a side = black centre AND white neighbour on that side.
struct AllWords {
    uint32_t e, s, l, r, u, d, pk;
};
__device__ __forceinline__ AllWords all_words(uint32_t c, uint32_t ln, uint32_t rn, uint32_t u,
                                              uint32_t d, uint32_t f) {
    const uint32_t a = ln | rn | u | d, b = ~c;
    return {c | ~a | f, (b & a) | f, (b & ln) | f, (b & rn) | f, (b & u) | f, (b & d) | f, c | f};
}

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

// Load CW (8, 4 or 1) consecutive uint32 words with one 256/128/32-bit load.
template <int CW>
__device__ __forceinline__ void load_chunk(const char *p, uint32_t (&v)[CW]) {
    if constexpr (CW == 1) {
        v[0] = __ldg(reinterpret_cast<const uint32_t *>(p));
    } else if constexpr (CW == 8) {
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
    if constexpr (CW == 1) {
        __stcs(p, v[0]);
    } else if constexpr (CW == 8) {
        asm volatile("st.global.cs.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]),
                     "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                     : "memory");
    } else {
        __stcs(reinterpret_cast<uint4 *>(p), make_uint4(v[0], v[1], v[2], v[3]));
    }
}

// K1 item store: one CW-word vector store, or (H16: 16-byte aligned rows) two
// 128-bit stores of an 8-word item.
template <int CW, bool H16>
__device__ __forceinline__ void store_item(uint32_t *p, const uint32_t (&v)[CW]) {
    if constexpr (H16) {
        __stcs(reinterpret_cast<uint4 *>(p), make_uint4(v[0], v[1], v[2], v[3]));
        __stcs(reinterpret_cast<uint4 *>(p + 4), make_uint4(v[4], v[5], v[6], v[7]));
    } else {
        store_chunk<CW>(p, v);
    }
}

// Item = CW pixel words of one row (memory order == pixel order for uint32 rows;
// uint64 rows swap the halves of each word pair).  RS rows per strip.
// PBM P4 rows (1 = black, MSB-first bytes).  A little-endian
// load of 4 P4 bytes is the pixel-order word with its bytes reversed (pi) and
// inverted.  AND / OR / NOT commute with pi, so only the horizontal shifts need
// pixel order: the P4 kernel keeps up / centre / down rows as loaded, byte-swaps
// the centre row once for the funnel shifts (black polarity: ~Ln, ~Rn), swaps
// the shifted result back, and evaluates the edge formula in the P4 domain:
//   out = c & ~(pi(~Ln & ~Rn) & u & d)      (1 = black edge pixel)
__device__ __forceinline__ uint32_t p4_pi(uint32_t v) { return __byte_perm(v, 0, 0x0123); }

// Unsigned 32-bit division by a launch constant without the IDIV sequence
// (Granlund-Montgomery): q = (umulhi(n, m) + n) >> l, exact for all n < 2^32.
struct FastDiv {
    uint32_t m;
    int l;
};
inline FastDiv make_fastdiv(uint32_t d) {       // host; d >= 1
    int l = 0;
    while (((uint64_t)1 << l) < d) ++l;
    const uint64_t m = ((((uint64_t)1 << l) - d) << 32) / d + 1;
    return {(uint32_t)m, l};
}
__device__ __forceinline__ uint32_t fdiv(uint32_t n, FastDiv f) {
    return (uint32_t)(((uint64_t)__umulhi(n, f.m) + n) >> f.l);
}

// K1 per-launch constants beyond RegParams: the thread -> (strip, item) and
// row -> row-in-image divisions.  Valid when strips * items and nrows < 2^32
// (k1_setup checks; the callers fall back to the tile kernel otherwise).
struct K1Div {
    FastDiv items, h;
};
inline bool k1_setup(const RegParams &p, K1Div &d) {
    if (p.nstrips * (int64_t)p.items + kThreads >= ((int64_t)1 << 32) || p.row_hi >= ((int64_t)1 << 32))
        return false;
    d.items = make_fastdiv((uint32_t)p.items);
    d.h = make_fastdiv(p.h);
    return true;
}

// ALIGNED: w % (32 * CW) == 0 (C3, C4 and P4 at those sizes) -- every item is
// whole, there are no padding bits and the only border work at the right edge
// is the fill word to the right of a row's last item, so the per-word tail
// test (pixel w-1 fill, padding force) is compiled out.
// UNAL: rows are only 4-byte aligned (packed rows that are not 16-byte multiples,
// e.g. the drop-in's uint64 words at w = 8000; P4 payloads of w % 32 == 0 or
// 25..31).  An item's 4 words are loaded one by one (default), or cut out of the
// two aligned 16-byte chunks around them (`unal_words` = 0: two L1-cached vector
// loads and a word select by the row's misalignment -- measured slower: 8192 x
// 8000 u32 4.95 vs 4.43 us, 8.6 vs 6.6 us serially); a row's last item may read
// into the next row (padding positions) but never past `in_end`.  CW must be 4.
template <int SWAP, int RS, int CW, int OUT, bool HALO, bool P4 = false, bool ALIGNED = false,
          bool UNAL = false, bool H16 = false>
__global__ void __launch_bounds__(kThreads, P4 ? (RS == 4 ? 3 : 4) : 0)   // P4: 3 (4-row) or 4 CTAs/SM; 0 = unset
edge_reg_packed_kernel(const RegParams p, const K1Div dv) {
    static_assert(!H16 || (CW == 8 && !UNAL && !P4), "H16: 8-word items from 16-byte rows");
    pdl_wait();
    pdl_trigger();
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;   // < 2^32 (k1_setup)
    const int lane = threadIdx.x & 31;
    const uint32_t strip = fdiv(t, dv.items);
    const int c = (int)(t - strip * (uint32_t)p.items);
    const bool live = strip < p.nstrips;
    const int64_t g0 = p.row_lo + (int64_t)strip * RS;
    const int pw0 = CW * c;
    const uint32_t fw = p.fillword;
    const int64_t rb = p.in_row_bytes;

    // ---- issue every load of the strip up front; staged row i = global row g0-1+i.
    // Rows outside [0, nrows) are loaded from a clamped (valid) address: their
    // values are never used -- the first/last row of every image takes the fill
    // (top / bot below) unless a halo pointer supplies the neighbour row -- so
    // no predicates or fill moves are needed here.
    const char *col = p.in + 4 * pw0;
    const int64_t last = p.nrows - 1;
    const bool need_l = live && c > 0 && lane == 0;
    const bool need_r = live && c + 1 < p.items && lane == 31;
    uint32_t v[RS + 2][CW];
    uint32_t lwx[RS], rwx[RS];
#pragma unroll
    for (int i = 0; i < RS + 2; ++i) {
        const int64_t gi = g0 - 1 + i;
        const char *ptr = col + min(max(gi, (int64_t)0), last) * rb;
        if (HALO) {
            if (i == 0 && gi < 0 && p.above) ptr = p.above + 4 * pw0;
            if (i >= 1 && gi == p.nrows && p.below) ptr = p.below + 4 * pw0;   // partial last strip too
        }
        if constexpr (UNAL) {
            static_assert(CW == 4, "UNAL items are 4 words");
            const int m = (int)(((uintptr_t)ptr >> 2) & 3);      // word misalignment of the row
            const char *a0 = ptr - 4 * m;                       // 16-byte aligned
            if (!p.unal_words && a0 + 32 <= p.in_end) {
                // L1-cached: lane L's second chunk is lane L+1's first
                const uint4 x = __ldg(reinterpret_cast<const uint4 *>(a0));
                const uint4 y = __ldg(reinterpret_cast<const uint4 *>(a0 + 16));
                const uint32_t t[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    v[i][q] = m == 0 ? t[q] : m == 1 ? t[q + 1] : m == 2 ? t[q + 2] : t[q + 3];
            } else {                                            // the buffer's last bytes
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    v[i][q] = ptr + 4 * q + 4 <= p.in_end ? __ldg((const uint32_t *)ptr + q) : 0u;
            }
        } else if constexpr (H16) {
            // rows that are 16-byte but not 32-byte multiples (the drop-in's uint64
            // words at w % 128 in 65..127, e.g. 8000 px = 1008 B): 8-word items
            // as two 128-bit loads, so the per-item work stays amortised over 8 words
            // L1-allocating: a 32-byte sector holds lane L's second half and lane
            // L+1's first (rows start at 16 mod 32), so the second request hits L1
            const uint4 x = __ldg(reinterpret_cast<const uint4 *>(ptr));
            const uint4 y = __ldg(reinterpret_cast<const uint4 *>(ptr + 16));
            v[i][0] = x.x; v[i][1] = x.y; v[i][2] = x.z; v[i][3] = x.w;
            v[i][4] = y.x; v[i][5] = y.y; v[i][6] = y.z; v[i][7] = y.w;
        } else {
            load_chunk<CW>(ptr, v[i]);               // P4: raw bytes, converted per use
        }
        if (i >= 1 && i <= RS) {
            // P4: raw bytes, byte-swapped at use (converting here would make the
            // warp wait for this load before issuing the next rows' loads); the
            // defaults (black polarity) are invariant under the byte swap
            lwx[i - 1] = P4 ? ~fw : fw;
            rwx[i - 1] = P4 ? 0xFFFFFFFFu : 0u;
            if (need_l) lwx[i - 1] = __ldg((const uint32_t *)ptr + (SWAP ? -2 : -1));
            if (need_r) rwx[i - 1] = __ldg((const uint32_t *)ptr + (SWAP ? CW + 1 : CW));
        }
    }

    const bool tail = pw0 + CW - 1 >= p.pl;
    const int nst = min(CW, p.wp - pw0);
    const uint32_t pad_pi = P4 ? p4_pi(p.padmask) : 0u;
    uint32_t y = live ? (uint32_t)g0 - fdiv((uint32_t)g0, dv.h) * p.h : 0u;
    int64_t o = g0 * p.out_stride + pw0;
#pragma unroll
    for (int r = 0; r < RS; ++r) {
        // pixel-order views of up / centre / down
        uint32_t cu[CW], cc[CW], cd[CW];
#pragma unroll
        for (int q = 0; q < CW; ++q) {
            cu[q] = v[r][q ^ SWAP];
            cc[q] = P4 ? p4_pi(v[r + 1][q]) : v[r + 1][q ^ SWAP];   // P4: pixel order, 1 = black
            cd[q] = v[r + 2][q ^ SWAP];
        }
        uint32_t lw = __shfl_up_sync(0xFFFFFFFFu, cc[CW - 1], 1);
        uint32_t rw = __shfl_down_sync(0xFFFFFFFFu, cc[0], 1);
        if (lane == 0) lw = P4 ? p4_pi(lwx[r]) : lwx[r];
        if (lane == 31) rw = P4 ? p4_pi(rwx[r]) : rwx[r];
        if (c == 0) lw = P4 ? ~fw : fw;
        if (ALIGNED && c + 1 == p.items) rw = P4 ? ~fw : fw;   // pixel w is outside: the fill
        const int64_t g = g0 + r;
        if (live && g < p.row_hi) {
            const bool top = (y == 0) && !(HALO && p.above);
            const bool bot = (y == p.h - 1) && !(HALO && p.below);
            const uint32_t ufill = P4 ? ~fw : fw;
            // Neighbour planes of word q (pixel order; P4: black polarity) with the
            // fill at pixel w-1 and the padding force on the row's last item.
            auto planes = [&](int q, uint32_t &ln, uint32_t &rn, uint32_t &u, uint32_t &d,
                              uint32_t &f) {
                const uint32_t left = q == 0 ? lw : cc[q - 1];
                const uint32_t right = q == CW - 1 ? rw : cc[q + 1];
                ln = __funnelshift_r(cc[q], left, 1);
                rn = __funnelshift_l(right, cc[q], 1);
                u = top ? ufill : cu[q];
                d = bot ? ufill : cd[q];
                f = 0u;
                if (!ALIGNED && tail) {
                    const int pw = pw0 + q;
                    if (pw == p.pl) {
                        rn = (rn & ~p.lastbit) | ((P4 ? ~fw : fw) & p.lastbit);
                        f = P4 ? pad_pi : p.padmask;
                    } else if (pw > p.pl) {
                        f = 0xFFFFFFFFu;
                    }
                }
            };
            if constexpr (OUT == kOutAll) {
                uint32_t lnv[CW], rnv[CW], uv[CW], dv2[CW], fv[CW];
#pragma unroll
                for (int q = 0; q < CW; ++q) planes(q, lnv[q], rnv[q], uv[q], dv2[q], fv[q]);
                // one output at a time, rebuilt from the neighbour planes
                auto put = [&](uint32_t *dst, int which) {
                    if (dst == nullptr) return;
                    uint32_t tw[CW];
#pragma unroll
                    for (int q = 0; q < CW; ++q) {
                        const AllWords x = all_words(cc[q], lnv[q], rnv[q], uv[q], dv2[q], fv[q]);
                        tw[q ^ SWAP] = which == 0 ? x.e : which == 1 ? x.s : which == 2 ? x.l
                                     : which == 3 ? x.r : which == 4 ? x.u : which == 5 ? x.d : x.pk;
                    }
                    if (nst == CW && p.vst) {
                        store_item<CW, H16>(dst + o, tw);
                    } else {
                        for (int q = 0; q < nst; ++q) dst[o + q] = tw[q];
                    }
                };
                put(p.o_edges, 0);
                put(p.o_eset, 1);
                put(p.o_side[0], 2);
                put(p.o_side[1], 3);
                put(p.o_side[2], 4);
                put(p.o_side[3], 5);
                put(p.o_packed, 6);
            } else {
                uint32_t ve[CW], vs[CW];
                auto word = [&](int q) {
                    uint32_t ln, rn, u, d, f;
                    planes(q, ln, rn, u, d, f);
                    if (P4) {
                        // ln / rn are ~Ln / ~Rn here (black polarity); the force is
                        // already in P4 byte order.  out = c & ~(pi(~Ln & ~Rn) & u & d)
                        ve[q] = v[r + 1][q] & ~(p4_pi(ln & rn) & u & d) & ~f;
                        vs[q] = 0u;
                    } else {
                        const uint32_t a = ln | rn | u | d;
                        ve[q ^ SWAP] = cc[q] | ~a | f;
                        vs[q ^ SWAP] = (~cc[q] & a) | f;
                    }
                };
#pragma unroll
                for (int q = 0; q < CW; ++q) word(q);
                if (nst == CW && p.vst) {
                    if (OUT != kOutEset) store_item<CW, H16>(p.o_edges + o, ve);
                    if (OUT != kOutEdges) store_item<CW, H16>(p.o_eset + o, vs);
                } else {
                    for (int q = 0; q < nst; ++q) {
                        if (OUT != kOutEset) p.o_edges[o + q] = ve[q];
                        if (OUT != kOutEdges) p.o_eset[o + q] = vs[q];
                    }
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
// General (thresholded) pack of 32 bytes, specialised on t < 128 / t >= 128 so
// each 4-byte compare is 3 ops (the t-independent form needs a 4-input
// function): bit 7 of byte k of ge(v) = (byte k >= t).  Two words of flags merge
// as ga | gb >> 4 (flags at 7,15,23,31 and 3,11,19,27) and one multiply by
// 2^31+2^22+2^13+2^4 gathers them in pixel order into bits 31..38.
template <bool HI>
__device__ __forceinline__ uint32_t ge4(uint32_t v, uint32_t tl) {
    const uint32_t x = (v | 0x80808080u) - tl;   // bit 7: low 7 bits of the byte >= t & 0x7f
    return HI ? (v & x & 0x80808080u)             // t >= 128: byte >= 128 and low bits >= tl
              : ((v | x) & 0x80808080u);          // t < 128: byte >= 128 or low bits >= tl
}

template <bool HI>
__device__ __forceinline__ uint32_t pack8_t(uint32_t a, uint32_t b, uint32_t tl) {
    const uint32_t t = ge4<HI>(a, tl) | (ge4<HI>(b, tl) >> 4);
    return (uint32_t)(((uint64_t)t * 0x80402010ull) >> 31) & 0xFFu;
}

template <bool HI>
__device__ __forceinline__ uint32_t pack32_t(uint4 a, uint4 b, uint32_t tl) {
    return (pack8_t<HI>(a.x, a.y, tl) << 24) | (pack8_t<HI>(a.z, a.w, tl) << 16) |
           (pack8_t<HI>(b.x, b.y, tl) << 8) | pack8_t<HI>(b.z, b.w, tl);
}

__device__ __forceinline__ uint32_t pack32(uint4 a, uint4 b, const Thr &T) {
    return T.m ? pack32_t<false>(a, b, T.tl) : pack32_t<true>(a, b, T.tl);   // launch-uniform
}

// 8 bytes that are all 0 or 1 -> 8 bits MSB-first: x*16 + y puts the flags of
// x at bits 4,12,20,28 and of y at 0,8,16,24 (no carries: bytes <= 1), then the
// same collision-free multiply as pack8.
__device__ __forceinline__ uint32_t pack8_01(uint32_t x, uint32_t y) {
    const uint64_t prod = (uint64_t)(x * 16u + y) * 0x80402010ull;
    return (uint32_t)(prod >> 28) & 0xFFu;
}

// pack32 with a fast path for canonical 0/1 pixel bytes (what to_array and a
// binarisation produce): one test per 32 bytes skips the per-byte nonzero
// normalisation; any other byte value takes the general path.  Exact for all
// inputs (nonzero -> white, bitimage.py:124,133).
__device__ __forceinline__ uint32_t pack32_any(uint4 a, uint4 b, const Thr &T) {
    if (T.t == 1u) {     // launch-uniform: thresholded launches skip the 0/1 test
        const uint32_t hi = (a.x | a.y | a.z | a.w | b.x | b.y | b.z | b.w) & 0xFEFEFEFEu;
        if (hi == 0u) {
            return (pack8_01(a.x, a.y) << 24) | (pack8_01(a.z, a.w) << 16) |
                   (pack8_01(b.x, b.y) << 8) | pack8_01(b.z, b.w);
        }
    }
    return pack32(a, b, T);
}

// ld.global.nc.u8 under a predicate, no branch (lanes with p == 0 keep `dflt`).
__device__ __forceinline__ uint32_t ldg_u8_if(bool p, const char *ptr, uint32_t dflt) {
    uint32_t v = dflt;
    asm volatile(
        "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.global.nc.u8 %0, [%1];\n}\n"
        : "+r"(v)
        : "l"(ptr), "r"((uint32_t)p));
    return v;
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
// contiguous rows, h == G * RPI with G <= GMAX <= 8.  GMAX sizes the register
// file for the up-front loads: C2 (G = 4) with GMAX = 4 needs ~half the
// registers of GMAX = 8, so more warps are resident -- 4096 images in one wave.
template <int LWPR, int OUT, int GMAX = 8>
__global__ void __launch_bounds__(kThreads)
edge_warp_img_kernel(const RegParams p, int G, int64_t nimg) {
    pdl_wait();
    if (!p.pdl_late) pdl_trigger();
    const Thr T = make_thr(p.thr);
    constexpr int WPR = 1 << LWPR;
    constexpr int RPI = 32 >> LWPR;
    const int64_t img = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (img >= nimg) return;                      // whole warps exit together
    const int lane = threadIdx.x & 31;
    const int rl = lane >> LWPR, wi = lane & (WPR - 1);
    const uint32_t fw = p.fillword;
    const char *src = p.in + img * (int64_t)G * 1024 + 32 * lane;
    uint4 a[GMAX], b[GMAX];
#pragma unroll
    for (int k = 0; k < GMAX; ++k)
        if (k < G) ldg_stream_v8(src + 1024 * k, a[k], b[k]);
    uint32_t wd[GMAX];
#pragma unroll
    for (int k = 0; k < GMAX; ++k) wd[k] = k < G ? pack32_any(a[k], b[k], T) : 0xFFFFFFFFu;

    uint32_t *oe = p.o_edges + img * (int64_t)G * 32 + lane;
    uint32_t *os = p.o_eset + img * (int64_t)G * 32 + lane;
    const bool last_word = (wi == WPR - 1);
#pragma unroll
    for (int k = 0; k < GMAX; ++k) {
        if (k >= G) break;
        const uint32_t cw = wd[k];
        // rows above / below inside this row group, and across the group boundary
        const uint32_t up_in = __shfl_up_sync(0xFFFFFFFFu, cw, WPR);
        const uint32_t dn_in = __shfl_down_sync(0xFFFFFFFFu, cw, WPR);
        const uint32_t up_x = __shfl_sync(0xFFFFFFFFu, k > 0 ? wd[k > 0 ? k - 1 : 0] : fw,
                                          (lane + 32 - WPR) & 31);
        const uint32_t dn_x = __shfl_sync(0xFFFFFFFFu,
                                          k + 1 < G ? wd[k + 1 < GMAX ? k + 1 : GMAX - 1] : fw,
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
    if (p.pdl_late) pdl_trigger();
}

// K2 one-shot strips.  UNAL: rows start at any byte (row lengths that are not
// 16-byte multiples, strided views): a word's 32 bytes come from the 9 aligned
// 32-bit words around them (L1-cached loads) and one byte permute per word;
// never read past the aligned 4 (8: 64-bit loads) bytes holding the buffer's last
// byte.  Output words go to column c ^ oswap (1: the drop-in's uint64 layout; the
// u64 row's last u32 word may be pure padding).
// Aligned 4-row strips at 64 registers (4 CTAs/SM; ~20 bytes of spills): a 4096^2
// raster's 512 CTAs are one wave instead of 1.15 of the 74-register build's 444
// (4.58 -> 4.36 us, 8.25 -> 6.38 us on one stream; 16x1024^2 6.31 -> 5.52 us).  The
// UNAL variants were mixed (16x1024x1000: 8.7 -> 7.7 us serial, 3.97 -> 4.15 overlapped).
#ifndef K2_MINB
#define K2_MINB 4
#endif
template <int RS, int OUT, bool HALO, bool V8, int UNAL = 0>   // UNAL: 0, 1 (any byte), 4, 8 (row alignment)
__global__ void __launch_bounds__(kThreads, (RS == 4 && UNAL == 0 && OUT != kOutAny) ? K2_MINB : 0)
edge_reg_u8_kernel(const RegParams p) {
    pdl_wait();
    pdl_trigger();
    const Thr T = make_thr(p.thr);
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
    const bool inrow = x0 < p.w;                       // else a pure padding word (u64 rows)
    const bool need_l = live && c > 0 && lane == 0;
    const bool need_r = live && c + 1 < p.items && lane == 31 && x0 + 32 < p.w;

    const char *base = p.in + (g0 - 1) * rb + x0;
    const int i_lo = g0 == 0 ? 1 : 0;
    const int64_t lim = p.nrows - (g0 - 1);
    uint32_t wd[RS + 2];
    uint32_t lbit[RS], rbit[RS];
    {
        uint4 ra[RS + 2], rb2[RS + 2];
        uint32_t usem = 0u;                            // UNAL: bit i = staged row i was loaded
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
            if constexpr (UNAL == 1) {
                // Branch-free, so the loads of all RS + 2 rows are issued before the first
                // use (with a branch per row -- row present? buffer end? -- every row's
                // loads waited for the previous row's: 1024 x 256 x 250 26.9 -> 24.3 us,
                // 64 x 256 x 250 2.43 -> 1.98 us).  A row that does not exist reads the
                // buffer's first bytes and is whitened after the pack; words past the
                // buffer's last byte (the last row's last item: padding positions) read
                // the buffer's last word instead.  (The same change to the 8- / 4-byte
                // aligned variants cost registers -- 77 / 100 -- and 10 % on large
                // batches: 256 x 500 x 1000 30.1 -> 33.3 us; they keep their branches.)
                const bool use = ok && inrow;
                usem |= use ? (1u << i) : 0u;
                const char *src = use ? ptr : p.in;
                // any byte: the 9 aligned words around the 32 bytes + one permute each
                const uintptr_t pa = (uintptr_t)src;
                const char *a4 = reinterpret_cast<const char *>(pa & ~(uintptr_t)3);
                const char *lastw = reinterpret_cast<const char *>(((uintptr_t)p.in_end - 1) & ~(uintptr_t)3);
                const uint32_t sel = 0x3210u + 0x1111u * (uint32_t)(pa & 3);
                uint32_t tw[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) {
                    const char *a = a4 + 4 * k;
                    tw[k] = __ldg(reinterpret_cast<const uint32_t *>(a < lastw ? a : lastw));
                }
                ra[i] = make_uint4(__byte_perm(tw[0], tw[1], sel), __byte_perm(tw[1], tw[2], sel),
                                   __byte_perm(tw[2], tw[3], sel), __byte_perm(tw[3], tw[4], sel));
                rb2[i] = make_uint4(__byte_perm(tw[4], tw[5], sel), __byte_perm(tw[5], tw[6], sel),
                                    __byte_perm(tw[6], tw[7], sel), __byte_perm(tw[7], tw[8], sel));
            } else if (ok && inrow) {
                if constexpr (UNAL == 8 || UNAL == 4) {
                    // rows 8- / 4-byte aligned: the 32 bytes as 4 x 64-bit / 8 x 32-bit
                    // loads (a row's last word may read into the next row, never past
                    // in_end)
                    uint32_t tw[8];
                    if (ptr + 32 <= p.in_end) {
                        if (UNAL == 8 || ((uintptr_t)ptr & 7) == 0) {   // this row 8-byte aligned
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const uint2 q = __ldg(reinterpret_cast<const uint2 *>(ptr) + k);
                                tw[2 * k] = q.x; tw[2 * k + 1] = q.y;
                            }
                        } else {                        // 4 mod 8: 32 + 3 x 64 + 32 bits
                            tw[0] = __ldg(reinterpret_cast<const uint32_t *>(ptr));
#pragma unroll
                            for (int k = 0; k < 3; ++k) {
                                const uint2 q = __ldg(reinterpret_cast<const uint2 *>(ptr + 4) + k);
                                tw[2 * k + 1] = q.x; tw[2 * k + 2] = q.y;
                            }
                            tw[7] = __ldg(reinterpret_cast<const uint32_t *>(ptr) + 7);
                        }
                    } else {                                   // the buffer's last bytes
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            uint32_t v = 0u;
                            for (int j = 0; j < 4; ++j)
                                if (ptr + 4 * k + j < p.in_end)
                                    v |= (uint32_t)(uint8_t)__ldg(ptr + 4 * k + j) << (8 * j);
                            tw[k] = v;
                        }
                    }
                    ra[i] = make_uint4(tw[0], tw[1], tw[2], tw[3]);
                    rb2[i] = make_uint4(tw[4], tw[5], tw[6], tw[7]);
                } else if (V8) {
                    ldg_stream_v8(ptr, ra[i], rb2[i]);
                } else {
                    ra[i] = ldg_stream_v4(ptr);
                    if (has_hi) rb2[i] = ldg_stream_v4(ptr + 16);
                }
            }
            if (i >= 1 && i <= RS) {
                // the neighbour bytes across warps (lanes 0 / 31), raw: comparing them
                // here made the warp wait for each byte before issuing the next row's
                // loads (rows that are not 1024-px multiples; 256 x 480 x 640: ncu
                // long-scoreboard 7.0 against 2.5 on 512-px rows)
                lbit[i - 1] = 0xFFFFFFFFu;
                rbit[i - 1] = 0xFFFFFFFFu;
                if (ok && need_l) lbit[i - 1] = (uint8_t)ptr[-1];
                if (ok && need_r) rbit[i - 1] = (uint8_t)ptr[32];
            }
        }
#pragma unroll
        for (int r = 0; r < RS; ++r) {
            lbit[r] = lbit[r] == 0xFFFFFFFFu ? fw : (lbit[r] >= (uint32_t)T.t ? 1u : 0u);
            rbit[r] = rbit[r] == 0xFFFFFFFFu ? 0u : (rbit[r] >= (uint32_t)T.t ? 0x80000000u : 0u);
        }
#pragma unroll
        for (int i = 0; i < RS + 2; ++i) {
            wd[i] = pack32_any(ra[i], rb2[i], T);
            if (UNAL == 1 && !((usem >> i) & 1u)) wd[i] = 0xFFFFFFFFu;
        }
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
    int64_t o = g0 * p.out_stride + (c ^ p.oswap);
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
            if (OUT != kOutEset && p.o_edges) __stcs(p.o_edges + o, cw | ~any | force);
            if (OUT != kOutEdges) __stcs(p.o_eset + o, (~cw & any) | force);
            if (p.o_packed) __stcs(p.o_packed + o, cw | force);   // from_array's words
        }
        o += p.out_stride;
        if (++y == p.h) y = 0;
    }
}

// K2r: uint8 pixels, long strips with a rolling register window.  A thread
// owns one output word (32 pixels) of RSL consecutive rows and keeps the next
// 2-3 rows' 256-bit loads in flight while it packs and emits the current
// one, so the 2 halo rows cost 2/RSL instead of 2/RS (the one-shot K2's
// dominant overhead on big pages, BASELINE config C5).  Ring of Q raw
// slots (Q-1 rows in flight); the loop is unrolled by Q so slot indices are static.
template <int RSL, int Q, int OUT, bool HALO>
__global__ void __launch_bounds__(kThreads)
edge_roll_u8_kernel(const RegParams p) {
    pdl_wait();
    pdl_trigger();
    const Thr T = make_thr(p.thr);
    static_assert(RSL % Q == 0 && Q >= 4, "strip must be a multiple of the ring");
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

    // staged row i (global g0-1+i), i in [0, RSL+2): raw 32 bytes, plus for the
    // warp's edge lanes the neighbouring pixels (bit 0: x0-1, bit 31: x0+32).
    // Loads are branch-free: a row that does not exist reads row 0 of the
    // raster instead (always valid) and is marked absent in `okm`.
    const int nvis = live ? (int)(lim < RSL + 2 ? lim : RSL + 2) : 0;   // rows i < nvis exist
    const char *safe = p.in + x0;
    uint4 ra[Q], rb2[Q];
    uint32_t ebl[Q], ebr[Q];       // raw neighbour bytes across warps, compared at use (see K2)
    uint32_t okm = 0u;                                                 // bit slot: row present
    auto issue = [&](int i, int slot) {
        const char *ptr = base + i * rb;
        bool ok = i >= i_lo && i < nvis;
        if (HALO) {
            if (i == 0 && g0 == 0 && p.above && live) { ptr = p.above + x0; ok = true; }
            if (i == lim && i < RSL + 2 && p.below && live) { ptr = p.below + x0; ok = true; }
        }
        ldg_stream_v8(ok ? ptr : safe, ra[slot], rb2[slot]);
        okm = ok ? (okm | (1u << slot)) : (okm & ~(1u << slot));
        ebl[slot] = ldg_u8_if(ok && need_l, ptr - 1, 0u);
        ebr[slot] = ldg_u8_if(ok && need_r, ptr + 32, 0u);
    };
    auto edge_bits = [&](int slot) -> uint32_t {
        return (ebl[slot] >= (uint32_t)T.t ? 1u : 0u) | (ebr[slot] >= (uint32_t)T.t ? 0x80000000u : 0u);
    };
    auto word = [&](int slot) -> uint32_t {
        return (okm >> slot) & 1u ? pack32_any(ra[slot], rb2[slot], T) : 0xFFFFFFFFu;
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

    // prologue: staged rows 0 (halo above) .. Q-1 in flight; pack rows 0 and 1
#pragma unroll
    for (int i = 0; i < Q; ++i) issue(i, i);
    uint32_t w_up = word(0);
    uint32_t w_c = word(1);
    uint32_t e_c = edge_bits(1);
    for (int r0 = 0; r0 < RSL; r0 += Q) {
#pragma unroll
        for (int k = 0; k < Q; ++k) {
            const int r = r0 + k;                      // output row; staged row r+1 is centre
            issue(r + Q, k);                           // rows r+2 .. r+Q stay in flight
            const int sd = (k + 2) % Q;                // staged row r+2 = down neighbour
            const uint32_t w_d = word(sd);
            uint32_t lw = __shfl_up_sync(0xFFFFFFFFu, w_c, 1);
            uint32_t rw = __shfl_down_sync(0xFFFFFFFFu, w_c, 1);
            if (lane == 0) lw = e_c;
            if (lane == 31) rw = e_c;
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
            e_c = edge_bits(sd);
            o += p.out_stride;
            if (++y == p.h) y = 0;
        }
    }
}

// ---------------------------------------------------------------- K2t: uint8, per-warp TMA ring

// mbarrier / TMA helpers (shared with edge_stream.cuh's design, redeclared here
// to keep this header standalone).
__device__ __forceinline__ uint32_t sm_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void wbar_init(uint64_t *b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm_addr(b)));
}
__device__ __forceinline__ void wbar_expect(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_addr(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void wbar_wait(uint64_t *b, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred P1;\n"
        "W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra W_%=;\n}\n" ::"r"(
            sm_addr(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void wtma(void *dst, const void *src, uint32_t bytes, uint64_t *b) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(sm_addr(dst)),
        "l"(src), "r"(bytes), "r"(sm_addr(b))
        : "memory");
}

// K2p: the K2w batch shape (small uint8 images, one warp per image) with the
// whole batch requested from DRAM at kernel start.  K2w issues each image's
// loads from registers, so a batch is 1.15 waves at C2 and the last 15 % of
// images start a full load latency late; here every warp's lane 0 issues one
// `cp.async.bulk` (TMA) per image it owns into shared memory -- up to
// IPW images per warp, the CTA's 8 warps holding <= 8 * IPW * G KB -- each
// tracked by its own mbarrier, so with one CTA per SM all ~16 MiB of C2 are in
// flight at once; each warp then computes its images in arrival order with
// K2w's register math, reading its lane's 32 bytes of each row group from
// shared memory.  Warps get a balanced contiguous range of images (global warp
// gw owns images [gw*N/W, (gw+1)*N/W)).
template <int LWPR, int OUT, int IPW>
__global__ void __launch_bounds__(kThreads, 1)
edge_warp_img_tma_kernel(const RegParams p, int G, int64_t nimg, int64_t nwarps) {
    extern __shared__ __align__(128) unsigned char k2p_smem[];
    constexpr int WPR = 1 << LWPR;
    constexpr int RPI = 32 >> LWPR;
    constexpr int WARPS = kThreads / 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t gw = (int64_t)blockIdx.x * WARPS + warp;
    if (gw >= nwarps) return;                              // whole warp (no CTA barriers)
    const int64_t i0 = gw * nimg / nwarps, i1 = (gw + 1) * nimg / nwarps;
    const int cnt = (int)(i1 - i0);                        // <= IPW (host sizes nwarps)
    const uint32_t img_bytes = (uint32_t)G * 1024u;
    // [mbarriers of all warps | image buffers]: the header holds WARPS * IPW
    // barriers, rounded up to 128 bytes (k2p_smem_bytes on the host)
    constexpr int HDR = (WARPS * IPW * 8 + 127) / 128 * 128;
    uint64_t *bars = reinterpret_cast<uint64_t *>(k2p_smem) + warp * IPW;
    unsigned char *buf = k2p_smem + HDR + (size_t)warp * IPW * img_bytes;
    if (lane == 0) {
        for (int k = 0; k < cnt; ++k) wbar_init(&bars[k]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    pdl_wait();
    pdl_trigger();
    if (lane == 0) {
        for (int k = 0; k < cnt; ++k) {
            wbar_expect(&bars[k], img_bytes);
            wtma(buf + (size_t)k * img_bytes, p.in + (i0 + k) * (int64_t)img_bytes, img_bytes,
                 &bars[k]);
        }
    }
    const Thr T = make_thr(p.thr);
    const int rl = lane >> LWPR, wi = lane & (WPR - 1);
    const uint32_t fw = p.fillword;
    const bool last_word = (wi == WPR - 1);
    for (int k = 0; k < cnt; ++k) {
        wbar_wait(&bars[k], 0);
        const unsigned char *src = buf + (size_t)k * img_bytes + 32 * lane;
        uint32_t wd[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            if (g < G) {
                const uint4 a = *reinterpret_cast<const uint4 *>(src + 1024 * g);
                const uint4 b = *reinterpret_cast<const uint4 *>(src + 1024 * g + 16);
                wd[g] = pack32_any(a, b, T);
            } else {
                wd[g] = 0xFFFFFFFFu;
            }
        }
        const int64_t img = i0 + k;
        uint32_t *oe = p.o_edges + img * (int64_t)G * 32 + lane;
        uint32_t *os = p.o_eset + img * (int64_t)G * 32 + lane;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            if (g >= G) break;
            const uint32_t cw = wd[g];
            const uint32_t up_in = __shfl_up_sync(0xFFFFFFFFu, cw, WPR);
            const uint32_t dn_in = __shfl_down_sync(0xFFFFFFFFu, cw, WPR);
            const uint32_t up_x = __shfl_sync(0xFFFFFFFFu, g > 0 ? wd[g > 0 ? g - 1 : 0] : fw,
                                              (lane + 32 - WPR) & 31);
            const uint32_t dn_x = __shfl_sync(0xFFFFFFFFu, g + 1 < G ? wd[g + 1 < 8 ? g + 1 : 7] : fw,
                                              (lane + WPR) & 31);
            const uint32_t u = rl > 0 ? up_in : (g > 0 ? up_x : fw);
            const uint32_t d = rl < RPI - 1 ? dn_in : (g + 1 < G ? dn_x : fw);
            uint32_t lw = __shfl_up_sync(0xFFFFFFFFu, cw, 1);
            const uint32_t rw = __shfl_down_sync(0xFFFFFFFFu, cw, 1);
            if (wi == 0) lw = fw;
            const uint32_t ln = __funnelshift_r(cw, lw, 1);
            uint32_t rn = __funnelshift_l(rw, cw, 1);
            if (last_word) rn = (rn & ~1u) | (fw & 1u);   // pixel w-1 reads the fill
            const uint32_t any = ln | rn | u | d;
            if (OUT != kOutEset) __stcs(oe + 32 * g, cw | ~any);
            if (OUT != kOutEdges) __stcs(os + 32 * g, ~cw & any);
        }
    }
}

// One warp owns a 1024-pixel row segment (32 output words, one per lane) of a
// strip of RSL rows.  Its lane 0 streams the strip's RSL+2 staged rows (the
// segment plus 16 bytes either side for the neighbour pixels) into a private
// D-slot shared-memory ring with `cp.async.bulk` (TMA), each slot tracked by an
// mbarrier transaction count, so D row segments are in flight per warp without
// holding them in registers -- which is what lets 32 warps per SM keep ~200 KB
// in flight (the register ring of K2r tops out near 75 KB).  Lanes read their
// 32 bytes from shared memory, pack, and emit exactly like K2r.  No CTA-wide
// barriers: warps of a CTA are independent.
template <int RSL, int D, int OUT, bool HALO>
__global__ void __launch_bounds__(kThreads)
edge_tma_u8_kernel(const RegParams p, int64_t nseg, int64_t nwarps) {
    const Thr T = make_thr(p.thr);
    constexpr int SLOT = 1056;                       // 16 + 1024 + 16 bytes
    constexpr int WARPS = kThreads / 32;
    extern __shared__ __align__(128) char tsm[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    char *ring = tsm + (size_t)wid * D * SLOT;
    uint64_t *bars = reinterpret_cast<uint64_t *>(tsm + (size_t)WARPS * D * SLOT) + wid * D;
    if (lane == 0) {
        for (int s = 0; s < D; ++s) wbar_init(&bars[s]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    pdl_wait();
    pdl_trigger();
    const int64_t gw = (int64_t)blockIdx.x * WARPS + wid;
    if (gw >= nwarps) return;                        // whole warp
    const int64_t strip = gw / nseg;
    const int seg = (int)(gw - strip * nseg);
    const int64_t g0 = p.row_lo + strip * RSL;
    const int64_t x0 = (int64_t)seg * 1024;
    const int c = seg * 32 + lane;                   // this lane's output word
    const uint32_t fw = p.fillword;
    const int64_t rb = p.in_row_bytes;
    const int64_t wr = (p.w + 15) & ~(int64_t)15;    // readable bytes per row
    const int64_t b_lo = x0 > 0 ? x0 - 16 : 0;       // copied byte range of a row
    const int64_t b_hi = x0 + 1040 < wr ? x0 + 1040 : wr;
    const uint32_t seg_bytes = (uint32_t)(b_hi - b_lo);
    const int dst_off = (int)(b_lo - (x0 - 16));     // 16 for the first segment, else 0
    const int nst = RSL + 2;                         // staged rows
    static_assert(RSL >= 2, "fetch order needs two own rows");

    // staged row i <-> global row g0-1+i; returns the row pointer or nullptr
    auto row_of = [&](int i) -> const char * {
        const int64_t g = g0 - 1 + i;
        if (g >= 0 && g < p.nrows) return p.in + g * rb;
        if (HALO) {
            if (g == -1) return p.above;
            if (g == p.nrows && i < nst) return p.below;
        }
        return nullptr;
    };
    // fetch order (see K2t2): below halo first, own rows, above halo last
    auto order = [&](int k) { return k == 0 ? nst - 1 : (k == nst - 1 ? 0 : k); };
    auto issue = [&](int k) {                        // lane 0 only; k = fetch position
        if (k >= nst) return;
        const char *row = row_of(order(k));
        if (row == nullptr) return;
        uint64_t *b = &bars[k % D];
        wbar_expect(b, seg_bytes);
        wtma(ring + (k % D) * SLOT + dst_off, row + b_lo, seg_bytes, b);
    };
    if (lane == 0)
        for (int k = 0; k < D; ++k) issue(k);

    uint32_t keep = 0xFFFFFFFFu, fixb = 0u, force = 0u;
    if (c == p.pl) {
        keep = ~p.lastbit;
        fixb = fw & p.lastbit;
        force = p.padmask;
    } else if (c > p.pl) {
        force = 0xFFFFFFFFu;
    }
    const bool live_col = c < p.wp;
    const uint32_t y0 = (uint32_t)(g0 % p.h);
    uint32_t phase = 0u;                             // per-slot parity bits
    auto fetch = [&](int k, uint32_t &w, uint32_t &e) {
        const int slot = k % D;
        w = 0xFFFFFFFFu; e = 0u;
        if (row_of(order(k)) != nullptr) {
            wbar_wait(&bars[slot], (phase >> slot) & 1u);
            phase ^= 1u << slot;
            const char *src = ring + slot * SLOT + 16 + 32 * lane;
            const uint4 a = *reinterpret_cast<const uint4 *>(src);
            const uint4 b = *reinterpret_cast<const uint4 *>(src + 16);
            w = pack32_any(a, b, T);
            if (lane == 0) e = (uint8_t)src[-1] >= T.t ? 1u : 0u;
            if (lane == 31) e = (uint8_t)src[32] >= T.t ? 0x80000000u : 0u;
        }
        // the slot is free (consumed, or never filled because the row does not
        // exist): refill it with the row D fetch positions later
        __syncwarp();
        if (lane == 0) issue(k + D);
    };
    auto emit = [&](int r, uint32_t y, uint32_t w_up, uint32_t w_c, uint32_t w_dn, uint32_t e_c) {
        uint32_t lw = __shfl_up_sync(0xFFFFFFFFu, w_c, 1);
        uint32_t rw = __shfl_down_sync(0xFFFFFFFFu, w_c, 1);
        if (lane == 0) lw = e_c;
        if (lane == 31) rw = e_c;
        if (c == 0) lw = fw;
        if (live_col && g0 + r < p.row_hi) {
            const int64_t o = (g0 + r) * p.out_stride + c;
            const uint32_t u = (y == 0 && !(HALO && p.above)) ? fw : w_up;
            const uint32_t d = (y == p.h - 1 && !(HALO && p.below)) ? fw : w_dn;
            const uint32_t ln = __funnelshift_r(w_c, lw, 1);
            const uint32_t rn = (__funnelshift_l(rw, w_c, 1) & keep) | fixb;
            const uint32_t any = ln | rn | u | d;
            if (OUT != kOutEset) __stcs(p.o_edges + o, w_c | ~any | force);
            if (OUT != kOutEdges) __stcs(p.o_eset + o, (~w_c & any) | force);
        }
    };
    uint32_t w_dn_halo, w_c0, e_c0, w_c, e_c, t;
    fetch(0, w_dn_halo, t);                          // staged nst-1 (below halo)
    fetch(1, w_c0, e_c0);                            // staged 1: output row 0's centre
    fetch(2, w_c, e_c);                              // staged 2
    const uint32_t w_c1 = w_c;
    uint32_t w_up = w_c0;
    uint32_t y = y0 + 1 >= p.h ? (y0 + 1) % p.h : y0 + 1;
    for (int k = 3; k < nst - 1; ++k) {              // output rows 1 .. RSL-2
        uint32_t w_new, e_new;
        fetch(k, w_new, e_new);
        emit(k - 2, y, w_up, w_c, w_new, e_c);
        if (++y == p.h) y = 0;
        w_up = w_c; w_c = w_new; e_c = e_new;
    }
    emit(RSL - 1, y, w_up, w_c, w_dn_halo, e_c);
    uint32_t w_up_halo;
    fetch(nst - 1, w_up_halo, t);                    // staged 0 (above halo)
    emit(0, y0, w_up_halo, w_c0, w_c1, e_c0);
}

// K2t2: same ring, but a warp owns a 2048-pixel row segment and every lane two
// output words (word L and word 32+L of the segment), halving the per-row fixed
// cost (barrier wait, refill, row bookkeeping) per word -- K2t was issue-bound
// at ~200 instructions per 1 KB row segment.  Staged rows are addressed with
// integer offsets from one base pointer; only the first/last staged rows can be
// absent or come from the halo buffers.
// UNAL: uint8 rows at any byte offset (row lengths that are not 16-byte
// multiples).  A staged row segment starts at the 16-byte granule holding its
// first byte, delta = (address & 15) bytes early, so lane L's aligned 32 bytes
// are pixels x0 + 32L - delta ..; each lane packs them as for aligned rows and
// shifts the packed word left by delta bits, taking the low bits from the next
// lane's packed word (one shuffle + one funnel shift per word; lane 31 packs 16
// more bytes).  Every copy stays inside the granules of valid row bytes.
template <int RSL, int D, int OUT, bool HALO, bool UNAL = false>
__global__ void __launch_bounds__(kThreads, 3)   // smem allows 3 CTAs/SM: up to 80 regs, no spills
edge_tma2_u8_kernel(const RegParams p, int64_t nseg, int64_t nwarps) {
    static_assert(!(UNAL && HALO), "UNAL: no halo rows");
    const Thr T = make_thr(p.thr);
    constexpr int SEG = 2048;                        // pixels (bytes) per warp segment
    constexpr int SLOT = UNAL ? 16 + SEG + 48 : 16 + SEG + 16;
    constexpr int WARPS = kThreads / 32;
    extern __shared__ __align__(128) char tsm[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    char *ring = tsm + (size_t)wid * D * SLOT;
    uint64_t *bars = reinterpret_cast<uint64_t *>(tsm + (size_t)WARPS * D * SLOT) + wid * D;
    if (lane == 0) {
        for (int s = 0; s < D; ++s) wbar_init(&bars[s]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    pdl_wait();
    pdl_trigger();
    const int64_t gw = (int64_t)blockIdx.x * WARPS + wid;
    if (gw >= nwarps) return;
    const int64_t strip = gw / nseg;
    const int seg = (int)(gw - strip * nseg);
    // strip height: the template constant, or (RSL == 0) the launch's p.rsl -- the host
    // fits mid-size rasters into whole waves of resident warps with it
    const int rsl = RSL > 0 ? RSL : p.rsl;
    const int64_t g0 = p.row_lo + strip * rsl;
    const int64_t x0 = (int64_t)seg * SEG;
    const int ca = seg * 64 + lane, cb = ca + 32;    // this lane's two output words
    // their uint32 store columns: uint64 output stores pixel word c at c ^ 1
    // (the row stride is then even, so the swap stays inside the row)
    const int cas = ca ^ p.oswap, cbs = cb ^ p.oswap;
    const uint32_t fw = p.fillword;
    const int64_t rb = p.in_row_bytes;
    const int64_t wr = (p.w + 15) & ~(int64_t)15;
    const int64_t b_lo = x0 > 0 ? x0 - 16 : 0;
    const int64_t b_hi = x0 + SEG + 16 < wr ? x0 + SEG + 16 : wr;
    const uint32_t seg_bytes = (uint32_t)(b_hi - b_lo);
    const int dst_off = (int)(b_lo - (x0 - 16));
    const int NST = rsl + 2;                         // rsl >= 2: the fetch order needs two own rows
    // staged rows i in [i_lo, i_hi) lie inside `in`; row 0 / row lim may be halos
    const int i_lo = g0 == 0 ? 1 : 0;
    const int64_t lim = p.nrows - (g0 - 1);
    const int i_hi = lim < NST ? (int)lim : NST;
    const char *base = p.in + (g0 - 1) * rb + b_lo;
    const bool top_halo = HALO && g0 == 0 && p.above != nullptr;
    const bool bot_halo = HALO && lim < NST && p.below != nullptr;
    auto exists = [&](int i) {
        return (i >= i_lo && i < i_hi) || (top_halo && i == 0) || (bot_halo && i == i_hi);
    };
    auto order = [&](int k) { return k == 0 ? NST - 1 : (k == NST - 1 ? 0 : k); };
    auto issue = [&](int k) {                        // lane 0 only; k = fetch position
        if (k >= NST) return;
        const int i = order(k);
        if (!exists(i)) return;
        const char *src = base + i * rb;
        if (top_halo && i == 0) src = p.above + b_lo;
        if (bot_halo && i == i_hi) src = p.below + b_lo;
        uint64_t *b = &bars[k % D];
        if constexpr (UNAL) {
            // [granule of the first byte, end of the granule of the last byte)
            const uintptr_t a0 = (uintptr_t)src & ~(uintptr_t)15;
            const int64_t end_px = x0 + SEG + 16 < p.w ? x0 + SEG + 16 : p.w;
            const uintptr_t a1 = ((uintptr_t)(src - b_lo + end_px) + 15) & ~(uintptr_t)15;
            wbar_expect(b, (uint32_t)(a1 - a0));
            wtma(ring + (k % D) * SLOT + dst_off, (const char *)a0, (uint32_t)(a1 - a0), b);
        } else {
            wbar_expect(b, seg_bytes);
            wtma(ring + (k % D) * SLOT + dst_off, src, seg_bytes, b);
        }
    };
    if (lane == 0)
        for (int k = 0; k < D; ++k) issue(k);

    auto tail_consts = [&](int c, uint32_t &keep, uint32_t &fixb, uint32_t &force) {
        keep = 0xFFFFFFFFu; fixb = 0u; force = 0u;
        if (c == p.pl) { keep = ~p.lastbit; fixb = fw & p.lastbit; force = p.padmask; }
        else if (c > p.pl) force = 0xFFFFFFFFu;
    };
    uint32_t ka, fa, ga, kb, fb, gb;
    tail_consts(ca, ka, fa, ga);
    tail_consts(cb, kb, fb, gb);
    const bool la = ca < p.wp, lb_ = cb < p.wp;
    const uint32_t y0 = (uint32_t)(g0 % p.h);
    uint32_t phase = 0u;
    // One staged row: wait for its slot, pack both words, free the slot and
    // refill it with the row D positions later in the fetch order.
    auto fetch = [&](int k, uint32_t &a, uint32_t &b, uint32_t &el, uint32_t &er) {
        const int i = order(k), slot = k % D;
        a = 0xFFFFFFFFu; b = 0xFFFFFFFFu; el = 0u; er = 0u;
        if (exists(i)) {
            wbar_wait(&bars[slot], (phase >> slot) & 1u);
            phase ^= 1u << slot;
            const char *s = ring + slot * SLOT + 16;
            a = pack32_any(*reinterpret_cast<const uint4 *>(s + 32 * lane),
                           *reinterpret_cast<const uint4 *>(s + 32 * lane + 16), T);
            b = pack32_any(*reinterpret_cast<const uint4 *>(s + 1024 + 32 * lane),
                           *reinterpret_cast<const uint4 *>(s + 1024 + 32 * lane + 16), T);
            int dl = 0;
            if constexpr (UNAL) {
                dl = (int)((uintptr_t)(base + i * rb) & 15);        // warp-uniform
                uint32_t xb_ = 0u;                                // lane 31: bytes 2048 .. 2063
                if (lane == 31)
                    xb_ = pack32_any(*reinterpret_cast<const uint4 *>(s + SEG),
                                     make_uint4(0u, 0u, 0u, 0u), T);
                const uint32_t b0 = __shfl_sync(0xFFFFFFFFu, b, 0);
                uint32_t na = __shfl_down_sync(0xFFFFFFFFu, a, 1);
                uint32_t nb = __shfl_down_sync(0xFFFFFFFFu, b, 1);
                if (lane == 31) { na = b0; nb = xb_; }
                a = __funnelshift_l(na, a, dl);
                b = __funnelshift_l(nb, b, dl);
            }
            if (lane == 0) el = (uint8_t)s[dl - 1] >= T.t ? 1u : 0u;
            if (lane == 31) er = (uint8_t)s[dl + SEG] >= T.t ? 0x80000000u : 0u;
        }
        __syncwarp();
        if (lane == 0) issue(k + D);                 // slot free (consumed or unused)
    };
    // Output row r of the strip: up / centre / down words of both halves.
    auto emit = [&](int r, uint32_t y, uint32_t ua, uint32_t ub, uint32_t xa, uint32_t xb,
                    uint32_t na, uint32_t nb, uint32_t el, uint32_t er) {
        const uint32_t a_up = __shfl_up_sync(0xFFFFFFFFu, xa, 1);
        const uint32_t a_dn = __shfl_down_sync(0xFFFFFFFFu, xa, 1);
        const uint32_t b_up = __shfl_up_sync(0xFFFFFFFFu, xb, 1);
        const uint32_t b_dn = __shfl_down_sync(0xFFFFFFFFu, xb, 1);
        const uint32_t a31 = __shfl_sync(0xFFFFFFFFu, xa, 31);   // word 31 (left of word 32)
        const uint32_t b0 = __shfl_sync(0xFFFFFFFFu, xb, 0);     // word 32 (right of word 31)
        const uint32_t lwa = lane == 0 ? (ca == 0 ? fw : el) : a_up;
        const uint32_t rwa = lane == 31 ? b0 : a_dn;
        const uint32_t lwb = lane == 0 ? a31 : b_up;
        const uint32_t rwb = lane == 31 ? er : b_dn;
        if (g0 + r < p.row_hi) {
            const int64_t orow = (g0 + r) * p.out_stride;
            const int64_t oa = orow + cas, ob = orow + cbs;
            const bool top = y == 0 && !(HALO && p.above);
            const bool bot = y == p.h - 1 && !(HALO && p.below);
            const uint32_t uA = top ? fw : ua, uB = top ? fw : ub;
            const uint32_t dA = bot ? fw : na, dB = bot ? fw : nb;
            const uint32_t lnA = __funnelshift_r(xa, lwa, 1);
            const uint32_t rnA = (__funnelshift_l(rwa, xa, 1) & ka) | fa;
            const uint32_t anyA = lnA | rnA | uA | dA;
            const uint32_t lnB = __funnelshift_r(xb, lwb, 1);
            const uint32_t rnB = (__funnelshift_l(rwb, xb, 1) & kb) | fb;
            const uint32_t anyB = lnB | rnB | uB | dB;
            if (OUT == kOutAll) {
                const AllWords A = all_words(xa, lnA, rnA, uA, dA, ga);
                const AllWords B = all_words(xb, lnB, rnB, uB, dB, gb);
                uint32_t *dst[7] = {p.o_edges, p.o_eset, p.o_side[0], p.o_side[1], p.o_side[2],
                                    p.o_side[3], p.o_packed};
                const uint32_t va[7] = {A.e, A.s, A.l, A.r, A.u, A.d, A.pk};
                const uint32_t vb[7] = {B.e, B.s, B.l, B.r, B.u, B.d, B.pk};
#pragma unroll
                for (int k = 0; k < 7; ++k) {
                    if (dst[k] == nullptr) continue;
                    if (la) __stcs(dst[k] + oa, va[k]);
                    if (lb_) __stcs(dst[k] + ob, vb[k]);
                }
            } else {
                if (la) {
                    if (OUT != kOutEset) __stcs(p.o_edges + oa, xa | ~anyA | ga);
                    if (OUT != kOutEdges) __stcs(p.o_eset + oa, (~xa & anyA) | ga);
                }
                if (lb_) {
                    if (OUT != kOutEset) __stcs(p.o_edges + ob, xb | ~anyB | gb);
                    if (OUT != kOutEdges) __stcs(p.o_eset + ob, (~xb & anyB) | gb);
                }
            }
        }
    };
    // Fetch order: below-halo row first (it is the NEXT strip's first row, which
    // that warp fetches at the same moment), then the strip's own rows, and the
    // above-halo row last (the PREVIOUS strip's last row, fetched by that warp at
    // the same moment).  The two shared rows are then read from DRAM once and
    // served to the second reader from L2: ncu showed 2/RSL extra DRAM reads
    // with the in-order fetch.
    uint32_t dwa, dwb, t0, t1;                        // below halo (staged NST-1)
    fetch(0, dwa, dwb, t0, t1);
    uint32_t c0a, c0b, el0, er0;                      // staged 1 = output row 0's centre
    fetch(1, c0a, c0b, el0, er0);
    uint32_t ua = c0a, ub = c0b, xa, xb, el, er;      // staged 2
    fetch(2, xa, xb, el, er);
    const uint32_t c1a = xa, c1b = xb;
    uint32_t y = y0 + 1 >= p.h ? (y0 + 1) % p.h : y0 + 1;
#pragma unroll 1   // one copy of the row body: the pack code is large (i-cache)
    for (int k = 3; k < NST - 1; ++k) {               // output rows 1 .. RSL-2
        uint32_t na, nb, nel, ner;
        fetch(k, na, nb, nel, ner);
        emit(k - 2, y, ua, ub, xa, xb, na, nb, el, er);
        if (++y == p.h) y = 0;
        ua = xa; ub = xb; xa = na; xb = nb; el = nel; er = ner;
    }
    emit(rsl - 1, y, ua, ub, xa, xb, dwa, dwb, el, er);
    uint32_t upa, upb;                                // above halo (staged 0)
    fetch(NST - 1, upa, upb, t0, t1);
    emit(0, y0, upa, upb, c0a, c0b, c1a, c1b, el0, er0);
}

}  // namespace bitedge

// edge_flat.cuh -- K1f: the fused edge kernel for packed rows whose length is
// NOT a multiple of the vector width (SURVEY 8(a) A7 on ragged widths: u32 rows
// of w = 8000 px are 250 words; the drop-in's uint64 BitImage words,
// bitimage.py:91-97, have an odd count whenever w % 128 is in 1..64).
//
// K1 walks column items of row strips, so on such rows every row starts at a
// different 16-byte phase and its items are loaded word by word.  K1f instead
// views the raster (contiguous rows: row stride == words per row == S) as ONE
// flat word array and gives every thread one aligned chunk of CW words of it:
//
//   * centre:  one aligned CW-word vector load of the chunk itself;
//   * up/down: the words at flat -S / +S are at a fixed phase RU = (-S) mod CW
//     / RD = S mod CW from the chunk grid -- the same for every chunk of the
//     launch -- so each lane loads the aligned chunk containing their start and
//     takes the remaining RU (RD) words from the next lane by warp shuffle
//     (consecutive lanes own consecutive chunks); RU is a template parameter,
//     so the realignment is register moves;
//   * left/right: the neighbouring lanes' edge words by shuffle (one scalar
//     load for lanes 0 / 31);
//   * row structure per word: column c = flat mod S and row = flat div S
//     (multiply-shift division by launch constants); column 0 takes the left
//     fill, the word holding pixel w-1 the right fill and the padding force,
//     pure padding words (uint64 rows) are forced to 1, and the first / last
//     row of every image take the vertical fill (bitimage.py:216-239);
//   * one aligned vector store of the chunk (output stride == input stride).
//
// Every load and store is an aligned 16/32-byte access; DRAM traffic stays one
// read of the input and one write of the output (up / centre / down rows of a
// chunk are the same lines other warps read: L2 hits).  Chunks near the first
// and last row (where a clamped vector load would not cover the words a
// straddling chunk needs) and the ragged last chunk reload their words one by
// one, bounded by the buffer.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "edge_reg.cuh"

namespace bitedge {

struct FlatParams {
    const uint32_t *in;      // CW*4-byte aligned
    uint32_t *o_edges;       // CW*4-byte aligned (or nullptr)
    uint32_t *o_eset;
    uint32_t nwords;         // nrows * S  (< 2^31)
    uint32_t S;              // row length == row stride, uint32 words (>= 2 * CW)
    uint32_t h;              // rows per image
    uint32_t nrows;
    int pl;                  // last pixel word (pixel order) holding a visible pixel
    uint32_t lastbit, padmask, fillword;
    uint32_t nchunks;        // ceil(nwords / CW)
    FastDiv div_s, div_h;
};

template <int CW>
__device__ __forceinline__ void flat_load(const uint32_t *p, uint32_t (&v)[CW]) {
    if constexpr (CW == 8) {
        asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                       "=r"(v[6]), "=r"(v[7])
                     : "l"(p));
    } else {
        const uint4 q = ldg_stream_v4(p);
        v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    }
}

// SWAP: uint64 words (pixel word p at uint32 index p ^ 1); chunks hold whole pairs.
//
// A warp owns 31 consecutive chunks; lane 31 holds the chunk after them (the next
// warp's first) only to feed the shuffles, so no lane reloads a neighbour's chunks and
// every load of the thread is issued before the first wait.  Every word is first
// evaluated as a word inside its row, inside its image (2 funnel shifts + 2 logic
// ops); only chunks holding column 0, the last pixel word or padding words redo those
// words with the row structure, and chunks in an image's first row or last two rows
// redo all of theirs -- before this split every word paid for the row tests (43
// thread instructions per word at 8192x8000 against the aligned K1's 21).
#ifndef K1F_MINB
#define K1F_MINB 5
#endif
//
// P4: the words are PBM P4 payload bytes (rows of whole 4-byte words; 1 = black,
// MSB-first bytes: the byte-reversed, inverted pixel-order word).  The plain path
// stays in the P4 domain as K1's P4 variant does -- only the two horizontal shifts
// run in pixel order: out = c & ~(pi(L & R) & u & d) -- and the row-structure words
// convert to the white pixel-order domain and back.
template <int CW, int SWAP, int RU, int OUT, bool P4 = false>
__global__ void __launch_bounds__(kThreads, CW == 8 ? (OUT == kOutAny ? 4 : K1F_MINB) : 0)
edge_flat_kernel(const __grid_constant__ FlatParams p) {
    static_assert(RU > 0 && RU < CW && (!SWAP || RU % 2 == 0), "phase");
    static_assert(!P4 || (SWAP == 0 && OUT == kOutEdges), "P4: uint32 rows, edges only");
    constexpr int RD = CW - RU;                       // S mod CW
    constexpr int LCW = CW == 8 ? 3 : 2;
    pdl_wait();
    pdl_trigger();
    const int lane = threadIdx.x & 31;
    const uint32_t t = (blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5)) * 31 + lane;
    const bool live = lane < 31 && t < p.nchunks;
    const uint32_t q = t < p.nchunks ? t : p.nchunks - 1;   // dead lanes mirror the last chunk
    const int base = (int)(q * CW);                   // nwords <= 2^30: 32-bit word offsets
    const int S = (int)p.S, nw = (int)p.nwords;
    const int full = nw >> LCW;                       // chunks entirely inside the buffer
    auto chunk_at = [&](int w0, uint32_t (&v)[CW]) {  // clamped aligned chunk
        const int c = min(max(w0 >> LCW, 0), full - 1);
        flat_load<CW>(p.in + (size_t)c * CW, v);
    };

    // ---- loads: up (aligned part + next lane), centre, down (aligned part + next lane)
    uint32_t u0[CW], cm[CW], d0[CW];
    chunk_at(base - S - RU, u0);                      // multiples of CW
    chunk_at(base, cm);
    chunk_at(base + S - RD, d0);
    // the pixel word before the warp's chunks: memory word base-1 (u32) / base-2 (u64 pair)
    uint32_t lwm = 0u;
    if (lane == 0 && base >= 1 + SWAP) lwm = __ldg(p.in + base - 1 - SWAP);

    // up[j] = flat word base - S + j (memory order) = (u0 ++ next lane's u0)[RU + j]
    uint32_t up[CW], dw[CW];
#pragma unroll
    for (int j = 0; j < CW; ++j) {
        if (j + RU < CW) up[j] = u0[j + RU];
        else up[j] = __shfl_down_sync(0xFFFFFFFFu, u0[j + RU - CW], 1);
        if (j + RD < CW) dw[j] = d0[j + RD];
        else dw[j] = __shfl_down_sync(0xFFFFFFFFu, d0[j + RD - CW], 1);
    }

    // ---- chunks whose clamped vector loads may not cover what they need: the first
    // and last two rows' worth of chunks and the ragged tail -- reload word by word,
    // all loads in flight at once (an out-of-line word loop left the main path 1.5 %
    // faster at 32768x32000 and the slowest warp, hence a 16 MB raster, 25 % slower)
    const bool edge_zone = base < S + 2 * CW || base + S + 2 * CW > nw || base + CW > nw;
    if (edge_zone) {
#pragma unroll
        for (int j = 0; j < CW; ++j) {
            const int f = base + j;
            cm[j] = f < nw ? __ldg(p.in + f) : 0u;
            up[j] = f - S >= 0 && f - S < nw ? __ldg(p.in + f - S) : 0u;
            dw[j] = f + S < nw ? __ldg(p.in + f + S) : 0u;
        }
    }

    // ---- pixel order (uint64 rows swap each pair) and horizontal neighbours
    uint32_t cc[CW], cu[CW], cd[CW];
#pragma unroll
    for (int j = 0; j < CW; ++j) {
        cc[j] = P4 ? p4_pi(cm[j]) : cm[j ^ SWAP];     // P4: pixel order, 1 = black
        cu[j] = up[j ^ SWAP];                         // P4: as loaded
        cd[j] = dw[j ^ SWAP];
    }
    // pixel-order word before the chunk: lane-1's last; after: lane+1's first
    uint32_t lw = __shfl_up_sync(0xFFFFFFFFu, cc[CW - 1], 1);
    uint32_t rw = __shfl_down_sync(0xFFFFFFFFu, cc[0], 1);
    if (lane == 0) lw = P4 ? p4_pi(lwm) : lwm;
    if (!live) return;
    if (edge_zone && base + CW >= nw) rw = 0u;        // the buffer's last chunk: nothing after it

    // ---- every word as a word inside its row, inside its image
    uint32_t ve[CW], vs[CW];
#pragma unroll
    for (int j = 0; j < CW; ++j) {
        const uint32_t left = j == 0 ? lw : cc[j - 1];
        const uint32_t right = j == CW - 1 ? rw : cc[j + 1];
        if (P4) {
            const uint32_t lr = __funnelshift_r(cc[j], left, 1) & __funnelshift_l(right, cc[j], 1);
            ve[j] = cm[j] & ~(p4_pi(lr) & cu[j] & cd[j]);
            vs[j] = 0u;
            continue;
        }
        const uint32_t a = __funnelshift_r(cc[j], left, 1) | __funnelshift_l(right, cc[j], 1) |
                           cu[j] | cd[j];
        ve[j ^ SWAP] = cc[j] | ~a;
        vs[j ^ SWAP] = ~cc[j] & a;
    }

    // ---- row / column of the chunk's first word; words past the row end wrap
    const uint32_t r0 = fdiv((uint32_t)base, p.div_s);
    const uint32_t c0 = (uint32_t)base - r0 * p.S;
    const uint32_t y0 = r0 - fdiv(r0, p.div_h) * p.h;
    const uint32_t fw = p.fillword;
    // word j with its row structure: column 0 takes the left fill, the word holding
    // pixel w-1 the right fill and the padding force, pure padding words are forced to
    // 1, the first / last row of every image take the vertical fill
    auto word = [&](int j) {
        uint32_t c = c0 + j, y = y0;
        if (c >= p.S) {                               // S >= 2 * CW: at most one wrap
            c -= p.S;
            y = (y0 + 1 == p.h) ? 0 : y0 + 1;
        }
        // white pixel-order domain (P4: centre / neighbours inverted, up / down converted)
        const uint32_t cw = P4 ? ~cc[j] : cc[j];
        const uint32_t left = P4 ? ~(j == 0 ? lw : cc[j - 1]) : (j == 0 ? lw : cc[j - 1]);
        const uint32_t right = P4 ? ~(j == CW - 1 ? rw : cc[j + 1]) : (j == CW - 1 ? rw : cc[j + 1]);
        const uint32_t ln = __funnelshift_r(cw, c == 0 ? fw : left, 1);
        uint32_t rn = __funnelshift_l(right, cw, 1);
        const uint32_t u = y == 0 ? fw : (P4 ? ~p4_pi(cu[j]) : cu[j]);
        const uint32_t d = y == p.h - 1 ? fw : (P4 ? ~p4_pi(cd[j]) : cd[j]);
        uint32_t f = 0u;
        if ((int)c == p.pl) {
            rn = (rn & ~p.lastbit) | (fw & p.lastbit);
            f = p.padmask;
        } else if ((int)c > p.pl) {
            f = 0xFFFFFFFFu;
        }
        const uint32_t a = ln | rn | u | d;
        ve[j ^ SWAP] = P4 ? p4_pi(~(cw | ~a | f)) : (cw | ~a | f);   // P4: 1 = black, padding 0
        vs[j ^ SWAP] = (~cw & a) | f;
    };
    if (y0 == 0 || y0 + 2 >= p.h) {
        // first row / last two rows of an image (a chunk may run on into the next row)
#pragma unroll
        for (int j = 0; j < CW; ++j) word(j);
    } else if (c0 == 0 || (int)(c0 + CW) > p.pl) {
        // column 0 at word 0, or the row's last pixel word .. the next row's column 0
        const int jlo = p.pl - (int)c0, jhi = S - (int)c0;
#pragma unroll
        for (int j = 0; j < CW; ++j)
            if ((j == 0 && c0 == 0) || (j >= jlo && j <= jhi)) word(j);
    }
    if (base + CW <= nw) {
        if (OUT != kOutEset) store_chunk<CW>(p.o_edges + base, ve);
        if (OUT != kOutEdges) store_chunk<CW>(p.o_eset + base, vs);
    } else {
#pragma unroll
        for (int j = 0; j < CW; ++j) {
            if (base + j < nw) {
                if (OUT != kOutEset) p.o_edges[base + j] = ve[j];
                if (OUT != kOutEdges) p.o_eset[base + j] = vs[j];
            }
        }
    }
}

// ---------------------------------------------------------------- K1s
// The same flat view, staged through a per-warp ring in shared memory so each
// input word crosses L2 about once (K1f reads the rows above and below every
// chunk again: 3x L2 reads, L2-throughput-bound).
//
// Warp g owns the output words [g * span, (g + 1) * span) of the flat array and
// streams the input words [start - S - 2, end + S + 2) (16-byte aligned) through
// a circular buffer of RW = 2^LR words indexed by flat word index mod RW, in
// pieces cut at multiples of SEGW words: piece k lands in slot k mod NSLOT with
// one `cp.async.bulk` (lane 0) and its own mbarrier.  Each step the warp
// produces 256 output words (4 pairs per lane, 64-bit stores) from the ring: the
// centre pair, the pairs S words before / after it and the two neighbour words
// are shared-memory loads at any word offset; the row structure per word is as
// in K1f.  Before a step, the pieces it reads are waited for; then every piece
// whose slot's previous piece no later step reads is issued, so up to
// NSLOT - (pieces one step reads) pieces are in flight per warp.
struct FlatRingParams {
    const uint32_t *in;      // 16-byte aligned
    uint32_t *o_edges;       // 8-byte aligned (or nullptr)
    uint32_t *o_eset;
    uint32_t nwords;         // nrows * S, a multiple of 4, < 2^31
    uint32_t S, h;
    int pl;
    uint32_t lastbit, padmask, fillword;
    uint32_t span;           // output words per warp, a multiple of 256
    uint32_t nwarps;
    FastDiv div_s, div_h;
};

constexpr int kRingSegW = 256;                        // words per piece / slot

template <int SWAP, int OUT, int LR>
__global__ void __launch_bounds__(kThreads)
edge_flat_ring_kernel(const FlatRingParams p) {
    constexpr int RW = 1 << LR, MASK = RW - 1;
    constexpr int NSLOT = RW / kRingSegW;
    constexpr int WARPS = kThreads / 32;
    extern __shared__ __align__(128) uint32_t k1s_smem[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t *ring = k1s_smem + (size_t)wid * RW;
    uint64_t *bars = reinterpret_cast<uint64_t *>(k1s_smem + (size_t)WARPS * RW) + wid * NSLOT;
    if (lane == 0) {
        for (int i = 0; i < NSLOT; ++i) wbar_init(&bars[i]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    pdl_wait();
    pdl_trigger();
    const uint32_t gw = blockIdx.x * WARPS + wid;
    if (gw >= p.nwarps) return;                       // whole warp, no CTA barriers
    const int64_t S = p.S, nw = p.nwords;
    const int64_t o0 = (int64_t)gw * p.span;
    if (o0 >= nw) return;
    const int64_t o1 = o0 + p.span < nw ? o0 + p.span : nw;
    // input words this warp stages (16-byte granules; the buffer ends clamp)
    int64_t i0 = o0 - S - 2;
    i0 = i0 < 0 ? 0 : (i0 & ~(int64_t)3);
    int64_t i1 = (o1 + S + 2 + 3) & ~(int64_t)3;
    i1 = i1 > nw ? nw : i1;
    const int64_t k0 = i0 / kRingSegW, klast = (i1 - 1) / kRingSegW;
    int64_t issued = k0, ready = k0;                  // next piece to issue / to wait for
    auto issue_upto = [&](int64_t kend) {             // lane 0: pieces [issued, kend]
        if (kend > klast) kend = klast;
        if (issued <= kend) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (; issued <= kend; ++issued) {
            const int64_t a = issued * kRingSegW > i0 ? issued * kRingSegW : i0;
            const int64_t b = (issued + 1) * kRingSegW < i1 ? (issued + 1) * kRingSegW : i1;
            uint64_t *bar = &bars[issued % NSLOT];
            wbar_expect(bar, (uint32_t)(b - a) * 4u);
            wtma(ring + (a & MASK), p.in + a, (uint32_t)(b - a) * 4u, bar);
        }
    };
    if (lane == 0) issue_upto(k0 + NSLOT - 1);

    const uint32_t fw = p.fillword;
    const uint32_t h = p.h;
    const uint32_t S32 = p.S;
    // a step = 256 output words = 4 pairs per lane (pair q of lane l: words
    // f0 + 64q + 2l, +1 -- every shared-memory load of the warp is contiguous)
    for (int64_t f0 = o0; f0 < o1; f0 += 256) {
        int64_t need = (f0 + 255 + S + 2) / kRingSegW;
        need = need > klast ? klast : need;
        for (; ready <= need; ++ready)
            wbar_wait(&bars[ready % NSLOT], (uint32_t)(((ready - k0) / NSLOT) & 1));
        uint32_t c[4][2], u[4][2], d[4][2], lw[4], rw[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t f = f0 + 64 * q + 2 * lane;
            const uint2 m = *reinterpret_cast<const uint2 *>(ring + (f & MASK));
            c[q][0] = SWAP ? m.y : m.x;
            c[q][1] = SWAP ? m.x : m.y;
            uint32_t a0, a1, b0, b1;
            if ((S & 1) == 0) {                       // pairs stay 8-byte aligned
                const uint2 mu = *reinterpret_cast<const uint2 *>(ring + ((f - S) & MASK));
                const uint2 md = *reinterpret_cast<const uint2 *>(ring + ((f + S) & MASK));
                a0 = mu.x; a1 = mu.y; b0 = md.x; b1 = md.y;
            } else {
                a0 = ring[(f - S) & MASK]; a1 = ring[(f - S + 1) & MASK];
                b0 = ring[(f + S) & MASK]; b1 = ring[(f + S + 1) & MASK];
            }
            u[q][0] = SWAP ? a1 : a0; u[q][1] = SWAP ? a0 : a1;
            d[q][0] = SWAP ? b1 : b0; d[q][1] = SWAP ? b0 : b1;
            lw[q] = ring[(f - 1 - SWAP) & MASK];      // pixel word f - 1
            rw[q] = ring[(f + 2 + SWAP) & MASK];      // pixel word f + 2
        }
        // every lane has read this step's words: slots behind the next step's
        // lowest word are free
        __syncwarp();
        if (lane == 0) {
            const int64_t lo_next = f0 + 256 - S - 2;
            const int64_t kmin = lo_next <= i0 ? k0 : lo_next / kRingSegW;
            issue_upto(kmin + NSLOT - 1);
        }
        // row / column of the first pair; +64 words per pair (S >= 64: one wrap)
        const uint32_t fa = (uint32_t)(f0 + 2 * lane);
        const uint32_t r0 = fdiv(fa, p.div_s);
        uint32_t col = fa - r0 * S32;
        uint32_t y = r0 - fdiv(r0, p.div_h) * h;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t f = f0 + 64 * q + 2 * lane;
            if (q > 0) {
                col += 64;
                if (col >= S32) {
                    col -= S32;
                    y = y + 1 == h ? 0 : y + 1;
                }
            }
            uint32_t ve[2], vs[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                uint32_t cj = col + j, yj = y;
                if (j == 1 && cj == S32) {            // u32 rows of odd length: f + 1 wraps
                    cj = 0;
                    yj = y + 1 == h ? 0 : y + 1;
                }
                const uint32_t left = j == 0 ? lw[q] : c[q][0];
                const uint32_t right = j == 1 ? rw[q] : c[q][1];
                const uint32_t ln = __funnelshift_r(c[q][j], cj == 0 ? fw : left, 1);
                uint32_t rn = __funnelshift_l(right, c[q][j], 1);
                const uint32_t uu = yj == 0 ? fw : u[q][j];
                const uint32_t dd = yj == h - 1 ? fw : d[q][j];
                uint32_t force = 0u;
                if ((int)cj == p.pl) {
                    rn = (rn & ~p.lastbit) | (fw & p.lastbit);
                    force = p.padmask;
                } else if ((int)cj > p.pl) {
                    force = 0xFFFFFFFFu;
                }
                const uint32_t any = ln | rn | uu | dd;
                ve[j ^ SWAP] = c[q][j] | ~any | force;
                vs[j ^ SWAP] = (~c[q][j] & any) | force;
            }
            if (f < o1) {
                if (OUT != kOutEset)
                    __stcs(reinterpret_cast<uint2 *>(p.o_edges + f), make_uint2(ve[0], ve[1]));
                if (OUT != kOutEdges)
                    __stcs(reinterpret_cast<uint2 *>(p.o_eset + f), make_uint2(vs[0], vs[1]));
            }
        }
    }
}

}  // namespace bitedge

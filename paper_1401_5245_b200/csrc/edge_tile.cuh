// edge_tile.cuh -- the fused method-of-masks tile kernel (K1/K2/K3 of SURVEY.md 2.2).
//
// One CTA owns a tile of R rows x TQ pixel-order uint32 words of the global
// row space (all n*h rows of a batch, or one row slab).  It stages rows
// g0-1 .. g0+R (the tile plus a 1-row halo above and below) and one halo word
// left and right into shared memory as pixel-order words -- loading packed
// words with 128-bit loads, or loading uint8 pixels with 128-bit loads and
// packing 16 bytes -> 16 bits in registers (BitImage.from_array,
// bitimage.py:122-136) -- then every output word is a single pass of
//
//     Ln = funnelshift_r(c, left, 1)     shift RIGHT plane   (bitimage.py:224-229)
//     Rn = funnelshift_l(right, c, 1)    shift LEFT plane    (bitimage.py:230-239)
//     Un / Dn = rows above / below       shift DOWN / UP     (bitimage.py:216-223)
//     edges   = c | ~(Ln | Rn | Un | Dn)  = NOT(OR_s (shift_s & ~c))
//     edgeset = ~c & (Ln | Rn | Un | Dn)
//
// with the border fill entering at pixel 0 (Ln), at pixel w-1 (Rn; not at the
// word LSB, bitimage.py:234-239), and at the first/last row of every image
// (Un/Dn), and every padding bit of every output forced to 1.
//
// Pixel-order words: a uint32 row is already in pixel order; a uint64 row
// (the reference's BitImage.words) holds its left 32 pixels in the HIGH half,
// i.e. at the odd uint32 address on little-endian, so pixel word p lives at
// uint32 index p ^ 1.  The loader swaps halves, so compute is format-blind.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace bitedge {

constexpr int kThreads = 256;

enum LoadKind : int {
    kPackedVec = 0,    // packed words, 128-bit loads (16-B aligned rows)
    kPackedScalar = 1, // packed words, 32-bit loads
    kU8Vec = 2,        // uint8 pixels, 128-bit loads
    kU8Byte = 3,       // uint8 pixels, byte loads (unaligned rows)
};

struct TileParams {
    const void *in;        // packed words or uint8 pixels
    const void *above;     // halo row -1 (or nullptr)
    const void *below;     // halo row `nrows` (or nullptr)
    int64_t in_stride;     // uint32 units (packed) or bytes (uint8)
    uint32_t *o_edges;
    uint32_t *o_eset;
    uint32_t *o_side[4];   // LEFT, RIGHT, UP, DOWN fundamental edges
    uint32_t *o_packed;
    int64_t out_stride;    // uint32 units
    int64_t nrows;         // rows in the global row space (n * h)
    int64_t h;             // rows per image
    int64_t w;             // pixels per row
    int64_t row_lo, row_hi;
    int wp;                // storage uint32 words per row (2*ceil(w/64) for u64)
    int pl;                // pixel word holding pixel w-1
    uint32_t lastbit;      // bit of pixel w-1 inside word pl
    uint32_t padmask;      // padding bits inside word pl
    uint32_t fillword;     // 0 or ~0
    int swap;              // 1 for uint64 storage
    int log_tq, log_r;     // tile = (1<<log_r) rows x (1<<log_tq) words
    int tiles_x;
};

__device__ __forceinline__ uint4 ldg_stream_v4(const void *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ uint32_t ldg_u32(const uint32_t *p) { return __ldg(p); }

// Nonzero-byte flags: bit 7 of each byte set iff the byte is nonzero.
__device__ __forceinline__ uint32_t nz_bytes(uint32_t v) {
    return (((v & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | v) & 0x80808080u;
}

// 8 bytes (a = pixels 0..3, b = pixels 4..7, little-endian: pixel 0 is the low
// byte) -> 8 bits MSB-first.  The flags of `a` sit at bits 4,12,20,28 and of
// `b` at 0,8,16,24; one 32x32->64 multiply by 2^31+2^22+2^13+2^4 moves them to
// bits 35..28 in pixel order with no two partial products colliding.
__device__ __forceinline__ uint32_t pack8(uint32_t a, uint32_t b) {
    uint32_t t = (nz_bytes(a) >> 3) | (nz_bytes(b) >> 7);
    uint64_t prod = (uint64_t)t * 0x80402010ull;
    return (uint32_t)(prod >> 28) & 0xFFu;
}

__device__ __forceinline__ uint32_t pack16(uint4 v) {
    return (pack8(v.x, v.y) << 8) | pack8(v.z, v.w);
}

// Byte-wise pack of pixels [x0, x0+16) of a row, pixels >= w read as white.
__device__ __forceinline__ uint32_t pack16_bytes(const uint8_t *row, int64_t x0, int64_t w) {
    uint32_t v = 0;
#pragma unroll
    for (int b = 0; b < 16; ++b) {
        int64_t x = x0 + b;
        uint32_t bit = 1u;
        if (x < w) bit = row[x] != 0;
        v = (v << 1) | bit;
    }
    return v;
}

template <int KIND>
__device__ __forceinline__ const void *row_ptr(const TileParams &p, int64_t g) {
    const int64_t elem = (KIND == kU8Vec || KIND == kU8Byte) ? 1 : 4;
    if (g >= 0 && g < p.nrows)
        return (const char *)p.in + g * p.in_stride * elem;
    if (g == -1) return p.above;
    if (g == p.nrows) return p.below;
    return nullptr;
}

template <int KIND>
__global__ void __launch_bounds__(kThreads)
edge_tile_kernel(const TileParams p) {
    extern __shared__ __align__(16) uint32_t smem[];
    const int TQ = 1 << p.log_tq;
    const int R = 1 << p.log_r;
    const int P = TQ + 8;                    // row pitch; interior starts at column 4
    uint8_t *flags = reinterpret_cast<uint8_t *>(smem + (R + 2) * P);
    const int tid = threadIdx.x;

    const int64_t tile = blockIdx.x;
    const int tx = (int)(tile % p.tiles_x);
    const int64_t g0 = p.row_lo + (tile / p.tiles_x) * (int64_t)R;
    const int q0 = tx * TQ;

    // ---- stage rows g0-1 .. g0+R into shared memory as pixel-order words ----
    // Halo words left (q0-1) and right (q0+TQ) of every staged row.  They exist
    // only when a row spans several column tiles (then TQ = 64 and R <= 64, so
    // one item per thread); otherwise both lie outside the row and hold the fill.
    const bool multi_col = p.tiles_x > 1;
    uint32_t halo_v = p.fillword;
    if (multi_col && tid < 2 * (R + 2)) {
        const int i = tid >> 1, right = tid & 1;
        const int pw = right ? q0 + TQ : q0 - 1;
        if (pw >= 0 && pw < p.wp) {
            if (KIND == kPackedVec || KIND == kPackedScalar) {
                const uint32_t *row = (const uint32_t *)row_ptr<KIND>(p, g0 - 1 + i);
                if (row != nullptr) halo_v = ldg_u32(row + (pw ^ p.swap));
            } else {
                // only the pixel adjacent to the tile matters: load that 16-pixel piece
                const uint8_t *row = (const uint8_t *)row_ptr<KIND>(p, g0 - 1 + i);
                const int64_t x0 = (int64_t)pw * 32 + (right ? 0 : 16);
                if (row != nullptr && x0 < p.w) {
                    const uint32_t half = pack16_bytes(row, x0, p.w);
                    halo_v = right ? (half << 16) : half;
                }
            }
        }
    }
    // Interior: batches of U loads are issued back to back before any result is
    // consumed, so every thread keeps U 16-byte requests in flight.
    constexpr int U = 8;
    if (KIND == kPackedVec) {
        const int log_ch = p.log_tq - 2;
        const int CH = 1 << log_ch;
        const int total = (R + 2) * CH;
        for (int base = tid; base < total; base += U * kThreads) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int idx = base + u * kThreads;
                v[u] = make_uint4(0u, 0u, 0u, 0u);
                if (idx < total) {
                    const int i = idx >> log_ch, pw = q0 + 4 * (idx & (CH - 1));
                    const uint32_t *row = (const uint32_t *)row_ptr<KIND>(p, g0 - 1 + i);
                    if (row != nullptr && pw < p.wp) v[u] = ldg_stream_v4(row + pw);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int idx = base + u * kThreads;
                if (idx < total) {
                    const int i = idx >> log_ch, c = idx & (CH - 1);
                    uint4 x = v[u];
                    if (p.swap) x = make_uint4(x.y, x.x, x.w, x.z);
                    *reinterpret_cast<uint4 *>(smem + i * P + 4 + 4 * c) = x;
                }
            }
        }
    } else if (KIND == kPackedScalar) {
        const int total = (R + 2) * TQ;
        for (int base = tid; base < total; base += U * kThreads) {
            uint32_t v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int idx = base + u * kThreads;
                v[u] = 0u;
                if (idx < total) {
                    const int i = idx >> p.log_tq, pw = q0 + (idx & (TQ - 1));
                    const uint32_t *row = (const uint32_t *)row_ptr<KIND>(p, g0 - 1 + i);
                    if (row != nullptr && pw < p.wp) v[u] = ldg_u32(row + (pw ^ p.swap));
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int idx = base + u * kThreads;
                if (idx < total) smem[(idx >> p.log_tq) * P + 4 + (idx & (TQ - 1))] = v[u];
            }
        }
    } else {
        // uint8 pixels: piece k of a tile row = 16 pixels = one half of word k/2;
        // a word's high half (u16 index 2*word+1) holds its left 16 pixels.
        uint16_t *sm16 = reinterpret_cast<uint16_t *>(smem);
        const int log_npc = p.log_tq + 1;
        const int NPC = 1 << log_npc;
        const int total = (R + 2) * NPC;
        if (KIND == kU8Vec) {
            for (int base = tid; base < total; base += U * kThreads) {
                uint4 v[U];
                uint32_t st[U];   // 0: vector piece, 1: partial (byte path), 2: outside
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int idx = base + u * kThreads;
                    st[u] = 2;
                    if (idx < total) {
                        const int i = idx >> log_npc, k = idx & (NPC - 1);
                        const int64_t x0 = (int64_t)(q0 + (k >> 1)) * 32 + (k & 1) * 16;
                        const uint8_t *row = (const uint8_t *)row_ptr<KIND>(p, g0 - 1 + i);
                        if (row != nullptr && x0 < p.w) {
                            if (x0 + 16 <= p.w) {
                                v[u] = ldg_stream_v4(row + x0);
                                st[u] = 0;
                            } else {
                                st[u] = 1;
                            }
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int idx = base + u * kThreads;
                    if (idx < total) {
                        const int i = idx >> log_npc, k = idx & (NPC - 1);
                        uint32_t half = 0xFFFFu;
                        if (st[u] == 0) {
                            half = pack16(v[u]);
                        } else if (st[u] == 1) {
                            const int64_t x0 = (int64_t)(q0 + (k >> 1)) * 32 + (k & 1) * 16;
                            half = pack16_bytes((const uint8_t *)row_ptr<KIND>(p, g0 - 1 + i),
                                                x0, p.w);
                        }
                        sm16[2 * (i * P + 4 + (k >> 1)) + ((k & 1) ? 0 : 1)] = (uint16_t)half;
                    }
                }
            }
        } else {
            for (int idx = tid; idx < total; idx += kThreads) {
                const int i = idx >> log_npc, k = idx & (NPC - 1);
                const int64_t x0 = (int64_t)(q0 + (k >> 1)) * 32 + (k & 1) * 16;
                const uint8_t *row = (const uint8_t *)row_ptr<KIND>(p, g0 - 1 + i);
                uint32_t half = 0xFFFFu;
                if (row != nullptr && x0 < p.w) half = pack16_bytes(row, x0, p.w);
                sm16[2 * (i * P + 4 + (k >> 1)) + ((k & 1) ? 0 : 1)] = (uint16_t)half;
            }
        }
    }
    for (int idx = tid; idx < 2 * (R + 2); idx += kThreads) {
        const int i = idx >> 1, right = idx & 1;
        smem[i * P + 4 + (right ? TQ : -1)] = idx == tid ? halo_v : p.fillword;
    }
    // per-row border flags: bit0 -> row above is outside the image, bit1 -> below
    for (int i = tid; i < R; i += kThreads) {
        const int64_t g = g0 + i;
        uint8_t f = 0;
        if (g < p.row_hi) {
            const int64_t y = g % p.h;
            if (y == 0 && !(g == 0 && p.above != nullptr)) f |= 1;
            if (y == p.h - 1 && !(g == p.nrows - 1 && p.below != nullptr)) f |= 2;
        }
        flags[i] = f;
    }
    __syncthreads();

    // ---- one fused pass per output word ----
    const uint32_t fw = p.fillword;
    for (int idx = tid; idx < R * TQ; idx += kThreads) {
        const int i = idx >> p.log_tq, j = idx & (TQ - 1);
        const int64_t g = g0 + i;
        if (g >= p.row_hi) break;
        const int pw = q0 + j;
        if (pw >= p.wp) continue;
        const uint32_t *s = smem + (i + 1) * P + 4 + j;
        const uint32_t c = s[0];
        const uint32_t f = flags[i];
        const uint32_t u = (f & 1) ? fw : s[-P];
        const uint32_t d = (f & 2) ? fw : s[P];
        const uint32_t l = (pw == 0) ? fw : s[-1];
        const uint32_t r = s[1];
        const uint32_t ln = __funnelshift_r(c, l, 1);   // (c >> 1) | (l << 31)
        uint32_t rn = __funnelshift_l(r, c, 1);         // (c << 1) | (r >> 31)
        uint32_t pad = 0u, dead = 0u;
        if (pw >= p.pl) {
            if (pw == p.pl) {
                rn = (rn & ~p.lastbit) | (fw & p.lastbit);  // pixel w-1 reads the fill
                pad = p.padmask;
            } else {
                dead = ~0u;                                  // all-padding word
            }
        }
        const uint32_t any = ln | rn | u | d;
        const int64_t o = g * p.out_stride + (pw ^ p.swap);
        const uint32_t force = pad | dead;
        if (p.o_edges) p.o_edges[o] = c | ~any | force;
        if (p.o_eset) p.o_eset[o] = (~c & any) | force;
        if (p.o_side[0]) p.o_side[0][o] = (ln & ~c) | force;
        if (p.o_side[1]) p.o_side[1][o] = (rn & ~c) | force;
        if (p.o_side[2]) p.o_side[2][o] = (u & ~c) | force;
        if (p.o_side[3]) p.o_side[3][o] = (d & ~c) | force;
        if (p.o_packed) p.o_packed[o] = c | force;
    }
}

}  // namespace bitedge

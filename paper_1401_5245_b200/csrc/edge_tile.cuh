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
    kP32Vec = 0,       // uint32 row words, 128-bit loads (16-B aligned rows)
    kP64Vec = 1,       // uint64 row words, 128-bit loads, halves swapped into pixel order
    kPScalar = 2,      // packed words of either format, 32-bit loads
    kU8Vec = 3,        // uint8 pixels, 128-bit loads
    kU8Byte = 4,       // uint8 pixels, byte loads (unaligned rows)
};

enum OutKind : int {
    kOutEdges = 0,     // detect_edges_mask only (the hot path)
    kOutEset = 1,      // EdgeSet only
    kOutAny = 2,       // any subset of the optional outputs
    kOutAll = 3,       // register kernels: edges / EdgeSet / 4 sides / packed, each if non-null
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
    int thr;               // uint8 pack: white iff sample >= thr (1 = from_array)
};

__device__ __forceinline__ uint4 ldg_stream_v4(const void *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ uint32_t ldg_u32(const uint32_t *p) { return __ldg(p); }

// Programmatic dependent launch (no-ops unless launched with the PDL attribute):
// wait until the previous grid on the stream has completed and its writes are
// visible, and let the next grid start launching once this CTA's work is issued.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Pixel rule of the uint8 -> bit pack: white iff sample >= t.  t = 1 is
// BitImage.from_array's "nonzero = white" (bitimage.py:124,133); any other t is
// binarize.threshold ("sample >= t -> White"), fused into the
// edge kernels as SURVEY 8(f) F2.
struct Thr {
    uint32_t t;     // threshold 0..255
    uint32_t tl;    // (t & 0x7f) replicated into every byte
    uint32_t m;     // ~0 when t < 128, else 0
};

__device__ __forceinline__ Thr make_thr(int t) {
    Thr T;
    T.t = (uint32_t)t;
    T.tl = ((uint32_t)t & 0x7Fu) * 0x01010101u;
    T.m = t < 128 ? 0xFFFFFFFFu : 0u;
    return T;
}

// Bit 7 of each byte set iff byte >= t: with b = 128*bh + bl, bl >= tl is the
// no-borrow bit of ((bl | 0x80) - tl); then ge = bh | that (t < 128) or
// bh & that (t >= 128), one LOP3 either way.  For t = 1 this is "byte != 0".
__device__ __forceinline__ uint32_t ge_bytes(uint32_t v, const Thr &T) {
    const uint32_t x = (v | 0x80808080u) - T.tl;     // == ((v & 0x7F..) | 0x80..) - tl
    return ((v & x) | (T.m & (v | x))) & 0x80808080u;
}

// 8 bytes (a = pixels 0..3, b = pixels 4..7, little-endian: pixel 0 is the low
// byte) -> 8 bits MSB-first.  The flags of `a` sit at bits 4,12,20,28 and of
// `b` at 0,8,16,24; one 32x32->64 multiply by 2^31+2^22+2^13+2^4 moves them to
// bits 35..28 in pixel order with no two partial products colliding.
__device__ __forceinline__ uint32_t pack8(uint32_t a, uint32_t b, const Thr &T) {
    uint32_t t = (ge_bytes(a, T) >> 3) | (ge_bytes(b, T) >> 7);
    uint64_t prod = (uint64_t)t * 0x80402010ull;
    return (uint32_t)(prod >> 28) & 0xFFu;
}

__device__ __forceinline__ uint32_t pack16(uint4 v, const Thr &T) {
    return (pack8(v.x, v.y, T) << 8) | pack8(v.z, v.w, T);
}

// Byte-wise pack of pixels [x0, x0+16) of a row, pixels >= w read as white.
__device__ __forceinline__ uint32_t pack16_bytes(const uint8_t *row, int64_t x0, int64_t w,
                                                 const Thr &T) {
    uint32_t v = 0;
#pragma unroll
    for (int b = 0; b < 16; ++b) {
        int64_t x = x0 + b;
        uint32_t bit = 1u;
        if (x < w) bit = row[x] >= T.t;
        v = (v << 1) | bit;
    }
    return v;
}


// Pointer to global row g of the staged range, or nullptr when that row does
// not exist (outside the raster with no halo buffer).
template <int KIND>
__device__ __forceinline__ const char *row_ptr(const TileParams &p, int64_t g) {
    constexpr int64_t elem = (KIND == kU8Vec || KIND == kU8Byte) ? 1 : 4;
    if (g >= 0 && g < p.nrows) return (const char *)p.in + g * p.in_stride * elem;
    if (g == -1) return (const char *)p.above;
    if (g == p.nrows) return (const char *)p.below;
    return nullptr;
}

// Stage one 4-word chunk / 16-pixel piece of a row into shared memory.
template <int KIND>
__device__ __forceinline__ void stage_item(uint32_t *srow, const char *row, int c, int pw0,
                                           int64_t x0, const TileParams &p) {
    if (KIND == kP32Vec || KIND == kP64Vec) {
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (row != nullptr && pw0 < p.wp) v = ldg_stream_v4((const uint32_t *)row + pw0);
        if (KIND == kP64Vec) v = make_uint4(v.y, v.x, v.w, v.z);
        *reinterpret_cast<uint4 *>(srow + 4 * c) = v;
    } else if (KIND == kPScalar) {
        uint32_t v = 0u;
        if (row != nullptr && pw0 < p.wp) v = ldg_u32((const uint32_t *)row + (pw0 ^ p.swap));
        srow[c] = v;
    } else {
        uint32_t half = 0xFFFFu;
        if (row != nullptr && x0 < p.w) {
            const Thr T = make_thr(p.thr);
            if (KIND == kU8Vec && x0 + 16 <= p.w) half = pack16(ldg_stream_v4(row + x0), T);
            else half = pack16_bytes((const uint8_t *)row, x0, p.w, T);
        }
        reinterpret_cast<uint16_t *>(srow)[2 * (c >> 1) + ((c & 1) ? 0 : 1)] = (uint16_t)half;
    }
}

template <int KIND, int OUT>
__global__ void __launch_bounds__(kThreads)
edge_tile_kernel(const TileParams p) {
    extern __shared__ __align__(16) uint32_t smem[];
    const Thr T = make_thr(p.thr);
    constexpr bool U8 = (KIND == kU8Vec || KIND == kU8Byte);
    const int log_tq = p.log_tq;
    const int TQ = 1 << log_tq;
    const int R = 1 << p.log_r;
    const int P = TQ + 8;                    // row pitch; interior starts at column 4
    uint8_t *flags = reinterpret_cast<uint8_t *>(smem + (R + 2) * P);
    const int tid = threadIdx.x;

    const int tx = (int)(blockIdx.x % (unsigned)p.tiles_x);
    const int64_t g0 = p.row_lo + (int64_t)(blockIdx.x / (unsigned)p.tiles_x) * R;
    const int q0 = tx * TQ;

    // ---- stage rows g0-1 .. g0+R (smem rows 0 .. R+1) as pixel-order words ----
    // Items per staged row: 4-word chunks (packed, vector), words (scalar) or
    // 16-pixel pieces (uint8).  The item count divides the thread count, so a
    // thread keeps the same column item for every row it stages.
    const int log_items = (KIND == kP32Vec || KIND == kP64Vec) ? log_tq - 2
                          : (U8 ? log_tq + 1 : log_tq);
    const int items = 1 << log_items;
    const int c = tid & (items - 1);
    const int rstep = kThreads >> log_items;          // staged rows per pass
    const int pw0 = (KIND == kP32Vec || KIND == kP64Vec) ? q0 + 4 * c : q0 + c;
    const int64_t x0 = (int64_t)q0 * 32 + 16 * c;     // uint8: first pixel of the piece
    {
        // main rows (smem 1..R): global rows g0 .. g0+R-1, all inside `in`
        const int nvalid = (int)min((int64_t)R, p.nrows - g0);
        const int64_t rs = p.in_stride * (U8 ? 1 : 4);             // bytes per row
        const char *base = (const char *)p.in + g0 * rs;
        // staged main row r: inside the raster, or -- for a partial last tile of a
        // slab -- the halo row below the slab (global row nrows), or nothing
        auto row_at = [&](int r) -> const char * {
            if (r < nvalid) return base + r * rs;
            if (r == nvalid && nvalid < R) return (const char *)p.below;
            return nullptr;
        };
        constexpr int U = 4;
        for (int r0 = tid >> log_items; r0 < R; r0 += U * rstep) {
            if (KIND == kP32Vec || KIND == kP64Vec || KIND == kU8Vec) {
                // issue up to U independent 16-byte loads before consuming any
                uint4 v[U];
                bool full[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int r = r0 + u * rstep;
                    full[u] = false;
                    v[u] = make_uint4(0u, 0u, 0u, 0u);
                    const char *row = r < R ? row_at(r) : nullptr;
                    if (row != nullptr) {
                        if (U8) {
                            if (x0 + 16 <= p.w) { v[u] = ldg_stream_v4(row + x0); full[u] = true; }
                        } else if (pw0 < p.wp) {
                            v[u] = ldg_stream_v4((const uint32_t *)row + pw0);
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int r = r0 + u * rstep;
                    if (r < R) {
                        uint32_t *srow = smem + (r + 1) * P + 4;
                        if (U8) {
                            uint32_t half = 0xFFFFu;
                            if (full[u]) half = pack16(v[u], T);
                            else if (row_at(r) != nullptr && x0 < p.w)
                                half = pack16_bytes((const uint8_t *)row_at(r), x0, p.w, T);
                            reinterpret_cast<uint16_t *>(srow)[2 * (c >> 1) + ((c & 1) ? 0 : 1)] =
                                (uint16_t)half;
                        } else {
                            uint4 x = v[u];
                            if (KIND == kP64Vec) x = make_uint4(x.y, x.x, x.w, x.z);
                            *reinterpret_cast<uint4 *>(srow + 4 * c) = x;
                        }
                    }
                }
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int r = r0 + u * rstep;
                    if (r < R)
                        stage_item<KIND>(smem + (r + 1) * P + 4, row_at(r), c, pw0, x0, p);
                }
            }
        }
        // halo rows: smem 0 = global g0-1, smem R+1 = global g0+R
        if (tid < 2 * items) {
            const int side = tid >> log_items;
            const int64_t g = side ? g0 + R : g0 - 1;
            stage_item<KIND>(smem + (side ? R + 1 : 0) * P + 4, row_ptr<KIND>(p, g), c, pw0, x0, p);
        }
    }
    // Column halo words (q0-1, q0+TQ) exist only when a row spans several
    // column tiles (then TQ = 64 and R <= 64: one item per thread); otherwise
    // they lie outside the row and hold the fill.
    if (tid < 2 * (R + 2)) {
        const int i = tid >> 1, right = tid & 1;
        const int pw = right ? q0 + TQ : q0 - 1;
        uint32_t v = p.fillword;
        if (p.tiles_x > 1 && pw >= 0 && pw < p.wp) {
            const char *row = row_ptr<KIND>(p, g0 - 1 + i);
            if (row != nullptr) {
                if (!U8) {
                    v = ldg_u32((const uint32_t *)row + (pw ^ p.swap));
                } else {
                    const int64_t hx = (int64_t)pw * 32 + (right ? 0 : 16);
                    if (hx < p.w) {
                        const uint32_t half = pack16_bytes((const uint8_t *)row, hx, p.w, T);
                        v = right ? (half << 16) : half;
                    }
                }
            }
        }
        smem[i * P + 4 + (right ? TQ : -1)] = v;
    } else {
        for (int idx = tid; idx < 2 * (R + 2); idx += kThreads)
            smem[(idx >> 1) * P + 4 + ((idx & 1) ? TQ : -1)] = p.fillword;
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
    // Thread -> fixed word column j, rows r, r + NG, ...; every per-column
    // quantity (border column, pixel w-1 fix, padding) is loop-invariant.
    const int j = tid & (TQ - 1);
    const int NG = kThreads >> log_tq;
    const int pw = q0 + j;
    if (pw >= p.wp) return;
    const uint32_t fw = p.fillword;
    const bool first_col = (pw == 0);
    uint32_t keep = 0xFFFFu | 0xFFFF0000u, fixb = 0u, force = 0u;
    if (pw == p.pl) {
        keep = ~p.lastbit;                 // pixel w-1 reads the fill (bitimage.py:234-239)
        fixb = fw & p.lastbit;
        force = p.padmask;
    } else if (pw > p.pl) {
        force = 0xFFFFFFFFu;               // all-padding word
    }
    const int rmax = (int)min((int64_t)R, p.row_hi - g0);
    const int64_t ostep = (int64_t)NG * p.out_stride;
    int64_t o = (g0 + (tid >> log_tq)) * p.out_stride + (pw ^ p.swap);
    const uint32_t *s = smem + ((tid >> log_tq) + 1) * P + 4 + j;
    const int sstep = NG * P;
    for (int r = tid >> log_tq; r < rmax; r += NG, s += sstep, o += ostep) {
        const uint32_t cc = s[0];
        const uint32_t f = flags[r];
        const uint32_t u = (f & 1) ? fw : s[-P];
        const uint32_t d = (f & 2) ? fw : s[P];
        const uint32_t l = first_col ? fw : s[-1];
        const uint32_t ln = __funnelshift_r(cc, l, 1);           // (c >> 1) | (l << 31)
        const uint32_t rn = (__funnelshift_l(s[1], cc, 1) & keep) | fixb;  // (c << 1) | (r >> 31)
        const uint32_t any = ln | rn | u | d;
        if (OUT == kOutEdges) {
            __stcs(p.o_edges + o, cc | ~any | force);
        } else if (OUT == kOutEset) {
            __stcs(p.o_eset + o, (~cc & any) | force);
        } else {
            if (p.o_edges) p.o_edges[o] = cc | ~any | force;
            if (p.o_eset) p.o_eset[o] = (~cc & any) | force;
            if (p.o_side[0]) p.o_side[0][o] = (ln & ~cc) | force;
            if (p.o_side[1]) p.o_side[1][o] = (rn & ~cc) | force;
            if (p.o_side[2]) p.o_side[2][o] = (u & ~cc) | force;
            if (p.o_side[3]) p.o_side[3][o] = (d & ~cc) | force;
            if (p.o_packed) p.o_packed[o] = cc | force;
        }
    }
}

}  // namespace bitedge

// capi_p4.cu -- PBM P4 payloads at the kernel boundary:
// decode / encode kernels and the fused P4 -> edges -> P4 path through K1.
#include "capi_internal.cuh"
#include "edge_reg.cuh"
#include "edge_flat.cuh"

using namespace bitedge;
using namespace bitedge::capi;

namespace bitedge {
namespace capi {

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

// P4 payloads of ANY width in one pass (F1 for rows that are not 16-byte
// multiples, e.g. the CLI's arbitrary PBM files): rows are ceil(w/8) bytes
// packed back to back, so a row starts at any byte.  Thread = one 32-pixel word
// of one row: it reads its (up to) 4 bytes of the row above, the row and the
// row below, plus the byte either side of its centre bytes for the horizontal
// neighbours -- byte loads, L1-cached, shared by the neighbouring threads --
// evaluates the edge formula in the white domain (exactly K1's, with the fill at
// pixel 0, pixel w-1 and every image's first / last row) and stores its bytes
// (P4 polarity, padding bits 0 as the encoder writes them).
__device__ __forceinline__ uint32_t p4_ld8(const uint8_t *p) {
    uint32_t v;
    asm volatile("ld.global.nc.u8 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ uint32_t p4_ld32(const uint8_t *p) {
    return __ldg(reinterpret_cast<const uint32_t *>(p));
}

// Little-endian 4 bytes of the payload at byte offset `off` (bytes at or past
// `total` read as 0).  With a 4-byte aligned payload: two aligned loads and a
// funnel shift; at the very end of the buffer, or for an unaligned payload,
// byte loads (never a byte outside [0, total)).
__device__ __forceinline__ uint32_t p4_get4(const uint8_t *in, int64_t off, int64_t total,
                                            bool al) {
    const int64_t a = off & ~(int64_t)3;
    if (al && a + 8 <= total)
        return __funnelshift_r(p4_ld32(in + a), p4_ld32(in + a + 4), (uint32_t)(off & 3) * 8);
    uint32_t v = 0u;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (off + k < total) v |= p4_ld8(in + off + k) << (8 * k);
    return v;
}

// Thread = one 32-pixel word column of a strip of R rows (rows walked with the
// up / centre / down words rolling in registers: one new row of 4 bytes per
// output row, plus the byte either side of the centre word for the horizontal
// neighbours), so the per-thread setup is paid once per R words.
template <int R>
__global__ void __launch_bounds__(256)
p4_edges_bytes_kernel(const uint8_t *__restrict__ in, uint8_t *__restrict__ out, WordGeom g,
                      int64_t rb, uint32_t nstrips, FastDiv dv_wp, FastDiv dv_h) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;    // < 2^32 (host check)
    const uint32_t strip = fdiv(t, dv_wp);
    if (strip >= nstrips) return;
    const int pw = (int)(t - strip * (uint32_t)g.wp);
    const int64_t nbytes = g.nrows * rb;
    const uint32_t fw = g.fillword;
    const bool al = ((uintptr_t)in & 3) == 0;
    const int64_t b0 = 4 * (int64_t)pw;
    const int nb = rb - b0 < 4 ? (int)(rb - b0) : 4;
    // bytes past the row (the next row's) read as black in P4 = white here:
    // they are padding positions, forced below
    const uint32_t keep = nb == 4 ? 0xFFFFFFFFu : ~(0xFFFFFFFFu >> (8 * nb));
    const bool tail = pw == g.pl, has_r = b0 + 4 < rb;
    const uint32_t r0 = strip * R;                               // < 2^32 (host check)
    uint32_t y = r0 - fdiv(r0, dv_h) * (uint32_t)g.h;
    int64_t off = (int64_t)r0 * rb + b0;
    // white-domain, pixel-order word of the 4 bytes at byte offset o
    auto word = [&](int64_t o) {
        return ~(__byte_perm(p4_get4(in, o, nbytes, al), 0, 0x0123) & keep);
    };
    uint32_t up = y == 0 ? fw : word(off - rb);
    uint32_t c = word(off);
#pragma unroll
    for (int i = 0; i < R; ++i) {
        if (r0 + i >= g.nrows) break;
        const bool last = y == (uint32_t)g.h - 1;
        const uint32_t nx = r0 + i + 1 < g.nrows ? word(off + rb) : fw;
        const uint32_t d = last ? fw : nx;
        // its bit 0: pixel 32*pw - 1 (last bit of the byte before); bit 31: pixel 32*pw + 32
        const uint32_t lw = pw > 0 ? ~p4_ld8(in + off - 1) : fw;
        const uint32_t rw = has_r ? ~(p4_ld8(in + off + 4) << 24) : fw;
        const uint32_t ln = __funnelshift_r(c, lw, 1);
        uint32_t rn = __funnelshift_l(rw, c, 1);
        uint32_t f = 0u;
        if (tail) {                               // pixel w-1 reads the fill; padding -> 1
            rn = (rn & ~g.lastbit) | (fw & g.lastbit);
            f = g.padmask;
        }
        const uint32_t e = ~(c | ~(ln | rn | up | d) | f);   // P4: 1 = black edge pixel
        uint8_t *o = out + off;
        if (nb == 4 && ((uintptr_t)o & 3) == 0) {
            *reinterpret_cast<uint32_t *>(o) = __byte_perm(e, 0, 0x0123);   // bytes in P4 order
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (k < nb) o[k] = (uint8_t)(e >> (24 - 8 * k));
        }
        up = last ? fw : c;                       // the next row starts a new image after `last`
        c = nx;
        y = last ? 0u : y + 1;
        off += rb;
    }
}

// K1p: P4 payloads whose rows are not whole 4-byte words, viewed -- like K1f --
// as ONE flat byte array (rows of rb bytes back to back): thread = one aligned
// chunk of CW words (32 bytes when the buffers are 32-byte aligned, else 16);
// the rows above / below are the bytes rb before / after, at a fixed byte phase
// from the chunk grid (RDW words + s bytes: RDW a template constant, s
// uniform), taken from the lane's own aligned chunk and the next lane's by
// funnel shifts; the neighbour pixels from the neighbouring lanes (a byte load
// at warp edges).  The output has the input's flat layout, so every store is
// one aligned vector store -- no row is ever written by two threads.
//
// Row boundaries fall inside words at byte granularity, but only in the one or
// two chunks per row that hold a row's first or last byte.  Every other chunk
// ("plain") is evaluated in the P4 domain as loaded (1 = black; AND / OR / NOT
// commute with the byte reversal, so only the two horizontal shifts run in
// pixel order): out = c & ~(pi(L & R) & u & d), ~10 instructions per word.  A
// chunk with a row boundary tests each of its words; the word holding a row's
// first / last byte gets its row structure as bit masks (first pixel of a row:
// left fill; pixel w-1: right fill; padding bits; top / bottom row of an image:
// vertical fill).  Before the split every word paid for the masks (~55
// instructions: issue-bound, 2.0 TB/s at 32000x32002).  Chunks within two rows
// of the buffer ends load byte by byte.
struct P4FlatParams {
    const uint8_t *in;       // 4*CW-byte aligned
    uint8_t *out;            // 4*CW-byte aligned
    uint32_t nbytes;         // nrows * rb < 2^31
    uint32_t rb, h, nchunks;
    uint32_t wlast;          // (w - 1) % 8: bit of pixel w-1 in its byte (MSB = 0)
    uint32_t fw;
    int s;                   // rb % 4 (byte part of the down phase)
    FastDiv div_rb, div_h;
};

__device__ __forceinline__ uint32_t p4w(uint32_t mem) {            // P4 LE word -> white, pixel order
    return ~__byte_perm(mem, 0, 0x0123);
}

// One word that holds a row's first and / or last byte, or lies in an image's top /
// bottom row: its row structure as bit masks, white domain.  cbj / left / right:
// black-domain pixel-order words (left: bit 0 = the pixel before, right: bit 31 = the
// pixel after); upm / dwm: the words rb bytes before / after, as loaded; jb: the byte
// of its row the word starts at; y: that row's index in its image.
__device__ __forceinline__ uint32_t p4_row_word(const P4FlatParams &p, uint32_t cbj, uint32_t left,
                                                uint32_t right, uint32_t upm, uint32_t dwm,
                                                uint32_t jb, uint32_t y) {
    const uint32_t fw = p.fw, hm1 = p.h - 1;
    const uint32_t eb = p.rb - jb;            // bytes left in the row from this word's byte 0
    const uint32_t y1 = y == hm1 ? 0u : y + 1;
    // bits of the bytes that belong to the next row (eb < 4)
    const uint32_t nxt = eb < 4 ? (0xFFFFFFFFu >> (8 * eb)) : 0u;
    uint32_t lfix = jb == 0 ? 0x80000000u : 0u;            // first pixel of a row
    if (eb < 4) lfix |= 0x80000000u >> (8 * eb);
    uint32_t rfix = 0u, pad = 0u;                          // pixel w-1 / padding of the row
    if (eb <= 4) {
        const uint32_t bit = 31 - 8 * (eb - 1) - p.wlast;  // pixel w-1
        rfix = 1u << bit;
        pad = (rfix - 1u) & (0xFFFFFFFFu >> (8 * (eb - 1))) & ~nxt;
    }
    const uint32_t umask = (y == 0 ? ~nxt : 0u) | (y1 == 0 ? nxt : 0u);
    const uint32_t dmask = (y == hm1 ? ~nxt : 0u) | (y1 == hm1 ? nxt : 0u);
    const uint32_t c = ~cbj;
    const uint32_t ln = (__funnelshift_r(c, ~left, 1) & ~lfix) | (fw & lfix);
    const uint32_t rn = (__funnelshift_l(~right, c, 1) & ~rfix) | (fw & rfix);
    const uint32_t u = (p4w(upm) & ~umask) | (fw & umask);
    const uint32_t d = (p4w(dwm) & ~dmask) | (fw & dmask);
    const uint32_t e = c | ~(ln | rn | u | d) | pad;      // white domain, padding 1
    return __byte_perm(~e, 0, 0x0123);                    // P4: 1 = black, padding 0
}

// A chunk near the buffer ends (where the clamped vector loads do not cover what it
// needs) or the ragged last chunk, word by word from byte loads; out of line.
__device__ __noinline__ void p4_flat_edge_chunk(const P4FlatParams &p, int base, int cw,
                                                uint32_t jb, uint32_t y) {
    const int rb = (int)p.rb, nb = (int)p.nbytes;
#pragma unroll 1
    for (int j = 0; j < cw; ++j) {
        const int b0 = base + 4 * j;
        if (b0 >= nb) break;
        if (j > 0) {
            jb += 4;
            while (jb >= p.rb) {
                jb -= p.rb;
                y = y == p.h - 1 ? 0u : y + 1;
            }
        }
        uint32_t c = 0u, uu = 0u, dd = 0u;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int b = b0 + k;
            if (b < nb) c |= (uint32_t)p.in[b] << (8 * k);
            if (b - rb >= 0 && b - rb < nb) uu |= (uint32_t)p.in[b - rb] << (8 * k);
            if (b + rb < nb) dd |= (uint32_t)p.in[b + rb] << (8 * k);
        }
        const uint32_t left = b0 > 0 ? (uint32_t)p.in[b0 - 1] : 0u;
        const uint32_t right = b0 + 4 < nb ? (uint32_t)p.in[b0 + 4] << 24 : 0u;
        const uint32_t o = p4_row_word(p, __byte_perm(c, 0, 0x0123), left, right, uu, dd, jb, y);
        if (b0 + 4 <= nb) {
            *reinterpret_cast<uint32_t *>(p.out + b0) = o;
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (b0 + k < nb) p.out[b0 + k] = (uint8_t)(o >> (8 * k));
        }
    }
}

template <int CW, int RDW, bool EDGE_INLINE>
__global__ void __launch_bounds__(256, CW == 8 ? 5 : 0)
p4_flat_kernel(const __grid_constant__ P4FlatParams p) {
    constexpr int CB = 4 * CW;
    constexpr int LCB = CW == 8 ? 5 : 4;
    pdl_wait();
    pdl_trigger();
    // a warp owns 31 consecutive chunks; lane 31 only loads and shuffles the chunk after
    // them (the next warp's first), so no lane reloads a neighbour's chunks
    const int lane = threadIdx.x & 31;
    const uint32_t t = (blockIdx.x * 8 + (threadIdx.x >> 5)) * 31 + lane;
    const bool live = lane < 31 && t < p.nchunks;
    const uint32_t q = t < p.nchunks ? t : p.nchunks - 1;
    const int base = (int)(q * CB);                     // nbytes <= 2^30: 32-bit byte offsets
    const int rb = (int)p.rb, nb = (int)p.nbytes;
    const int full = nb >> LCB;
    auto chunk = [&](int b0, uint32_t (&v)[CW]) {       // clamped aligned chunk
        const int c = min(max(b0 >> LCB, 0), full - 1);
        flat_load<CW>(reinterpret_cast<const uint32_t *>(p.in + (size_t)c * CB), v);
    };
    // down phase RD = rb % CB = 4 * RDW + s (s = rb % 4 in 1..3); up phase RU = CB - RD
    const int s = p.s;
    const int RD = 4 * RDW + s;
    const int RU = CB - RD;
    uint32_t u0[CW], cm[CW], d0[CW];
    chunk(base - rb - RU, u0);
    chunk(base, cm);
    chunk(base + rb - RD, d0);
    uint32_t lwb = 0u;                                  // the byte before the warp's chunks
    if (lane == 0 && base > 0) lwb = p4_ld8(p.in + base - 1);
    // (u0 ++ next lane's u0) from byte RU = 4 * (CW - 1 - RDW) + (4 - s); (d0 ++ next
    // lane's d0) from byte RD: one funnel shift per word
    uint32_t up[CW], dw[CW];
    {
        uint32_t U[2 * CW];
#pragma unroll
        for (int j = 0; j < CW; ++j) {
            U[j] = u0[j];
            U[CW + j] = __shfl_down_sync(0xFFFFFFFFu, u0[j], 1);
        }
        const uint32_t su = 32 - 8 * s;
#pragma unroll
        for (int j = 0; j < CW; ++j)
            up[j] = __funnelshift_r(U[j + CW - 1 - RDW], U[j + CW - RDW], su);
    }
    {
        uint32_t D[2 * CW];
#pragma unroll
        for (int j = 0; j < CW; ++j) {
            D[j] = d0[j];
            D[CW + j] = __shfl_down_sync(0xFFFFFFFFu, d0[j], 1);
        }
        const uint32_t sd = 8 * s;
#pragma unroll
        for (int j = 0; j < CW; ++j)
            dw[j] = __funnelshift_r(D[j + RDW], D[j + RDW + 1], sd);
    }
    // chunks within two rows of the buffer ends (clamped vector loads) and the ragged
    // tail.  EDGE_INLINE (small payloads, where the slowest warp is the kernel time):
    // reload their words from bytes here, all loads in flight at once; otherwise they are
    // redone out of line below, keeping this code out of the large rasters' main path
    const bool edge_zone = base < rb + 2 * CB || base + rb + 2 * CB > nb || base + CB > nb;
    if (EDGE_INLINE && edge_zone) {
#pragma unroll
        for (int j = 0; j < CW; ++j) {
            uint32_t c = 0u, uu = 0u, dd = 0u;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int b = base + 4 * j + k;
                if (b < nb) c |= (uint32_t)p.in[b] << (8 * k);
                if (b - rb >= 0 && b - rb < nb) uu |= (uint32_t)p.in[b - rb] << (8 * k);
                if (b + rb < nb) dd |= (uint32_t)p.in[b + rb] << (8 * k);
            }
            cm[j] = c; up[j] = uu; dw[j] = dd;
        }
    }
    // black-domain pixel-order centre words; neighbours across lanes
    uint32_t cb[CW];
#pragma unroll
    for (int j = 0; j < CW; ++j) cb[j] = __byte_perm(cm[j], 0, 0x0123);
    uint32_t lw = __shfl_up_sync(0xFFFFFFFFu, cb[CW - 1], 1);   // bit 0: the pixel before the chunk
    const uint32_t rw = __shfl_down_sync(0xFFFFFFFFu, cb[0], 1);  // bit 31: the pixel after
    if (lane == 0) lw = lwb;
    if (!live) return;

    // ---- every word as a word inside its row, inside its image (P4 domain)
    uint32_t o[CW];
#pragma unroll
    for (int j = 0; j < CW; ++j) {
        const uint32_t left = j == 0 ? lw : cb[j - 1];
        const uint32_t right = j == CW - 1 ? rw : cb[j + 1];
        const uint32_t lr = __funnelshift_r(cb[j], left, 1) & __funnelshift_l(right, cb[j], 1);
        o[j] = cm[j] & ~(__byte_perm(lr, 0, 0x0123) & up[j] & dw[j]);
    }
    // ---- row structure: byte jb of row r starts the chunk
    const uint32_t r = fdiv((uint32_t)base, p.div_rb);
    uint32_t jb = (uint32_t)base - r * p.rb;
    uint32_t y = r - fdiv(r, p.div_h) * p.h;
    const uint32_t hm1 = p.h - 1;
    // out-of-line edge chunks (their loads and shuffles above served the neighbours)
    if (!EDGE_INLINE && edge_zone) {
        p4_flat_edge_chunk(p, base, CW, jb, y);
        return;
    }
    // chunks holding a row's first or last byte, or in an image's top / bottom row,
    // redo the words concerned
    if (jb == 0 || jb + CB >= p.rb || y == 0 || y == hm1) {
#pragma unroll
        for (int j = 0; j < CW; ++j) {
            if (j > 0) {
                jb += 4;
                if (jb >= p.rb) {                 // rb >= 4: at most one row start per word
                    jb -= p.rb;
                    y = y == hm1 ? 0u : y + 1;
                }
            }
            if (jb != 0 && p.rb - jb > 4 && y != 0 && y != hm1) continue;
            o[j] = p4_row_word(p, cb[j], j == 0 ? lw : cb[j - 1], j == CW - 1 ? rw : cb[j + 1],
                               up[j], dw[j], jb, y);
        }
    }
    if (!EDGE_INLINE || base + CB <= nb) {
        store_chunk<CW>(reinterpret_cast<uint32_t *>(p.out + base), o);
    } else {
#pragma unroll
        for (int j = 0; j < CW; ++j)
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (base + 4 * j + k < nb) p.out[base + 4 * j + k] = (uint8_t)(o[j] >> (8 * k));
    }
}

}  // namespace capi
}  // namespace bitedge


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
    if (rb % 16 == 0 && al(p4_in, 16) && al(p4_out, 16) && !knob(KN_P4_UNFUSED) &&
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
        K1Div dv;
        if (grid <= 0x7FFFFFFFLL && k1_setup(rp, dv)) {
            const bool aligned = cw == 8 && w % 256 == 0 && !knob(KN_K1_GENERIC);
            if (aligned && rs == 4)
                launch_k(edge_reg_packed_kernel<0, 4, 8, kOutEdges, false, true, true>, (unsigned)grid,
                         0, st, rp, dv);
            else if (aligned)
                launch_k(edge_reg_packed_kernel<0, 2, 8, kOutEdges, false, true, true>, (unsigned)grid,
                         0, st, rp, dv);
            else if (cw == 8 && rs == 4)
                launch_k(edge_reg_packed_kernel<0, 4, 8, kOutEdges, false, true>, (unsigned)grid, 0,
                         st, rp, dv);
            else if (cw == 8)
                launch_k(edge_reg_packed_kernel<0, 2, 8, kOutEdges, false, true>, (unsigned)grid, 0,
                         st, rp, dv);
            else if (rs == 4)
                launch_k(edge_reg_packed_kernel<0, 4, 4, kOutEdges, false, true>, (unsigned)grid, 0,
                         st, rp, dv);
            else
                launch_k(edge_reg_packed_kernel<0, 2, 4, kOutEdges, false, true>, (unsigned)grid, 0,
                         st, rp, dv);
            return cuda_check("edge_reg_packed_kernel<P4>");
        }
    }
    // byte-granular rows (rb % 4 != 0) >= 4 bytes in 16-byte aligned buffers: K1p (the
    // payload as one flat byte array, aligned vector loads and stores; 32-byte
    // chunks when both buffers allow, BITEDGE_P4_FLAT16 keeps 16-byte chunks;
    // BITEDGE_P4_FLAT_MAX caps the payload size in bytes).  Rows of whole 4-byte
    // words run K1 UNAL below (8000x8000: 7.0 us).
    int64_t flat_max = (int64_t)1 << 30;                   // 32-bit byte offsets in the kernel
    if (const char *v = knob(KN_P4_FLAT_MAX)) flat_max = atoll(v);
    const int64_t p4_bytes = n * h * rb;
    if (rb >= 4 && rb % 4 != 0 && p4_bytes >= 32 && p4_bytes <= flat_max &&
        al(p4_in, 16) && al(p4_out, 16) &&
        !knob(KN_P4_UNFUSED) && !knob(KN_P4_BYTES) && !knob(KN_P4_NO_FLAT)) {
        // 32-byte chunks from 3072-byte rows up: shorter rows put a row boundary in most
        // warps' chunks, and the per-word fix-up pass is shorter over 4 words
        // (32000x32002: 54.9 vs 57.7 us; 16000x16002: 18.1 vs 17.5; 8000x8001: 8.3 vs 7.1)
        const bool c8 = al(p4_in, 32) && al(p4_out, 32) && !knob(KN_P4_FLAT16) &&
                        (rb >= 3072 || knob(KN_P4_FLAT32));
        const int cb = c8 ? 32 : 16;
        P4FlatParams fp;
        memset(&fp, 0, sizeof(fp));
        fp.in = p4_in; fp.out = p4_out;
        fp.nbytes = (uint32_t)p4_bytes;
        fp.rb = (uint32_t)rb; fp.h = (uint32_t)h;
        fp.nchunks = (fp.nbytes + cb - 1) / cb;
        fp.wlast = (uint32_t)((w - 1) % 8);
        fp.fw = G.fillword;
        fp.s = (int)(rb % 4);
        fp.div_rb = make_fastdiv((uint32_t)rb);
        fp.div_h = make_fastdiv((uint32_t)h);
        const unsigned grid = (fp.nchunks + 247) / 248;        // 8 warps x 31 chunks
        const int rdw = (int)((rb % cb) / 4);
#define BE_K1P(CW, R, E) case R: launch_kb(p4_flat_kernel<CW, R, E>, grid, 256u, 0, st, fp); break;
        // payloads under 4 MiB reload their edge chunks inline (4000x4001: 3.7 vs 4.2 us;
        // 16000x16002: 18.8 vs 17.5 us)
        if (c8) {
            switch (rdw) { BE_K1P(8, 0, false) BE_K1P(8, 1, false) BE_K1P(8, 2, false) BE_K1P(8, 3, false)
                           BE_K1P(8, 4, false) BE_K1P(8, 5, false) BE_K1P(8, 6, false) BE_K1P(8, 7, false) }
        } else if (p4_bytes < ((int64_t)4 << 20)) {
            switch (rdw) { BE_K1P(4, 0, true) BE_K1P(4, 1, true) BE_K1P(4, 2, true) BE_K1P(4, 3, true) }
        } else {
            switch (rdw) { BE_K1P(4, 0, false) BE_K1P(4, 1, false) BE_K1P(4, 2, false) BE_K1P(4, 3, false) }
        }
#undef BE_K1P
        return cuda_check("p4_flat_kernel");
    }
    // rows of whole 4-byte words (w % 32 == 0 or 25..31) that are not a multiple of the
    // vector width: K1f's flat view with the P4 conversions (edge_flat.cuh)
    if (rb % 4 == 0 && !knob(KN_P4_UNFUSED) && !knob(KN_P4_BYTES) && !knob(KN_NO_FLAT) &&
        !knob(KN_P4_NO_FLAT)) {
        const int64_t S = rb / 4, nwords = n * h * S;
        const int cw = (al(p4_in, 32) && al(p4_out, 32)) ? 8 : (al(p4_in, 16) && al(p4_out, 16)) ? 4 : 0;
        if (cw != 0 && S >= 16 && S % cw != 0 && nwords <= ((int64_t)1 << 30) &&
            h < ((int64_t)1 << 31)) {
            FlatParams fp;
            memset(&fp, 0, sizeof(fp));
            fp.in = (const uint32_t *)p4_in;
            fp.o_edges = (uint32_t *)p4_out;
            fp.nwords = (uint32_t)nwords; fp.S = (uint32_t)S; fp.h = (uint32_t)h;
            fp.nrows = (uint32_t)(n * h);
            fp.pl = G.pl; fp.lastbit = G.lastbit; fp.padmask = G.padmask; fp.fillword = G.fillword;
            fp.nchunks = (uint32_t)((nwords + cw - 1) / cw);
            fp.div_s = make_fastdiv((uint32_t)S);
            fp.div_h = make_fastdiv((uint32_t)h);
            const int ru = (int)((cw - S % cw) % cw);
            constexpr unsigned per_cta = (kThreads / 32) * 31;    // a warp owns 31 chunks
            const unsigned grid = (fp.nchunks + per_cta - 1) / per_cta;
#define BE_K1F_P4(CW, R) case R: launch_k(edge_flat_kernel<CW, 0, R, kOutEdges, true>, grid, 0, st, fp); break;
            if (cw == 8) {
                switch (ru) { BE_K1F_P4(8, 1) BE_K1F_P4(8, 2) BE_K1F_P4(8, 3) BE_K1F_P4(8, 4)
                              BE_K1F_P4(8, 5) BE_K1F_P4(8, 6) BE_K1F_P4(8, 7) }
            } else {
                switch (ru) { BE_K1F_P4(4, 1) BE_K1F_P4(4, 2) BE_K1F_P4(4, 3) }
            }
#undef BE_K1F_P4
            return cuda_check("edge_flat_kernel<P4>");
        }
    }
    // other rows of whole 4-byte words: K1 with 4-word items cut out of aligned 16-byte
    // chunks (UNAL)
    if (rb % 4 == 0 && al(p4_in, 4) && al(p4_out, 4) && !knob(KN_P4_UNFUSED) &&
        !knob(KN_P4_BYTES) && n * h < ((int64_t)1 << 31)) {
        RegParams rp;
        memset(&rp, 0, sizeof(rp));
        rp.in = (const char *)p4_in; rp.in_row_bytes = rb;
        rp.in_end = (const char *)p4_in + n * h * rb;
        rp.unal_words = knob(KN_UNAL_CHUNKS) == nullptr;   // words: measured faster
        rp.o_edges = (uint32_t *)p4_out; rp.out_stride = rb / 4;
        rp.nrows = n * h; rp.row_lo = 0; rp.row_hi = n * h;
        rp.h = (uint32_t)h; rp.w = w; rp.wp = G.wp; rp.pl = G.pl;
        rp.lastbit = G.lastbit; rp.padmask = G.padmask; rp.fillword = G.fillword;
        rp.thr = 1;
        rp.items = (G.wp + 3) / 4;
        rp.vst = 0;                                  // rows are 4-byte aligned: word stores
        const bool big = ((n * h + 3) / 4) * rp.items >= (int64_t)sm_count() * 4096 * 2;
        const int rs = big ? 4 : 2;
        rp.nstrips = (n * h + rs - 1) / rs;
        const int64_t grid = (rp.nstrips * rp.items + kThreads - 1) / kThreads;
        K1Div dv;
        if (grid <= 0x7FFFFFFFLL && k1_setup(rp, dv)) {
            if (rs == 4)
                launch_k(edge_reg_packed_kernel<0, 4, 4, kOutEdges, false, true, false, true>,
                         (unsigned)grid, 0, st, rp, dv);
            else
                launch_k(edge_reg_packed_kernel<0, 2, 4, kOutEdges, false, true, false, true>,
                         (unsigned)grid, 0, st, rp, dv);
            return cuda_check("edge_reg_packed_kernel<P4, word loads>");
        }
    }
    // any other row length: the byte-granular single-pass kernel
    constexpr int kR = 8;
    const int64_t nstrips = (n * h + kR - 1) / kR;
    const bool fits = nstrips * G.wp + 256 < ((int64_t)1 << 32) && n * h < ((int64_t)1 << 32) - kR;
    if (!knob(KN_P4_UNFUSED) && fits) {
        WordGeom g = word_geom(G, G.wp);
        const int64_t threads = nstrips * g.wp;
        p4_edges_bytes_kernel<kR><<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(
            p4_in, p4_out, g, rb, (uint32_t)nstrips, make_fastdiv((uint32_t)g.wp),
            make_fastdiv((uint32_t)g.h));
        return cuda_check("p4_edges_bytes_kernel");
    }
    // reference path (BITEDGE_P4_UNFUSED, or > 2^32 threads): decode -> K1 ->
    // encode through caller scratch (2 word rasters)
    if (scratch_or_null == nullptr)
        return fail(BE_EINVAL, "unaligned P4 rows (ceil(w/8) %% 16 != 0) need a scratch buffer of "
                               "2 * n * h * ceil(w/32) words");
    const int64_t words = n * h * G.wp;
    uint32_t *dec = scratch_or_null, *edg = scratch_or_null + words;
    if ((rc = be_p4_decode(p4_in, dec, 32, n, h, w, G.wp, stream))) return rc;
    if ((rc = be_edge_packed_u32(dec, edg, n, h, w, G.wp, fill_bit, 0, stream))) return rc;
    return be_p4_encode(edg, p4_out, 32, n, h, w, G.wp, stream);
}

// capi_words.cu -- the word-parallel kernels behind the BitImage primitives
// (bitimage.py:149-249: invert / AND / OR, shift, count_black, to_array) and the
// paper's per-pixel scan, with their C-ABI entry points.
#include "capi_internal.cuh"

using namespace bitedge;
using namespace bitedge::capi;

namespace bitedge {
namespace capi {

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

}  // namespace capi
}  // namespace bitedge

extern "C" {

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

}  // extern "C"

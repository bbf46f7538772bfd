/* Plain-C per-pixel Edge(p) scanner -- TEST INFRASTRUCTURE ONLY.
 *
 * Restates the paper's "traditional scanning" definition (PAPER.md:25-37,
 * SPEC.md:174-191): a pixel is an edge point iff it is black (0) and at least
 * one of its 4-neighbours (Fig. 1 indices 2,4,6,8) is white,
 * with out-of-raster neighbours taking the border fill.
 * Output follows detect_edges_mask's convention: edge pixels
 * black (0), everything else white (1), packed MSB-first into uint32 row
 * words with padding bits = 1 (bitimage.py:1-11, 101-104).
 *
 * This is an algorithm independent of the word-level mask method, fast enough
 * to check the full-size BASELINE configs (C4: 4 Gpx, C5: 4 Gpx) where the
 * numpy port (oracle/port.py) is too slow: every scanner splits its rows over
 * ORACLE_THREADS (default: all online cores) pthreads with parallel_for.
 * Only tests/ and bench.py's CPU legs may load it.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* Minimal pthread parallel-for over [0, total) (no OpenMP runtime dependency). */
typedef void (*range_fn)(void *ctx, int64_t lo, int64_t hi);
typedef struct { range_fn fn; void *ctx; int64_t lo, hi; } job_t;

static void *run_job(void *p) {
    job_t *j = (job_t *)p;
    j->fn(j->ctx, j->lo, j->hi);
    return NULL;
}

static int n_threads(void) {
    const char *e = getenv("ORACLE_THREADS");
    long t = e ? atol(e) : sysconf(_SC_NPROCESSORS_ONLN);
    if (t < 1) t = 1;
    if (t > 256) t = 256;
    return (int)t;
}

static void parallel_for(int64_t total, range_fn fn, void *ctx) {
    int t = n_threads();
    if (total < 64 || t == 1) { fn(ctx, 0, total); return; }
    if (t > total) t = (int)total;
    pthread_t th[256];
    job_t jobs[256];
    for (int i = 0; i < t; ++i) {
        jobs[i].fn = fn; jobs[i].ctx = ctx;
        jobs[i].lo = total * i / t; jobs[i].hi = total * (i + 1) / t;
        pthread_create(&th[i], NULL, run_job, &jobs[i]);
    }
    for (int i = 0; i < t; ++i) pthread_join(th[i], NULL);
}

int orc_threads(void) { return n_threads(); }

static inline int px_u8(const uint8_t *img, int64_t h, int64_t w, int64_t stride,
                        int64_t x, int64_t y, int fill) {
    if (x < 0 || y < 0 || x >= w || y >= h) return fill;
    return img[y * stride + x] != 0;               /* nonzero -> white (bitimage.py:124,133) */
}

static inline int px_p32(const uint32_t *img, int64_t h, int64_t w, int64_t stride,
                         int64_t x, int64_t y, int fill) {
    if (x < 0 || y < 0 || x >= w || y >= h) return fill;
    return (img[y * stride + (x >> 5)] >> (31 - (x & 31))) & 1u;
}

/* Edge(p) on one pixel: returns the OUTPUT bit (0 = edge). With edgeset=1 the
 * marker convention is used instead (1 = edge). */
#define EDGE_BIT(PX)                                                              \
    do {                                                                          \
        int p = PX(x, y);                                                         \
        int e = !p && (PX(x, y - 1) | PX(x - 1, y) | PX(x, y + 1) | PX(x + 1, y));\
        bit = edgeset ? e : !e;                                                   \
    } while (0)

/* in: uint8 [n, h, w] with row stride `in_stride` bytes (image stride h*in_stride);
 * out: uint32 [n, h, ceil(w/32)] contiguous. */
typedef struct {
    const uint8_t *in; uint32_t *out; int64_t h, w, in_stride; int fill, edgeset;
} scan_u8_ctx;

static void scan_u8_rows(void *vctx, int64_t lo, int64_t hi) {
    const scan_u8_ctx *c = (const scan_u8_ctx *)vctx;
    const int64_t h = c->h, w = c->w, in_stride = c->in_stride;
    const int fill = c->fill, edgeset = c->edgeset;
    const int64_t wp = (w + 31) / 32;
    for (int64_t ry = lo; ry < hi; ++ry) {
        const int64_t img_i = ry / h, y = ry % h;
        const uint8_t *img = c->in + img_i * h * in_stride;
        uint32_t *orow = c->out + ry * wp;
        for (int64_t k = 0; k < wp; ++k) {
            uint32_t word = 0;
            for (int b = 0; b < 32; ++b) {
                int64_t x = k * 32 + b;
                int bit = 1;                                   /* padding = 1 */
                if (x < w) {
#define PXU(xx, yy) px_u8(img, h, w, in_stride, (xx), (yy), fill)
                    EDGE_BIT(PXU);
#undef PXU
                }
                word = (word << 1) | (uint32_t)bit;
            }
            orow[k] = word;
        }
    }
}

void orc_scan_u8_packed32(const uint8_t *in, uint32_t *out, int64_t n, int64_t h, int64_t w,
                          int64_t in_stride, int fill, int edgeset) {
    scan_u8_ctx c = {in, out, h, w, in_stride, fill, edgeset};
    parallel_for(n * h, scan_u8_rows, &c);
}

/* in: packed uint32 rows [n, h, in_stride words] (padding bits ignored);
 * out: uint32 [n, h, ceil(w/32)] contiguous. */
typedef struct {
    const uint32_t *in; uint32_t *out; int64_t h, w, in_stride; int fill, edgeset;
} scan_p32_ctx;

static void scan_p32_rows(void *vctx, int64_t lo, int64_t hi) {
    const scan_p32_ctx *c = (const scan_p32_ctx *)vctx;
    const int64_t h = c->h, w = c->w, in_stride = c->in_stride;
    const int fill = c->fill, edgeset = c->edgeset;
    const int64_t wp = (w + 31) / 32;
    for (int64_t ry = lo; ry < hi; ++ry) {
        const int64_t img_i = ry / h, y = ry % h;
        const uint32_t *img = c->in + img_i * h * in_stride;
        uint32_t *orow = c->out + ry * wp;
        for (int64_t k = 0; k < wp; ++k) {
            uint32_t word = 0;
            for (int b = 0; b < 32; ++b) {
                int64_t x = k * 32 + b;
                int bit = 1;
                if (x < w) {
#define PXP(xx, yy) px_p32(img, h, w, in_stride, (xx), (yy), fill)
                    EDGE_BIT(PXP);
#undef PXP
                }
                word = (word << 1) | (uint32_t)bit;
            }
            orow[k] = word;
        }
    }
}

void orc_scan_p32(const uint32_t *in, uint32_t *out, int64_t n, int64_t h, int64_t w,
                  int64_t in_stride, int fill, int edgeset) {
    scan_p32_ctx c = {in, out, h, w, in_stride, fill, edgeset};
    parallel_for(n * h, scan_p32_rows, &c);
}

/* Row-slab variant: rows [0, rows) of a slab whose global neighbours above
 * (row -1) and below (row `rows`) come from `above` / `below` (NULL -> fill).
 * Used to check the row-sharded (halo) path. */
typedef struct {
    const uint32_t *slab, *above, *below; uint32_t *out; int64_t rows, w, stride; int fill;
} scan_slab_ctx;

static void scan_slab_rows(void *vctx, int64_t lo, int64_t hi) {
    const scan_slab_ctx *c = (const scan_slab_ctx *)vctx;
    const int64_t rows = c->rows, w = c->w, stride = c->stride;
    const int fill = c->fill;
    const int64_t wp = (w + 31) / 32;
    for (int64_t y = lo; y < hi; ++y) {
        for (int64_t k = 0; k < wp; ++k) {
            uint32_t word = 0;
            for (int b = 0; b < 32; ++b) {
                int64_t x = k * 32 + b;
                int bit = 1;
                if (x < w) {
                    int nb[4];
                    int cc = px_p32(c->slab, rows, w, stride, x, y, fill);
                    nb[0] = px_p32(c->slab, rows, w, stride, x - 1, y, fill);
                    nb[1] = px_p32(c->slab, rows, w, stride, x + 1, y, fill);
                    if (y > 0) nb[2] = px_p32(c->slab, rows, w, stride, x, y - 1, fill);
                    else nb[2] = c->above ? px_p32(c->above, 1, w, stride, x, 0, fill) : fill;
                    if (y + 1 < rows) nb[3] = px_p32(c->slab, rows, w, stride, x, y + 1, fill);
                    else nb[3] = c->below ? px_p32(c->below, 1, w, stride, x, 0, fill) : fill;
                    int e = !cc && (nb[0] | nb[1] | nb[2] | nb[3]);
                    bit = !e;
                }
                word = (word << 1) | (uint32_t)bit;
            }
            c->out[y * wp + k] = word;
        }
    }
}

void orc_scan_p32_slab(const uint32_t *slab, const uint32_t *above, const uint32_t *below,
                       uint32_t *out, int64_t rows, int64_t w, int64_t stride, int fill) {
    scan_slab_ctx c = {slab, above, below, out, rows, w, stride, fill};
    parallel_for(rows, scan_slab_rows, &c);
}

int orc_version(void) { return 1; }

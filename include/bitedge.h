/* bitedge.h -- C ABI of the B200 (sm_100a) method-of-masks edge detector.
 *
 * The reference (`bitedge`, /root/reference/pkg) is pure Python/numpy and has
 * no FFI; this ABI is the boundary its Python API binds to (ctypes, see
 * paper_1401_5245_b200/_capi.py and INTEGRATION.md).  Each entry point names
 * the reference operation it replaces.
 *
 * Raster layout (bitimage.py:1-11): one pixel per bit, 1 = white, 0 = black,
 * rows packed MSB-first (the MSB of a word is its leftmost pixel).  Two word
 * formats are accepted, selected by `word_bits`:
 *   64 -- native uint64 words, the reference's BitImage.words layout
 *         (bitimage.py:91-97); shape [n, h, row_stride] with
 *         row_stride >= ceil(w/64);
 *   32 -- uint32 row words, BASELINE.json's pre-packed format (configs 3, 4);
 *         row_stride >= ceil(w/32).
 * `row_stride_words` counts words of the selected format.  Images of a batch
 * are contiguous ([n][h][row_stride]).  Input padding bits (pixels >= w) may
 * hold anything and are never read for a visible output; every packed output
 * has its padding bits set to 1, as the reference's constructor forces
 * (bitimage.py:101-104).
 *
 * Border policy (bitimage.py:56-64): fill_bit 1 = WHITE_OUTSIDE (the default
 * of every reference entry point), 0 = BLACK_OUTSIDE.
 *
 * Conventions: the caller owns every buffer (device pointers unless stated);
 * nothing is allocated; every launch is asynchronous on `stream` (a
 * cudaStream_t, NULL = legacy default stream).  Return 0 on success, a
 * negative BE_E* code for invalid arguments (message in be_last_error(),
 * mapped to ValueError by the Python layer), or a positive cudaError_t.  The
 * library keeps no global mutable state besides a thread-local error string,
 * so it is reentrant; outputs never alias inputs unless stated.
 */
#ifndef BITEDGE_H
#define BITEDGE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BE_ABI_VERSION 1

enum {
    BE_OK = 0,
    BE_EINVAL = -1,     /* bad size / stride / pointer / enum */
    BE_EALIGN = -2,     /* misaligned pointer for the requested format */
    BE_ESHAPE = -3      /* operand dimensions disagree */
};

/* Direction enum, (dx, dy) with y growing downwards (bitimage.py:35-41). */
enum { BE_LEFT = 0, BE_RIGHT = 1, BE_UP = 2, BE_DOWN = 3 };

/* Binary/unary word ops (bitimage.py:181-205). */
enum { BE_OP_NOT = 0, BE_OP_AND = 1, BE_OP_OR = 2 };

/* Optional outputs of the fused edge kernel; any pointer may be NULL.
 *   edges    detect_edges_mask: NOT(OR of the four fundamental edges),
 *            edges black (0) on white
 *   edgeset  the pre-inversion OR, 1 = edge pixel
 *   side[s]  fundamental_edge(img, build_mask(img), s) for s = BE_LEFT..BE_DOWN,
 *            i.e. shift(img, opposite(s)) AND NOT img
 *   packed   the packed input itself (from_array, bitimage.py:122-136); only
 *            meaningful for the uint8 entry points
 * All outputs share word format and row stride. */
typedef struct be_outputs {
    void *edges;
    void *edgeset;
    void *side[4];
    void *packed;
} be_outputs;

/* ---- the fused hot path ------------------------------------------------- */

/* K1. detect_edges_mask on packed rasters (SPEC.md:165-168 composed from
 * bitimage.py:181-240): out = C | ~(Ln | Rn | Un | Dn), padding = 1.
 * emit_edgeset != 0 writes the EdgeSet instead. */
int be_edge_packed_u32(const uint32_t *in, uint32_t *out, int64_t n, int64_t h, int64_t w,
                       int64_t row_stride_words, int fill_bit, int emit_edgeset, void *stream);
int be_edge_packed_u64(const uint64_t *in, uint64_t *out, int64_t n, int64_t h, int64_t w,
                       int64_t row_stride_words, int fill_bit, int emit_edgeset, void *stream);

/* K2. BitImage.from_array (bitimage.py:122-136: nonzero byte -> white) fused
 * with K1.  `in` is uint8 [n, h, in_row_stride bytes]; `out` uint32 words with
 * out_row_stride_words; packed_in_or_null additionally receives the packed
 * input (same stride). */
int be_pack_edge_u8(const uint8_t *in, uint32_t *out, int64_t n, int64_t h, int64_t w,
                    int64_t in_row_stride, int64_t out_row_stride_words, int fill_bit,
                    uint32_t *packed_in_or_null, void *stream);

/* K3. K1 on a row slab of one image whose row -1 / row `rows` come from
 * neighbour slabs (the received halo rows) instead of the border fill; only
 * output rows [row_lo, row_hi) are written.  A NULL halo means the slab touches
 * the image border there and the fill applies (bitimage.py:216-223).
 * `row_stride_words` (the slab's and the output's stride, >= ceil(w/32)) is
 * one argument more than SURVEY.md 8(b) sketched: slabs cut from a padded
 * raster keep its stride. */
int be_edge_packed_halo_u32(const uint32_t *slab, const uint32_t *above_or_null,
                            const uint32_t *below_or_null, uint32_t *out, int64_t rows, int64_t w,
                            int64_t row_stride_words, int fill_bit, int64_t row_lo, int64_t row_hi,
                            void *stream);

/* K3e: output rows 0 and rows-1 of a slab only (the two rows that read a halo),
 * in one launch; same arguments and meaning as be_edge_packed_halo_u32 with the
 * row range fixed to {0, rows-1}.  Row-sharded callers compute rows
 * [1, rows-1) with be_edge_packed_halo_u32 while the halo rows are exchanged,
 * then this.  (Replaces, for the boundary rows, the vertical fill the
 * reference applies at rows 0 / H-1: bitimage.py:216-223.) */
int be_edge_packed_halo_ends_u32(const uint32_t *slab, const uint32_t *above_or_null,
                                 const uint32_t *below_or_null, uint32_t *out, int64_t rows,
                                 int64_t w, int64_t row_stride_words, int fill_bit, void *stream);

/* General form of K1/K2/K3 with every optional output (F3 of SURVEY 8(f)).
 * input_kind 0: packed words of `word_bits`; 1: uint8 pixels (in_row_stride
 * in bytes).  above/below as in K3 (n must be 1 when either is non-NULL). */
int be_edges_general(const void *in, int input_kind, int64_t in_row_stride,
                     const void *above_or_null, const void *below_or_null,
                     const be_outputs *outs, int word_bits, int64_t out_row_stride_words,
                     int64_t n, int64_t h, int64_t w, int fill_bit, int64_t row_lo,
                     int64_t row_hi, void *stream);

/* ---- BitImage primitives (bitimage.py), device-resident ------------------ */

/* from_array (bitimage.py:122-136): uint8 -> packed, nonzero = white, pad = 1. */
int be_pack_u8(const uint8_t *in, void *out, int word_bits, int64_t n, int64_t h, int64_t w,
               int64_t in_row_stride, int64_t out_row_stride_words, void *stream);
/* to_array (bitimage.py:149-153): packed -> uint8 {0,1}. */
int be_unpack_u8(const void *in, uint8_t *out, int word_bits, int64_t n, int64_t h, int64_t w,
                 int64_t in_row_stride_words, int64_t out_row_stride, void *stream);
/* invert / & / | (bitimage.py:181-205); b unused for NOT; padding = 1. */
int be_bitop(int op, const void *a, const void *b, void *out, int word_bits, int64_t n,
             int64_t h, int64_t w, int64_t row_stride_words, void *stream);
/* shift (bitimage.py:207-240): out(x, y) = in(x - dx, y - dy), outside = fill. */
int be_shift(const void *in, void *out, int word_bits, int64_t n, int64_t h, int64_t w,
             int64_t row_stride_words, int direction, int fill_bit, void *stream);
/* fundamental_edge with an explicit mask:
 * out = shift(img, opposite(side), fill) AND mask, fused in one pass. */
int be_shift_and(const void *img, const void *mask, void *out, int word_bits, int64_t n,
                 int64_t h, int64_t w, int64_t row_stride_words, int side, int fill_bit,
                 void *stream);
/* count_black (bitimage.py:244-249) per image into counts[n] (int64, device). */
int be_count_black(const void *in, int64_t *counts, int word_bits, int64_t n, int64_t h,
                   int64_t w, int64_t row_stride_words, void *stream);

/* detect_edges_scan: the paper's per-pixel Edge(p) scanner
 * on the device, bit by bit -- an algorithm independent of K1, exposed for the
 * reference API and as a full-size cross-check. */
int be_scan_edges(const void *in, void *out, int word_bits, int64_t n, int64_t h, int64_t w,
                  int64_t row_stride_words, int fill_bit, void *stream);

/* ---- grayscale input ------------------------------------- */

/* binarize.threshold (sample >= threshold -> white) fused with
 * detect_edges_mask: uint8 luminance [n][h][in_row_stride] -> edge words; the
 * binarised raster itself optionally lands in binary_or_null.  threshold = 1 is
 * exactly be_pack_edge_u8 (nonzero = white). */
int be_threshold_edge_u8(const uint8_t *in, uint32_t *out, int64_t n, int64_t h, int64_t w,
                         int64_t in_row_stride, int64_t out_row_stride_words, int threshold,
                         int fill_bit, uint32_t *binary_or_null, void *stream);
/* binarize.threshold alone: uint8 luminance -> packed raster (word_bits 32/64). */
int be_threshold_u8(const uint8_t *in, void *out, int word_bits, int64_t n, int64_t h, int64_t w,
                    int64_t in_row_stride, int64_t out_row_stride_words, int threshold,
                    void *stream);

/* ---- PBM P4 at the kernel boundary ----------------------- */

/* The P4 payload: rows of ceil(w/8) bytes, MSB-first, 1 = black.
 * decode: P4 -> packed raster (1 = white, padding 1; word_bits 32 or 64);
 * encode: packed raster -> P4 (padding bits written 0). */
int be_p4_decode(const uint8_t *p4, void *out, int word_bits, int64_t n, int64_t h, int64_t w,
                 int64_t out_row_stride_words, void *stream);
int be_p4_encode(const void *in, uint8_t *p4, int word_bits, int64_t n, int64_t h, int64_t w,
                 int64_t in_row_stride_words, void *stream);
/* detect_edges_mask from a P4 payload to a P4 payload, one kernel for every
 * width.  When a P4 row is a whole number of 16-byte chunks (w % 128 in
 * 121..128 or 0) kernel K1 reads and writes P4 directly (kept in the P4 byte
 * order; only the centre row is byte-swapped for the horizontal shifts,
 * 0.25 B/px); other rows start at any byte and a byte-granular kernel does the
 * same in one pass.  `scratch_or_null` (2 * n * h * ceil(w/32) words) is only
 * used with BITEDGE_P4_UNFUSED set: decode -> K1 -> encode, the reference path
 * the tests compare against. */
int be_p4_edges(const uint8_t *p4_in, uint8_t *p4_out, int64_t n, int64_t h, int64_t w,
                int fill_bit, uint32_t *scratch_or_null, void *stream);

/* ---- peer-memory halos (multi-GPU row sharding without a separate exchange) --
 * A rank exports its slab with be_ipc_export (64-byte cudaIpcMemHandle_t plus
 * the pointer's offset inside its allocation); its row neighbours import it with
 * be_ipc_open and pass pointers to the neighbour's boundary rows straight to
 * be_edge_packed_halo_u32 as `above` / `below`: the halo rows are then read over
 * NVLink by the edge kernel itself. */
int be_ipc_export(const void *dev_ptr, void *handle_out, int64_t *offset_out);
int be_ipc_open(const void *handle, int64_t offset, void **dev_ptr_out);
int be_ipc_close(void *dev_ptr, int64_t offset);


/* ---- host buffers (the end-to-end path) ----------------------------------- */

/* Edges of a batch that lives in HOST memory (pinned for overlap): uint8 pixels
 * [n][h][w] (input_kind 1, from_array + detect_edges_mask) or packed uint32 rows
 * [n][h][ceil(w/32)] (input_kind 0) -> host_out uint32 [n][h][ceil(w/32)].  The
 * batch is moved in chunks of chunk_images through two caller-provided device
 * buffer pairs (dev_in[i] >= chunk * input image bytes, dev_out[i] >= chunk *
 * output image bytes); chunk c runs H2D -> kernel -> D2H on stream (c % 2), so
 * copies in both directions overlap the kernels.  blocking != 0 waits for both
 * streams before returning. */
int be_host_edges(const void *host_in, int input_kind, uint32_t *host_out, int64_t n, int64_t h,
                  int64_t w, int fill_bit, void *const dev_in[2], uint32_t *const dev_out[2],
                  int64_t chunk_images, void *stream0, void *stream1, int blocking);

/* The same for ONE large host image (or one row slab of it), chunked by rows
 * (C3 / C4-sized rasters, where image chunks would leave nothing to overlap):
 * chunk c copies rows [r0 - 1, r1 + 1) in (the 1-row halos), computes rows
 * [r0, r1) with the halo kernel and copies them out, on stream (c % 2).
 * dev_in[i] >= (chunk_rows + 2) input rows, dev_out[i] >= chunk_rows output
 * rows.  Input rows are w bytes (input_kind 1) or ceil(w/32) uint32 words
 * (input_kind 0).  halo_flags: bit 0 = host_in starts with row -1 (the row
 * above a slab), bit 1 = it ends with row h; without them the border fill
 * applies there.  host_out receives rows 0 .. h-1. */
int be_host_edges_rows(const void *host_in, int input_kind, uint32_t *host_out, int64_t h,
                       int64_t w, int fill_bit, int halo_flags, void *const dev_in[2],
                       uint32_t *const dev_out[2], int64_t chunk_rows, void *stream0,
                       void *stream1, int blocking);

/* The drop-in host flow for ONE image in one call -- BitImage.from_array(a)
 * (bitimage.py:122-136) + detect_edges_mask / edge_set
 * + .words (bitimage.py:140-147): uint8 pixels [h][w] (nonzero = white) in
 * page-locked host memory are copied to dev_pix (>= h*w bytes), packed and
 * edge-detected in one kernel into dev_out (uint64 BitImage words
 * [h][ceil(w/64)]; the packed input also into dev_packed when non-NULL), and the
 * words are copied to host_out (page-locked, same shape).  With dev_pix and/or
 * dev_out NULL the kernel reads the pixels / writes the words over PCIe itself
 * (mapped page-locked memory; small images, w < 1024), which skips the copy
 * operations' fixed latency.  Returns once the stream is idle: host_out is
 * ready and every buffer may be reused. */
int be_host_detect_u64(const uint8_t *host_pix, int64_t h, int64_t w, int fill_bit,
                       int emit_edgeset, uint8_t *dev_pix_or_null, uint64_t *dev_packed_or_null,
                       uint64_t *dev_out_or_null, uint64_t *host_out, void *stream);

/* The same one-call flow for SMALL images from ANY host memory (the drop-in's
 * per-image hot path, C1/C2-sized rasters): the pixels (row stride
 * pix_row_stride bytes, need not be page-locked) are copied into the caller's
 * page-locked staging buffer stage_in (>= h*w bytes), ONE kernel reads them and
 * writes the uint64 words into page-locked stage_out (>= h*ceil(w/64)*8 bytes)
 * over PCIe, and after the stream drains the words are copied to words_out (any
 * host memory).  With dev_stage_or_null (>= h*w bytes of device memory) the
 * pixels cross PCIe by one copy-engine transfer into it instead and the kernel
 * reads HBM (faster past a few tens of KB).  w < 1024.  The staging buffers are reusable as soon as the call
 * returns (one pair per calling thread keeps the page-locked footprint fixed). */
int be_host_detect_u64_staged(const uint8_t *pix, int64_t pix_row_stride, int64_t h, int64_t w,
                              int fill_bit, int emit_edgeset, uint8_t *stage_in,
                              int64_t stage_in_bytes, uint64_t *stage_out,
                              int64_t stage_out_bytes, uint8_t *dev_stage_or_null,
                              uint64_t *words_out, void *stream);

/* ---- misc ----------------------------------------------------------------- */
const char *be_last_error(void);
int be_abi_version(void);
/* Re-read the BITEDGE_* dispatch knobs from the environment (they are read once,
 * on the first call). */
int be_reload_knobs(void);
/* Number of kernels this thread has launched through the ABI (for bench.py's
 * gpu_launches accounting). */
int64_t be_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* BITEDGE_H */

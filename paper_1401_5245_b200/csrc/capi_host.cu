// capi_host.cu -- host-buffer pipelines (the end-to-end path), CUDA IPC for
// peer-memory halos, and the ABI's bookkeeping entry points.  Owns the library's
// only state: a thread-local error string and launch counter, and the cached
// copy of the BITEDGE_* dispatch knobs (read once; be_reload_knobs).
#include "capi_internal.cuh"

#include <time.h>

#include <atomic>
#include <mutex>

using namespace bitedge;
using namespace bitedge::capi;

namespace bitedge {
namespace capi {
thread_local char g_err[512];
thread_local int64_t g_launches = 0;

const char *const kKnobNames[KN_COUNT] = {
    "BITEDGE_KERNEL", "BITEDGE_K1_GENERIC", "BITEDGE_UNAL_BYTES", "BITEDGE_NO_UNAL",
    "BITEDGE_NO_TMA", "BITEDGE_CW4", "BITEDGE_UNAL_CHUNKS", "BITEDGE_CW8",
    "BITEDGE_NO_WARPIMG", "BITEDGE_WARPIMG_G4", "BITEDGE_PDL_LATE", "BITEDGE_TMA1",
    "BITEDGE_FORCE_TMA", "BITEDGE_U64_TMA", "BITEDGE_TMA2_RSL8", "BITEDGE_TMA2_RSL32",
    "BITEDGE_NO_ROLL", "BITEDGE_RS", "BITEDGE_PRS", "BITEDGE_UNAL_RS4", "BITEDGE_P4_UNFUSED",
    "BITEDGE_P4_BYTES", "BITEDGE_PDL", "BITEDGE_NO_FLAT", "BITEDGE_K2P", "BITEDGE_SYNC_BLOCK", "BITEDGE_NO_H16", "BITEDGE_RING", "BITEDGE_NO_TMA_UNAL", "BITEDGE_P4_NO_FLAT", "BITEDGE_P4_FLAT16", "BITEDGE_P4_FLAT_MAX", "BITEDGE_P4_FLAT32", "BITEDGE_TMA2_MIN", "BITEDGE_TMA2_RSL", "BITEDGE_TMA2_MINW", "BITEDGE_ROLL_MIN"};
}  // namespace capi
}  // namespace bitedge

namespace {
// copies of the knob values (the environment's own strings may be freed when it changes)
char g_knob_val[bitedge::capi::KN_COUNT][64];
bool g_knob_set[bitedge::capi::KN_COUNT];
std::atomic<int> g_knobs_loaded{0};
std::mutex g_knob_mu;

void load_knobs_locked() {
    for (int k = 0; k < bitedge::capi::KN_COUNT; ++k) {
        const char *v = getenv(bitedge::capi::kKnobNames[k]);
        g_knob_set[k] = v != nullptr;
        if (v) snprintf(g_knob_val[k], sizeof(g_knob_val[k]), "%s", v);
    }
    g_knobs_loaded.store(1, std::memory_order_release);
}
}  // namespace

namespace bitedge {
namespace capi {
const char *knob(Knob k) {
    if (!g_knobs_loaded.load(std::memory_order_acquire)) {
        std::lock_guard<std::mutex> lk(g_knob_mu);
        if (!g_knobs_loaded.load(std::memory_order_relaxed)) load_knobs_locked();
    }
    return g_knob_set[k] ? g_knob_val[k] : nullptr;
}
}  // namespace capi
}  // namespace bitedge

extern "C" {

int be_reload_knobs(void) {
    std::lock_guard<std::mutex> lk(g_knob_mu);
    load_knobs_locked();
    return BE_OK;
}

const char *be_last_error(void) { return g_err; }
int be_abi_version(void) { return BE_ABI_VERSION; }
int64_t be_launch_count(void) { return g_launches; }

// ---- peer-memory halos: CUDA IPC export / import of a device buffer --------
typedef int (*cuMemGetAddressRange_t)(unsigned long long *, size_t *, unsigned long long);

int be_ipc_export(const void *dev_ptr, void *handle_out, int64_t *offset_out) {
    if (dev_ptr == nullptr || handle_out == nullptr || offset_out == nullptr)
        return fail(BE_EINVAL, "NULL argument");
    // the IPC handle names the whole allocation: find its base through the driver
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || fn == nullptr)
        return fail(e != cudaSuccess ? (int)e : BE_EINVAL, "cuMemGetAddressRange unavailable");
    unsigned long long base = 0;
    size_t size = 0;
    if (((cuMemGetAddressRange_t)fn)(&base, &size, (unsigned long long)(uintptr_t)dev_ptr) != 0)
        return fail(BE_EINVAL, "pointer is not a device allocation");
    cudaIpcMemHandle_t h;
    e = cudaIpcGetMemHandle(&h, (void *)(uintptr_t)base);
    if (e != cudaSuccess) return fail((int)e, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    memcpy(handle_out, &h, sizeof(h));
    *offset_out = (int64_t)((uintptr_t)dev_ptr - base);
    return BE_OK;
}

int be_ipc_open(const void *handle, int64_t offset, void **dev_ptr_out) {
    if (handle == nullptr || dev_ptr_out == nullptr) return fail(BE_EINVAL, "NULL argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void *base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail((int)e, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    *dev_ptr_out = (char *)base + offset;
    return BE_OK;
}

int be_ipc_close(void *dev_ptr, int64_t offset) {
    if (dev_ptr == nullptr) return fail(BE_EINVAL, "NULL argument");
    cudaError_t e = cudaIpcCloseMemHandle((char *)dev_ptr - offset);
    if (e != cudaSuccess) return fail((int)e, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
    return BE_OK;
}

int be_host_edges(const void *host_in, int input_kind, uint32_t *host_out, int64_t n, int64_t h,
                  int64_t w, int fill_bit, void *const dev_in[2], uint32_t *const dev_out[2],
                  int64_t chunk_images, void *stream0, void *stream1, int blocking) {
    Geometry G;
    int rc = make_geometry(G, 32, n, h, w, fill_bit);
    if (rc) return rc;
    if (n == 0) return BE_OK;
    if (!host_in || !host_out || !dev_in || !dev_out || !dev_in[0] || !dev_in[1] || !dev_out[0] ||
        !dev_out[1])
        return fail(BE_EINVAL, "host / device buffers must not be NULL");
    if (input_kind != 0 && input_kind != 1)
        return fail(BE_EINVAL, "input_kind must be 0 (packed u32) or 1 (uint8)");
    if (chunk_images < 1) return fail(BE_EINVAL, "chunk_images must be >= 1");
    const int64_t wp = G.wp;
    const size_t in_img = (size_t)h * (input_kind == 1 ? (size_t)w : (size_t)wp * 4);
    const size_t out_img = (size_t)h * wp * 4;
    cudaStream_t ss[2] = {S(stream0), S(stream1)};
    uint32_t *side[4] = {nullptr, nullptr, nullptr, nullptr};
    // chunk c runs entirely on stream c % 2: H2D -> kernel -> D2H.  In-stream
    // order protects the reuse of buffer c % 2 by chunk c + 2, and the two
    // streams let one chunk's H2D overlap the other's kernel and D2H.
    for (int64_t c = 0, lo = 0; lo < n; ++c, lo += chunk_images) {
        const int64_t k = (n - lo) < chunk_images ? (n - lo) : chunk_images;
        const int b = (int)(c & 1);
        cudaError_t e = cudaMemcpyAsync(dev_in[b], (const char *)host_in + lo * in_img, k * in_img,
                                        cudaMemcpyHostToDevice, ss[b]);
        if (e != cudaSuccess) return fail((int)e, "H2D: %s", cudaGetErrorString(e));
        rc = edges_impl(dev_in[b], input_kind, input_kind == 1 ? w : wp, nullptr, nullptr,
                        dev_out[b], nullptr, side, nullptr, 32, wp, k, h, w, fill_bit, 0, k * h,
                        ss[b]);
        if (rc) return rc;
        e = cudaMemcpyAsync((char *)host_out + lo * out_img, dev_out[b], k * out_img,
                            cudaMemcpyDeviceToHost, ss[b]);
        if (e != cudaSuccess) return fail((int)e, "D2H: %s", cudaGetErrorString(e));
    }
    if (blocking) {
        for (int b = 0; b < 2; ++b) {
            cudaError_t e = cudaStreamSynchronize(ss[b]);
            if (e != cudaSuccess) return fail((int)e, "sync: %s", cudaGetErrorString(e));
        }
    }
    return BE_OK;
}

// Completion wait of the drop-in's one-call flows (a few microseconds of GPU
// work per call, then the host reads the result): spin on an event query rather
// than cudaStreamSynchronize, whose wake-up under the default scheduling mode
// cost ~6 us of the ~15 us C1/C2 call on the B200 box (scripts/dropin_breakdown.py).
// BITEDGE_SYNC_BLOCK=1 restores cudaStreamSynchronize (A/B).
static cudaError_t wait_stream_spin(cudaStream_t st) {
    if (knob(KN_SYNC_BLOCK)) return cudaStreamSynchronize(st);
    thread_local cudaEvent_t ev = nullptr;
    if (ev == nullptr) {
        cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaEventRecord(ev, st);
    if (e != cudaSuccess) return e;
    while ((e = cudaEventQuery(ev)) == cudaErrorNotReady) {
    }
    return e;
}

int be_host_detect_u64(const uint8_t *host_pix, int64_t h, int64_t w, int fill_bit,
                       int emit_edgeset, uint8_t *dev_pix_or_null, uint64_t *dev_packed_or_null,
                       uint64_t *dev_out_or_null, uint64_t *host_out, void *stream) {
    Geometry G;
    int rc = make_geometry(G, 64, 1, h, w, fill_bit);
    if (rc) return rc;
    if (!host_pix || !host_out) return fail(BE_EINVAL, "host buffers must not be NULL");
    const bool zc = dev_pix_or_null == nullptr || dev_out_or_null == nullptr;
    if (zc && w >= 1024)
        return fail(BE_EINVAL, "zero-copy host access (NULL dev_pix / dev_out) needs w < 1024");
    // the kernel may only touch page-locked (mapped) host memory: refuse anything
    // else here rather than fault on the device
    auto pinned = [](const void *p) {
        cudaPointerAttributes a;
        if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return a.type == cudaMemoryTypeHost;
    };
    if (!dev_pix_or_null && !pinned(host_pix))
        return fail(BE_EINVAL, "zero-copy input must be page-locked host memory");
    if (!dev_out_or_null && !pinned(host_out))
        return fail(BE_EINVAL, "zero-copy output must be page-locked host memory");
    const int64_t wp = G.wp / 2;                                 // uint64 words per row
    cudaStream_t st = S(stream);
    const uint8_t *src = host_pix;                               // zero-copy: read over PCIe
    if (dev_pix_or_null) {
        cudaError_t e = cudaMemcpyAsync(dev_pix_or_null, host_pix, (size_t)h * w,
                                        cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) return fail((int)e, "H2D: %s", cudaGetErrorString(e));
        src = dev_pix_or_null;
    }
    uint64_t *dst = dev_out_or_null ? dev_out_or_null : host_out;   // zero-copy: write over PCIe
    uint32_t *side[4] = {nullptr, nullptr, nullptr, nullptr};
    // one launch: pack (bitimage.py:122-136) + edges, uint64 words
    rc = edges_impl(src, 1, w, nullptr, nullptr, emit_edgeset ? nullptr : (uint32_t *)dst,
                    emit_edgeset ? (uint32_t *)dst : nullptr, side,
                    (uint32_t *)dev_packed_or_null, 64, wp, 1, h, w, fill_bit, 0, h, st);
    if (rc) return rc;
    if (dev_out_or_null) {
        cudaError_t e = cudaMemcpyAsync(host_out, dev_out_or_null, (size_t)h * wp * 8,
                                        cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) return fail((int)e, "D2H: %s", cudaGetErrorString(e));
    }
    cudaError_t e = wait_stream_spin(st);
    if (e != cudaSuccess) return fail((int)e, "sync: %s", cudaGetErrorString(e));
    return BE_OK;
}

int be_host_detect_u64_staged(const uint8_t *pix, int64_t pix_row_stride, int64_t h, int64_t w,
                              int fill_bit, int emit_edgeset, uint8_t *stage_in,
                              int64_t stage_in_bytes, uint64_t *stage_out,
                              int64_t stage_out_bytes, uint8_t *dev_stage_or_null,
                              uint64_t *words_out, void *stream) {
    Geometry G;
    int rc = make_geometry(G, 64, 1, h, w, fill_bit);
    if (rc) return rc;
    if (!pix || !stage_in || !stage_out || !words_out)
        return fail(BE_EINVAL, "buffers must not be NULL");
    if (w >= 1024) return fail(BE_EINVAL, "the staged zero-copy flow needs w < 1024");
    if (pix_row_stride < w) return fail(BE_EINVAL, "pixel row stride < width");
    const int64_t wp = G.wp / 2;                                 // uint64 words per row
    if (h * w > stage_in_bytes || h * wp * 8 > stage_out_bytes)
        return fail(BE_EINVAL, "staging buffers too small for a %lldx%lld image",
                    (long long)w, (long long)h);
    // BITEDGE_TRACE_STAGED=1 (experiments): per-phase host time, printed every 2000 calls
    static const bool trace = getenv("BITEDGE_TRACE_STAGED") != nullptr;
    struct timespec ts[5];
    if (trace) clock_gettime(CLOCK_MONOTONIC, &ts[0]);
    // the caller's pixels (any host memory) into the page-locked staging buffer
    if (pix_row_stride == w) {
        memcpy(stage_in, pix, (size_t)(h * w));
    } else {
        for (int64_t y = 0; y < h; ++y)
            memcpy(stage_in + y * w, pix + y * pix_row_stride, (size_t)w);
    }
    if (trace) clock_gettime(CLOCK_MONOTONIC, &ts[1]);
    cudaStream_t st = S(stream);
    uint32_t *side[4] = {nullptr, nullptr, nullptr, nullptr};
    uint32_t *dst = (uint32_t *)stage_out;
    const uint8_t *src = stage_in;
    if (dev_stage_or_null) {
        // larger images: one copy-engine transfer (large PCIe requests) into HBM
        cudaError_t e = cudaMemcpyAsync(dev_stage_or_null, stage_in, (size_t)(h * w),
                                        cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) return fail((int)e, "H2D: %s", cudaGetErrorString(e));
        src = dev_stage_or_null;
    }
    // one launch reading the pixels (mapped page-locked staging over PCIe, or
    // HBM) and writing the words into the mapped page-locked staging buffer:
    // pack (bitimage.py:122-136) + edges, uint64 words
    rc = edges_impl(src, 1, w, nullptr, nullptr, emit_edgeset ? nullptr : dst,
                    emit_edgeset ? dst : nullptr, side, nullptr, 64, wp, 1, h, w, fill_bit, 0, h,
                    st);
    if (rc) return rc;
    if (trace) clock_gettime(CLOCK_MONOTONIC, &ts[2]);
    cudaError_t e = wait_stream_spin(st);
    if (e != cudaSuccess) return fail((int)e, "sync: %s", cudaGetErrorString(e));
    if (trace) clock_gettime(CLOCK_MONOTONIC, &ts[3]);
    memcpy(words_out, stage_out, (size_t)(h * wp * 8));
    if (trace) {
        clock_gettime(CLOCK_MONOTONIC, &ts[4]);
        static thread_local double acc[4];
        static thread_local int calls;
        for (int i = 0; i < 4; ++i)
            acc[i] += (ts[i + 1].tv_sec - ts[i].tv_sec) * 1e6 + (ts[i + 1].tv_nsec - ts[i].tv_nsec) * 1e-3;
        if (++calls == 2000) {
            fprintf(stderr, "[staged %lldx%lld] memcpy_in %.2f  launch %.2f  sync %.2f  memcpy_out %.2f us\n",
                    (long long)w, (long long)h, acc[0] / calls, acc[1] / calls, acc[2] / calls,
                    acc[3] / calls);
            calls = 0;
            for (int i = 0; i < 4; ++i) acc[i] = 0;
        }
    }
    return BE_OK;
}

int be_host_edges_rows(const void *host_in, int input_kind, uint32_t *host_out, int64_t h,
                       int64_t w, int fill_bit, int halo_flags, void *const dev_in[2],
                       uint32_t *const dev_out[2], int64_t chunk_rows, void *stream0,
                       void *stream1, int blocking) {
    Geometry G;
    int rc = make_geometry(G, 32, 1, h, w, fill_bit);
    if (rc) return rc;
    if (!host_in || !host_out || !dev_in || !dev_out || !dev_in[0] || !dev_in[1] || !dev_out[0] ||
        !dev_out[1])
        return fail(BE_EINVAL, "host / device buffers must not be NULL");
    if (input_kind != 0 && input_kind != 1)
        return fail(BE_EINVAL, "input_kind must be 0 (packed u32) or 1 (uint8)");
    if (chunk_rows < 1) return fail(BE_EINVAL, "chunk_rows must be >= 1");
    if (halo_flags & ~3) return fail(BE_EINVAL, "halo_flags must be a combination of 1 and 2");
    const int64_t wp = G.wp;
    const size_t in_row = input_kind == 1 ? (size_t)w : (size_t)wp * 4;
    const size_t out_row = (size_t)wp * 4;
    const bool has_above = halo_flags & 1, has_below = halo_flags & 2;
    // row r of the image is host row r + has_above; rows -1 / h exist iff flagged
    const char *hin = (const char *)host_in + (has_above ? in_row : 0);
    cudaStream_t ss[2] = {S(stream0), S(stream1)};
    uint32_t *side[4] = {nullptr, nullptr, nullptr, nullptr};
    // chunk c on stream c % 2: H2D of rows [r0-1, r1+1) -> halo kernel on rows
    // [r0, r1) -> D2H; in-stream order protects buffer c % 2 for chunk c + 2
    for (int64_t c = 0, r0 = 0; r0 < h; ++c, r0 += chunk_rows) {
        const int64_t r1 = (h - r0) < chunk_rows ? h : r0 + chunk_rows;
        const bool up = r0 > 0 || has_above, dn = r1 < h || has_below;
        const int64_t lo = up ? r0 - 1 : r0, hi = dn ? r1 + 1 : r1;
        const int b = (int)(c & 1);
        char *din = (char *)dev_in[b];
        cudaError_t e = cudaMemcpyAsync(din, hin + lo * (int64_t)in_row, (hi - lo) * in_row,
                                        cudaMemcpyHostToDevice, ss[b]);
        if (e != cudaSuccess) return fail((int)e, "H2D: %s", cudaGetErrorString(e));
        const char *slab = din + (r0 - lo) * in_row;
        const void *above = up ? (const void *)din : nullptr;
        const void *below = dn ? (const void *)(slab + (r1 - r0) * in_row) : nullptr;
        rc = edges_impl(slab, input_kind, input_kind == 1 ? w : wp, above, below, dev_out[b],
                        nullptr, side, nullptr, 32, wp, 1, r1 - r0, w, fill_bit, 0, r1 - r0, ss[b]);
        if (rc) return rc;
        e = cudaMemcpyAsync((char *)host_out + r0 * out_row, dev_out[b], (r1 - r0) * out_row,
                            cudaMemcpyDeviceToHost, ss[b]);
        if (e != cudaSuccess) return fail((int)e, "D2H: %s", cudaGetErrorString(e));
    }
    if (blocking) {
        for (int b = 0; b < 2; ++b) {
            cudaError_t e = cudaStreamSynchronize(ss[b]);
            if (e != cudaSuccess) return fail((int)e, "sync: %s", cudaGetErrorString(e));
        }
    }
    return BE_OK;
}

}  // extern "C"

"""Tensor API over device-resident batches (`bitedge.cuda`).

The reference has no batch type (`from_array` is 2-d only, bitimage.py:126-127);
this is the surface the benchmarks and the multi-GPU layer call.  Every
function launches hand-written sm_100a kernels through the C ABI
(include/bitedge.h) on the current torch stream; there is no CPU path.

Packed rasters are integer tensors of shape [N, H, S] or [H, S]:
  int32 / uint32  -> 32-bit MSB-first row words (BASELINE configs 3 and 4);
  int64 / uint64  -> the reference's native uint64 words (BitImage.words).
S is the row length in words (>= ceil(W / word_bits)); the last dimension
must be contiguous and images contiguous.  Pixel inputs are uint8 / int8 /
bool [N, H, W] (any nonzero byte is white, bitimage.py:124, 133).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

import torch

from . import _capi

WHITE_OUTSIDE = 1
BLACK_OUTSIDE = 0

_WORD_DTYPES = {torch.int32: 32, torch.int64: 64}
for _name, _bits in (("uint32", 32), ("uint64", 64)):
    if hasattr(torch, _name):
        _WORD_DTYPES[getattr(torch, _name)] = _bits
_PIXEL_DTYPES = (torch.uint8, torch.int8, torch.bool)


def fill_bit(border) -> int:
    """BorderPolicy (bitimage.py:56-64) or 0/1 -> fill bit."""
    v = getattr(border, "value", border)
    if v not in (0, 1) or isinstance(v, float):
        raise ValueError(f"border must be a BorderPolicy or 0/1, got {border!r}")
    return int(v)


def _require_cuda(t: torch.Tensor, what: str) -> None:
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{what} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor (there is no CPU path)")


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream(t: torch.Tensor) -> int:
    """The current stream of t's device as an integer handle (the ctypes
    argtypes take ints; the raw getter skips torch.cuda.Stream's ~3 us)."""
    if _raw_stream is not None:
        return _raw_stream(t.get_device())
    return torch.cuda.current_stream(t.device).cuda_stream


def _as3d(t: torch.Tensor, what: str) -> torch.Tensor:
    if t.dim() == 2:
        return t.unsqueeze(0)
    if t.dim() == 3:
        return t
    raise ValueError(f"{what} must be [H, S] or [N, H, S], got shape {tuple(t.shape)}")


def _row_stride(t3: torch.Tensor, what: str) -> int:
    n, h, s = t3.shape
    if s and t3.stride(2) != 1:
        raise ValueError(f"{what}: rows must be contiguous")
    rs = t3.stride(1) if h > 1 else max(s, t3.stride(1))
    if n > 1 and t3.stride(0) != h * rs:
        raise ValueError(f"{what}: images of a batch must be contiguous")
    return rs


def word_bits_of(t: torch.Tensor) -> int:
    try:
        return _WORD_DTYPES[t.dtype]
    except KeyError:
        raise ValueError(f"packed words must be int32/uint32/int64/uint64, got {t.dtype}") from None


def words_per_row(width: int, word_bits: int = 32) -> int:
    return -(-int(width) // word_bits)


def _packed(words: torch.Tensor, width: int, what: str = "words"):
    _require_cuda(words, what)
    wb = word_bits_of(words)
    w3 = _as3d(words, what)
    rs = _row_stride(w3, what)
    if w3.shape[2] < words_per_row(width, wb):
        raise ValueError(f"{what}: width {width} needs {words_per_row(width, wb)} words per row, "
                         f"got {w3.shape[2]}")
    return w3, wb, rs


def _new_like(w3: torch.Tensor, squeeze: bool, rs: int | None = None) -> torch.Tensor:
    """A fresh output for a primitive whose kernel writes out[row * rs + m] with
    the INPUT's row stride rs: allocated [N, H, rs] and viewed as [N, H, S], so a
    strided input view (rs > S) gets an output of the same geometry."""
    n, h, s = w3.shape
    rs = s if rs is None else rs
    out = torch.empty((n, h, rs), dtype=w3.dtype, device=w3.device)
    if rs != s:
        out = out[..., :s]
    return out[0] if squeeze else out


def _check_out(out: torch.Tensor, ref3: torch.Tensor, squeeze: bool, what="out"):
    _require_cuda(out, what)
    o3 = _as3d(out, what)
    if o3.shape != ref3.shape or o3.dtype != ref3.dtype:
        raise ValueError(f"{what} must have shape {tuple(ref3.shape)} and dtype {ref3.dtype}")
    return o3


def _ptr(t):
    return None if t is None else t.data_ptr()


# ------------------------------------------------------------------ hot path

def _dims(t: torch.Tensor, what: str):
    """(n, h, s, row_stride) of a [H, S] / [N, H, S] tensor without building
    views -- the same rules as _as3d + _row_stride, on the per-call hot path."""
    d = t.dim()
    if d == 2:
        n = 1
        h, s = t.shape
        sh, ss = t.stride()
        sn = 0
    elif d == 3:
        n, h, s = t.shape
        sn, sh, ss = t.stride()
    else:
        raise ValueError(f"{what} must be [H, S] or [N, H, S], got shape {tuple(t.shape)}")
    if s and ss != 1:
        raise ValueError(f"{what}: rows must be contiguous")
    rs = sh if h > 1 else max(s, sh)
    if n > 1 and sn != h * rs:
        raise ValueError(f"{what}: images of a batch must be contiguous")
    return n, h, s, rs


def edges_packed(words: torch.Tensor, width: int, border=WHITE_OUTSIDE, *, out=None,
                 edgeset: bool = False) -> torch.Tensor:
    """detect_edges_mask -- or the EdgeSet
    when `edgeset` -- of packed rasters, in one fused pass (kernel K1)."""
    _require_cuda(words, "words")
    wb = word_bits_of(words)
    n, h, s, rs = _dims(words, "words")
    width = int(width)
    if s < -(-width // wb):
        raise ValueError(f"words: width {width} needs {words_per_row(width, wb)} words per row, "
                         f"got {s}")
    fb = fill_bit(border)
    if out is None:
        o = torch.empty(words.shape, dtype=words.dtype, device=words.device)
        ors = s
    else:
        o = out
        o3 = _check_out(o, _as3d(words, "words"), words.dim() == 2)
        ors = _row_stride(o3, "out")
    if ors != rs:   # different input / output strides: the general entry point
        outs = _capi.be_outputs()
        if edgeset:
            outs.edgeset = o.data_ptr()
        else:
            outs.edges = o.data_ptr()
        _capi.call("be_edges_general", words.data_ptr(), 0, rs, None, None, ctypes.byref(outs), wb,
                   ors, n, h, width, fb, 0, n * h, _stream(words))
        return o
    rc = (_capi.fn("be_edge_packed_u64") if wb == 64 else _capi.fn("be_edge_packed_u32"))(
        words.data_ptr(), o.data_ptr(), n, h, width, rs, fb, int(edgeset), _stream(words))
    if rc:
        _capi.check(rc)
    return o


def pack_and_edges(pixels: torch.Tensor, border=WHITE_OUTSIDE, *, word_bits: int = 64,
                   edgeset: bool = False):
    """from_array + detect_edges_mask (or edge_set when `edgeset`) in ONE launch
    that also writes the packed input: returns (edges, packed) in `word_bits`
    words.  The drop-in BitImage uses it to fuse a deferred pack into edge
    detection."""
    _require_cuda(pixels, "pixels")
    if pixels.dtype not in _PIXEL_DTYPES:
        raise ValueError(f"pixels must be uint8/int8/bool (nonzero = white), got {pixels.dtype}")
    n, h, w, prs = _dims(pixels, "pixels")
    if w < 1 or h < 1:
        raise ValueError(f"image dimensions must be at least 1x1, got {w}x{h}")
    wp = -(-w // word_bits)
    dt = torch.int64 if word_bits == 64 else torch.int32
    shape = (n, h, wp) if pixels.dim() == 3 else (h, wp)
    e = torch.empty(shape, dtype=dt, device=pixels.device)
    pk = torch.empty(shape, dtype=dt, device=pixels.device)
    o = _capi.be_outputs()
    if edgeset:
        o.edgeset = e.data_ptr()
    else:
        o.edges = e.data_ptr()
    o.packed = pk.data_ptr()
    rc = _capi.fn("be_edges_general")(pixels.data_ptr(), 1, prs, None, None, ctypes.byref(o),
                                      word_bits, wp, n, h, w, fill_bit(border), 0, n * h,
                                      _stream(pixels))
    if rc:
        _capi.check(rc)
    return e, pk


# zero-copy bound for host_detect: the kernel reads / writes host memory over
# PCIe itself, which beats the copy operations' fixed latency for small images
_ZERO_COPY_BYTES = 1 << 20


def host_detect(host_pixels: torch.Tensor, border=WHITE_OUTSIDE, *, edgeset: bool = False,
                device=None, zero_copy: bool | None = None):
    """One host image through `be_host_detect_u64`: page-locked uint8 pixels
    [H, W] (nonzero = white) -> (edges, packed, words): the edges as CUDA int64
    BitImage words (None when the kernel wrote them straight to the host), the
    packed input as CUDA int64 words, and the edges as a read-only host uint64
    array -- from one call that uploads, packs + detects in one kernel,
    downloads and waits (the drop-in's `detect_edges_mask(BitImage.from_array(a)).words`).
    `zero_copy` (default: images up to 1 MiB, narrower than 1024 px): the kernel
    reads the pixels and writes the words over PCIe itself, no copy operations."""
    if host_pixels.is_cuda or not host_pixels.is_pinned() or host_pixels.dim() != 2 or \
            host_pixels.dtype != torch.uint8 or not host_pixels.is_contiguous():
        raise ValueError("host_pixels must be a contiguous page-locked uint8 [H, W] host tensor")
    h, w = host_pixels.shape
    if w < 1 or h < 1:
        raise ValueError(f"image dimensions must be at least 1x1, got {w}x{h}")
    if zero_copy is None:
        zero_copy = h * w <= _ZERO_COPY_BYTES and w < 1024
    dev = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    wp = -(-w // 64)
    packed = torch.empty((h, wp), dtype=torch.int64, device=dev)
    host = torch.empty((h, wp), dtype=torch.int64, pin_memory=True)
    if zero_copy:
        dpix = out = None
    else:
        dpix = torch.empty((h, w), dtype=torch.uint8, device=dev)
        out = torch.empty((h, wp), dtype=torch.int64, device=dev)
    rc = _capi.fn("be_host_detect_u64")(host_pixels.data_ptr(), h, w, fill_bit(border),
                                        1 if edgeset else 0,
                                        None if dpix is None else dpix.data_ptr(), packed.data_ptr(),
                                        None if out is None else out.data_ptr(), host.data_ptr(),
                                        _stream(packed))
    if rc:
        _capi.check(rc)
    words = host.numpy().view(np.uint64)
    words.setflags(write=False)
    return out, packed, words


# the drop-in's small-image flow (be_host_detect_u64_staged): one page-locked
# staging pair (plus one device staging buffer) per calling thread, reused by
# every call -- a fixed footprint however many images are in flight in Python
SMALL_MAX_PIXELS = 1 << 20
_tls = threading.local()
_staged_fn = None
_get_device = getattr(torch._C, "_cuda_getDevice", None)


class _Stage:
    __slots__ = ("pin_in", "pin_out", "in_ptr", "in_n", "out_ptr", "out_n", "device")

    def __init__(self, in_bytes, out_bytes, device):
        self.pin_in = torch.empty(in_bytes, dtype=torch.uint8, pin_memory=True)
        self.pin_out = torch.empty(out_bytes, dtype=torch.uint8, pin_memory=True)
        self.in_ptr, self.in_n = self.pin_in.data_ptr(), in_bytes
        self.out_ptr, self.out_n = self.pin_out.data_ptr(), out_bytes
        self.device = device


def _staging(in_bytes: int, out_bytes: int, device: int) -> _Stage:
    """This thread's page-locked staging pair for the ctypes path (grown on demand)."""
    st = getattr(_tls, "stage", None)
    if st is None or st.device != device or st.in_n < in_bytes or st.out_n < out_bytes:
        keep = (0, 0) if st is None or st.device != device else (st.in_n, st.out_n)
        st = _Stage(max(in_bytes, keep[0], 64 << 10), max(out_bytes, keep[1], 16 << 10), device)
        _tls.stage = st
    return st


try:  # CPython binding of the same call (csrc/dropin_ext.c): ~4 us less per call
    from . import _dropin
except ImportError:  # pragma: no cover - the ctypes path below runs the same kernel
    _dropin = None


def _dropin_stage(in_bytes: int, out_bytes: int, device: int) -> None:
    """(Re)allocate this thread's staging pair + private stream and register it
    with the CPython binding."""
    st = getattr(_tls, "ext_stage", None)
    if st is not None and st[5] == device:
        in_bytes, out_bytes = max(in_bytes, st[1]), max(out_bytes, st[3])
    pin_in = torch.empty(max(in_bytes, 64 << 10), dtype=torch.uint8, pin_memory=True)
    pin_out = torch.empty(max(out_bytes, 16 << 10), dtype=torch.uint8, pin_memory=True)
    stream = torch.cuda.Stream(torch.device("cuda", device))
    _tls.ext_stage = (pin_in, pin_in.numel(), pin_out, pin_out.numel(), stream, device)
    _dropin.set_stage(pin_in.data_ptr(), pin_in.numel(), pin_out.data_ptr(), pin_out.numel(),
                      stream.cuda_stream, device)


def host_detect_small(pix: np.ndarray, border=WHITE_OUTSIDE, *, edgeset: bool = False) -> np.ndarray:
    """`detect_edges_mask(BitImage.from_array(a)).words` for a small host image
    in ONE native call (`be_host_detect_u64_staged`): uint8 pixels [H, W] in any
    host memory (nonzero = white; W < 1024, H*W <= SMALL_MAX_PIXELS) -> a fresh
    read-only uint64 words array [H, ceil(W/64)].  The pixels go through this
    thread's page-locked staging pair; one kernel packs and detects, reading the
    pixels and writing the words over PCIe (a copy-engine transfer of the pixels
    was slower at every size up to 1 Mpx, scripts/dropin_breakdown.py)."""
    global _staged_fn
    if _dropin is not None:
        fb = getattr(border, "value", border)
        if fb != 0 and fb != 1:
            fb = fill_bit(border)
        dev = _get_device() if _get_device is not None else torch.cuda.current_device()
        es = 1 if edgeset else 0
        r = _dropin.detect_small(pix, fb, es, dev)
        if r is None:
            h, w = pix.shape
            if w >= 1024 or h * w > SMALL_MAX_PIXELS:
                raise ValueError("host_detect_small takes images narrower than 1024 px, <= 1 Mpx")
            _dropin_stage(h * w, h * ((w + 63) >> 6) * 8 + 128, dev)
            r = _dropin.detect_small(pix, fb, es, dev)
        return r
    if pix.ndim != 2 or pix.dtype != np.uint8 or pix.strides[1] != 1:
        raise ValueError("pix must be a uint8 [H, W] array with contiguous rows")
    h, w = pix.shape
    if w >= 1024 or h * w > SMALL_MAX_PIXELS:
        raise ValueError("host_detect_small takes images narrower than 1024 px, <= 1 Mpx")
    fb = getattr(border, "value", border)
    if fb != 0 and fb != 1:
        fb = fill_bit(border)
    dev = _get_device() if _get_device is not None else torch.cuda.current_device()
    n = h * w
    wp = (w + 63) >> 6
    st = getattr(_tls, "stage", None)
    if st is None or st.device != dev or st.in_n < n or st.out_n < h * wp * 8 + 128:
        st = _staging(n, h * wp * 8 + 128, dev)
    words = np.empty((h, wp), dtype=np.uint64)
    if _staged_fn is None:
        _staged_fn = _capi.fn("be_host_detect_u64_staged")
    rc = _staged_fn(pix.ctypes.data, pix.strides[0], h, w, fb, 1 if edgeset else 0,
                    st.in_ptr, st.in_n, st.out_ptr, st.out_n, None,
                    words.ctypes.data,
                    _raw_stream(dev) if _raw_stream is not None
                    else torch.cuda.current_stream(dev).cuda_stream)
    if rc:
        _capi.check(rc)
    words.flags.writeable = False
    return words


def _pixels(pixels: torch.Tensor, what="pixels"):
    _require_cuda(pixels, what)
    if pixels.dtype not in _PIXEL_DTYPES:
        raise ValueError(f"{what} must be uint8/int8/bool (nonzero = white), got {pixels.dtype}")
    p3 = _as3d(pixels, what)
    if p3.shape[2] < 1 or p3.shape[1] < 1:
        raise ValueError(f"image dimensions must be at least 1x1, got {p3.shape[2]}x{p3.shape[1]}")
    return p3, _row_stride(p3, what)


def pack_edges_u8(pixels: torch.Tensor, border=WHITE_OUTSIDE, *, out=None,
                  packed_out: torch.Tensor | None = None) -> torch.Tensor:
    """from_array + detect_edges_mask fused (kernel K2): uint8 [N,H,W] ->
    int32 [N,H,ceil(W/32)] MSB-first edge words.  `packed_out` (same shape)
    additionally receives the packed input."""
    squeeze = pixels.dim() == 2
    p3, prs = _pixels(pixels)
    n, h, w = p3.shape
    shape = (n, h, words_per_row(w, 32))
    o = out if out is not None else torch.empty(shape, dtype=torch.int32, device=p3.device)
    o3 = _as3d(o, "out")
    _require_cuda(o3, "out")
    if tuple(o3.shape) != shape or word_bits_of(o3) != 32:
        raise ValueError(f"out must be 32-bit words of shape {shape}")
    ors = _row_stride(o3, "out")
    pk = None
    if packed_out is not None:
        pk = _as3d(packed_out, "packed_out")
        if tuple(pk.shape) != shape or word_bits_of(pk) != 32 or _row_stride(pk, "packed_out") != ors:
            raise ValueError("packed_out must match out")
    _capi.call("be_pack_edge_u8", _ptr(p3), _ptr(o3), n, h, w, prs, ors, fill_bit(border), _ptr(pk),
               _stream(p3))
    return o[0] if (squeeze and out is None) else o


def threshold_edges_u8(gray: torch.Tensor, threshold: int, border=WHITE_OUTSIDE, *, out=None,
                       binary_out: torch.Tensor | None = None) -> torch.Tensor:
    """binarize.threshold (sample >= t -> white) fused with
    detect_edges_mask: uint8 luminance [N,H,W] -> int32 edge words, one pass
    (SURVEY 8(f) F2).  `binary_out` additionally receives the binarised raster."""
    t = int(threshold)
    if not 0 <= t <= 255:
        raise ValueError(f"threshold must be 0..255, got {threshold}")
    squeeze = gray.dim() == 2
    p3, prs = _pixels(gray, "gray")
    if p3.dtype != torch.uint8:
        raise ValueError("gray must be uint8 luminance")
    n, h, w = p3.shape
    shape = (n, h, words_per_row(w, 32))
    o = out if out is not None else torch.empty(shape, dtype=torch.int32, device=p3.device)
    o3 = _as3d(o, "out")
    if tuple(o3.shape) != shape or word_bits_of(o3) != 32:
        raise ValueError(f"out must be 32-bit words of shape {shape}")
    ors = _row_stride(o3, "out")
    bo = None
    if binary_out is not None:
        bo = _as3d(binary_out, "binary_out")
        if tuple(bo.shape) != shape or word_bits_of(bo) != 32 or _row_stride(bo, "binary_out") != ors:
            raise ValueError("binary_out must match out")
    _capi.call("be_threshold_edge_u8", _ptr(p3), _ptr(o3), n, h, w, prs, ors, t, fill_bit(border),
               _ptr(bo), _stream(p3))
    return o[0] if (squeeze and out is None) else o


def threshold_u8(gray: torch.Tensor, threshold: int, word_bits: int = 32) -> torch.Tensor:
    """binarize.threshold on the device: packed raster."""
    t = int(threshold)
    if not 0 <= t <= 255:
        raise ValueError(f"threshold must be 0..255, got {threshold}")
    squeeze = gray.dim() == 2
    p3, prs = _pixels(gray, "gray")
    n, h, w = p3.shape
    shape = (n, h, words_per_row(w, word_bits))
    o = torch.empty(shape, dtype=torch.int64 if word_bits == 64 else torch.int32, device=p3.device)
    _capi.call("be_threshold_u8", _ptr(p3), _ptr(o), word_bits, n, h, w, prs,
               _row_stride(o, "out"), t, _stream(p3))
    return o[0] if squeeze else o


def edges_general(inp: torch.Tensor, width: int | None = None, border=WHITE_OUTSIDE, *,
                  word_bits: int = 32, edges=True, edgeset=False, sides=False, packed=False,
                  above=None, below=None, row_lo: int = 0, row_hi: int | None = None,
                  outs: dict | None = None) -> dict:
    """Every output of the fused kernel from one read of the input (F3):
    'edges', 'edgeset', 'left'/'right'/'up'/'down' fundamental edges
     and 'packed'.  `inp` is packed words or uint8 pixels."""
    _require_cuda(inp, "input")
    if inp.dtype in _PIXEL_DTYPES:
        p3, irs = _pixels(inp, "input")
        kind = 1
        n, h, width = p3.shape
        wb = word_bits
        src = p3
    else:
        if width is None:
            raise ValueError("width is required for packed input")
        src, wb, irs = _packed(inp, width, "input")
        kind = 0
        n, h, _ = src.shape
    shape = (n, h, words_per_row(width, wb))
    dt = torch.int64 if wb == 64 else torch.int32
    names = []
    if edges:
        names.append("edges")
    if edgeset:
        names.append("edgeset")
    if sides:
        names += ["left", "right", "up", "down"]
    if packed:
        names.append("packed")
    res = dict(outs or {})
    for k in names:
        if k not in res:
            res[k] = torch.empty(shape, dtype=dt, device=src.device)
    ors = None
    for k, v in res.items():
        v3 = _as3d(v, k)
        if tuple(v3.shape) != shape or word_bits_of(v3) != wb:
            raise ValueError(f"output {k} must be {wb}-bit words of shape {shape}")
        r = _row_stride(v3, k)
        if ors is None:
            ors = r
        elif r != ors:
            raise ValueError("all outputs must share one row stride")
    o = _capi.be_outputs()
    o.edges = res["edges"].data_ptr() if "edges" in res else None
    o.edgeset = res["edgeset"].data_ptr() if "edgeset" in res else None
    for i, k in enumerate(("left", "right", "up", "down")):
        o.side[i] = res[k].data_ptr() if k in res else None
    o.packed = res["packed"].data_ptr() if "packed" in res else None
    if row_hi is None:
        row_hi = n * h
    _capi.call("be_edges_general", _ptr(src), kind, irs, _ptr(above), _ptr(below),
               ctypes.byref(o), wb, ors, n, h, int(width), fill_bit(border), int(row_lo),
               int(row_hi), _stream(src))
    return res


def edges_halo(slab: torch.Tensor, above, below, width: int, border=WHITE_OUTSIDE, *, out=None,
               row_lo: int = 0, row_hi: int | None = None) -> torch.Tensor:
    """Kernel K3: edges of a row slab [rows, S] (int32 words) whose row -1 /
    row `rows` are the neighbour slabs' boundary rows (`above` / `below`,
    [S] tensors with the slab's stride, or None at the image border)."""
    _require_cuda(slab, "slab")
    if slab.dim() != 2 or word_bits_of(slab) != 32:
        raise ValueError("slab must be a 2-d 32-bit word tensor")
    w3, wb, rs = _packed(slab, width, "slab")
    rows = slab.shape[0]
    for t, nm in ((above, "above"), (below, "below")):
        if t is not None:
            _require_cuda(t, nm)
            if t.dtype != slab.dtype or t.numel() < slab.shape[1] or t.stride(-1) != 1:
                raise ValueError(f"{nm} must be one contiguous row of the slab's dtype")
    o = torch.empty_like(slab) if out is None else out
    if o.shape != slab.shape or o.dtype != slab.dtype or o.stride() != slab.stride():
        raise ValueError("out must match the slab")
    if row_hi is None:
        row_hi = rows
    _capi.call("be_edge_packed_halo_u32", _ptr(slab), _ptr(above), _ptr(below), _ptr(o), rows,
               int(width), rs, fill_bit(border), int(row_lo), int(row_hi),
               _stream(slab))
    return o


def edges_halo_ends(slab: torch.Tensor, above, below, width: int, border=WHITE_OUTSIDE, *,
                    out) -> torch.Tensor:
    """Kernel K3e: output rows 0 and rows-1 of a row slab only -- the two rows
    that read a halo -- in one launch (`edges_halo` with the rows {0, rows-1});
    `out` must already hold (or later receive) the interior rows."""
    _require_cuda(slab, "slab")
    if slab.dim() != 2 or word_bits_of(slab) != 32:
        raise ValueError("slab must be a 2-d 32-bit word tensor")
    w3, wb, rs = _packed(slab, width, "slab")
    for t, nm in ((above, "above"), (below, "below")):
        if t is not None:
            _require_cuda(t, nm)
            if t.dtype != slab.dtype or t.numel() < slab.shape[1] or t.stride(-1) != 1:
                raise ValueError(f"{nm} must be one contiguous row of the slab's dtype")
    if out.shape != slab.shape or out.dtype != slab.dtype or out.stride() != slab.stride():
        raise ValueError("out must match the slab")
    _capi.call("be_edge_packed_halo_ends_u32", _ptr(slab), _ptr(above), _ptr(below), _ptr(out),
               slab.shape[0], int(width), rs, fill_bit(border), _stream(slab))
    return out


# ------------------------------------------------------------------ primitives

def pack_u8(pixels: torch.Tensor, word_bits: int = 32, out=None) -> torch.Tensor:
    """BitImage.from_array (bitimage.py:122-136) on the device."""
    _require_cuda(pixels, "pixels")
    if pixels.dtype not in _PIXEL_DTYPES:
        raise ValueError(f"pixels must be uint8/int8/bool (nonzero = white), got {pixels.dtype}")
    n, h, w, prs = _dims(pixels, "pixels")
    if w < 1 or h < 1:
        raise ValueError(f"image dimensions must be at least 1x1, got {w}x{h}")
    wp = -(-w // word_bits)
    dt = torch.int64 if word_bits == 64 else torch.int32
    if out is None:
        shape = (n, h, wp) if pixels.dim() == 3 else (h, wp)
        o = torch.empty(shape, dtype=dt, device=pixels.device)
        ors = wp
    else:
        o = out
        o3 = _as3d(o, "out")
        if tuple(o3.shape) != (n, h, wp) or word_bits_of(o3) != word_bits:
            raise ValueError(f"out must be {word_bits}-bit words of shape {(n, h, wp)}")
        ors = _row_stride(o3, "out")
    rc = _capi.fn("be_pack_u8")(pixels.data_ptr(), o.data_ptr(), word_bits, n, h, w, prs, ors,
                                _stream(pixels))
    if rc:
        _capi.check(rc)
    return o


def unpack_u8(words: torch.Tensor, width: int, out=None) -> torch.Tensor:
    """BitImage.to_array (bitimage.py:149-153) on the device: uint8 {0,1}."""
    squeeze = words.dim() == 2
    w3, wb, rs = _packed(words, width)
    n, h, _ = w3.shape
    o = out if out is not None else torch.empty((n, h, int(width)), dtype=torch.uint8,
                                                device=w3.device)
    o3 = _as3d(o, "out")
    if tuple(o3.shape) != (n, h, int(width)) or o3.dtype != torch.uint8:
        raise ValueError("out must be uint8 [N, H, W]")
    _capi.call("be_unpack_u8", _ptr(w3), _ptr(o3), wb, n, h, int(width), rs,
               _row_stride(o3, "out"), _stream(w3))
    return o[0] if (squeeze and out is None) else o


def _binary(name, op, a, b, width):
    squeeze = a.dim() == 2
    a3, wb, rs = _packed(a, width, "a")
    b3 = None
    if b is not None:
        b3, wb2, rs2 = _packed(b, width, "b")
        if b3.shape != a3.shape or wb2 != wb or rs2 != rs:
            raise ValueError("operands must have identical shape, dtype and stride")
    o = _new_like(a3, squeeze, rs)
    o3 = _as3d(o, "out")
    n, h, _ = a3.shape
    _capi.call("be_bitop", op, _ptr(a3), _ptr(b3), _ptr(o3), wb, n, h,
               int(width), rs, _stream(a3))
    return o


def invert(words, width):
    return _binary("invert", _capi.BE_OP_NOT, words, None, width)


def and_(a, b, width):
    return _binary("and", _capi.BE_OP_AND, a, b, width)


def or_(a, b, width):
    return _binary("or", _capi.BE_OP_OR, a, b, width)


def shift(words, width, direction: int, border=WHITE_OUTSIDE):
    """BitImage.shift (bitimage.py:207-240); direction BE_LEFT..BE_DOWN."""
    squeeze = words.dim() == 2
    w3, wb, rs = _packed(words, width)
    o = _new_like(w3, squeeze, rs)
    n, h, _ = w3.shape
    _capi.call("be_shift", _ptr(w3), _ptr(_as3d(o, "out")), wb, n, h, int(width), rs, int(direction),
               fill_bit(border), _stream(w3))
    return o


def shift_and(img, mask, width, side: int, border=WHITE_OUTSIDE):
    """fundamental_edge(img, mask, side) = shift(img, opposite(side)) & mask, fused."""
    squeeze = img.dim() == 2
    i3, wb, rs = _packed(img, width, "img")
    m3, wb2, rs2 = _packed(mask, width, "mask")
    if m3.shape != i3.shape or wb2 != wb or rs2 != rs:
        raise ValueError("img and mask must have identical shape, dtype and stride")
    o = _new_like(i3, squeeze, rs)
    n, h, _ = i3.shape
    _capi.call("be_shift_and", _ptr(i3), _ptr(m3), _ptr(_as3d(o, "out")), wb, n, h, int(width), rs,
               int(side), fill_bit(border), _stream(i3))
    return o


def count_black(words, width) -> torch.Tensor:
    """BitImage.count_black (bitimage.py:244-249) per image: int64 [N]."""
    w3, wb, rs = _packed(words, width)
    n, h, _ = w3.shape
    counts = torch.empty(n, dtype=torch.int64, device=w3.device)
    _capi.call("be_count_black", _ptr(w3), _ptr(counts), wb, n, h, int(width), rs,
               _stream(w3))
    return counts


def scan_edges(words, width, border=WHITE_OUTSIDE, *, out=None):
    """detect_edges_scan: per-pixel Edge(p) on the device."""
    squeeze = words.dim() == 2
    w3, wb, rs = _packed(words, width)
    if out is None:
        o = _new_like(w3, squeeze, rs)
    else:
        o = out
        if _row_stride(_check_out(o, w3, squeeze), "out") != rs:
            raise ValueError("out must have the input's row stride")
    n, h, _ = w3.shape
    _capi.call("be_scan_edges", _ptr(w3), _ptr(_as3d(o, "out")), wb, n, h, int(width), rs,
               fill_bit(border), _stream(w3))
    return o

"""PBM at the kernel boundary (reference: SPEC.md:273-316,
module `imageio` not shipped).

PBM stores 1 = black, MSB-first, rows padded to whole bytes; the rasters here
are 1 = white.  The inversion is absorbed at this boundary only.
Header parsing is host work; the P4 payload goes straight to the device and
is decoded / encoded by kernels -- and `detect_pbm` runs file -> GPU -> file
with kernel K1 reading and writing P4 bytes directly when the rows allow it.

    read_pbm(data) -> BitImage            P1 (ASCII) or P4 (raw)
    write_pbm(img, raw=True) -> bytes     P4 (padding bits written 0) or P1
    detect_pbm(data, border, raw=True)    edges of a PBM file, as a PBM file
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _capi
from .bitimage import BitImage, BorderPolicy, _device, _torch

_WS = b" \t\r\n\v\f"


def parse_header(data: bytes):
    """-> (magic, width, height, payload_offset).  Comments ('#' to end of line)
    are skipped; exactly one whitespace byte separates the height from a raw
    payload."""
    if len(data) < 2 or data[:1] != b"P" or data[1:2] not in (b"1", b"4"):
        raise ValueError("not a PBM file (magic P1/P4 expected) at offset 0")
    magic = data[:2].decode()
    pos = 2
    vals = []
    while len(vals) < 2:
        while pos < len(data) and (data[pos] in _WS or data[pos:pos + 1] == b"#"):
            if data[pos:pos + 1] == b"#":
                while pos < len(data) and data[pos] not in b"\r\n":
                    pos += 1
            else:
                pos += 1
        start = pos
        while pos < len(data) and data[pos:pos + 1].isdigit():
            pos += 1
        if start == pos:
            raise ValueError(f"malformed PBM header: expected a dimension at offset {start}")
        v = int(data[start:pos])
        if v < 1:
            raise ValueError(f"image dimensions must be at least 1x1 (offset {start})")
        vals.append(v)
    if pos >= len(data) or data[pos] not in _WS:
        raise ValueError(f"malformed PBM header: expected whitespace at offset {pos}")
    return magic, vals[0], vals[1], pos + 1


def _payload_tensor(data: bytes, offset: int, nbytes: int):
    torch = _torch()
    if len(data) - offset < nbytes:
        raise ValueError(f"short PBM payload: need {nbytes} bytes at offset {offset}, "
                         f"have {len(data) - offset}")
    host = torch.frombuffer(bytearray(data[offset:offset + nbytes]), dtype=torch.uint8)
    return host.to(_device())


def _stream():
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def read_pbm(data: bytes) -> BitImage:
    """PBM bytes -> BitImage."""
    magic, w, h, off = parse_header(data)
    if magic == "P4":
        rb = (w + 7) // 8
        payload = _payload_tensor(data, off, rb * h)
        torch = _torch()
        words = torch.empty((h, (w + 63) // 64), dtype=torch.int64, device=payload.device)
        _capi.call("be_p4_decode", ctypes.c_void_p(payload.data_ptr()),
                   ctypes.c_void_p(words.data_ptr()), 64, 1, h, w, words.shape[1], _stream())
        return BitImage._wrap(w, h, words)
    # P1: ASCII '0'/'1' tokens, whitespace optional between them
    body = data[off:]
    digits = np.frombuffer(body, dtype=np.uint8)
    keep = digits[(digits == ord("0")) | (digits == ord("1"))]
    if keep.size < w * h:
        raise ValueError(f"short PBM payload: need {w * h} samples after offset {off}, "
                         f"have {keep.size}")
    black = (keep[: w * h] == ord("1")).reshape(h, w)
    return BitImage.from_array((~black).astype(np.uint8))


def write_pbm(img: BitImage, raw: bool = True) -> bytes:
    """BitImage -> PBM bytes; P4 rows padded with 0 bits."""
    head = f"{'P4' if raw else 'P1'}\n{img.width} {img.height}\n".encode()
    if raw:
        torch = _torch()
        rb = (img.width + 7) // 8
        out = torch.empty(rb * img.height, dtype=torch.uint8, device=_device())
        _capi.call("be_p4_encode", ctypes.c_void_p(img.device_words().data_ptr()),
                   ctypes.c_void_p(out.data_ptr()), 64, 1, img.height, img.width,
                   img.words_per_row, _stream())
        return head + out.cpu().numpy().tobytes()
    black = 1 - img.to_array()
    lines = [" ".join(str(int(b)) for b in row) for row in black]
    return head + ("\n".join(lines) + "\n").encode()


def detect_p4(payload, n: int, h: int, w: int, border=BorderPolicy.WHITE_OUTSIDE, *, out=None):
    """Edges of a batch of P4 payloads already in HBM (uint8 tensor of
    n * h * ceil(w/8) bytes) -> P4 payload tensor of the same size (`out`, if
    given: a contiguous CUDA uint8 tensor of that many bytes)."""
    torch = _torch()
    rb = (w + 7) // 8
    if payload.numel() != n * h * rb or payload.dtype != torch.uint8 or not payload.is_cuda:
        raise ValueError(f"payload must be a CUDA uint8 tensor of {n * h * rb} bytes")
    if out is None:
        out = torch.empty_like(payload)
    elif (out.numel() != payload.numel() or out.dtype != torch.uint8 or not out.is_cuda
          or not out.is_contiguous()):
        raise ValueError(f"out must be a contiguous CUDA uint8 tensor of {n * h * rb} bytes")
    scratch = None
    if rb % 16 != 0 or os.environ.get("BITEDGE_P4_UNFUSED"):   # general (3-pass) path
        scratch = torch.empty(2 * n * h * ((w + 31) // 32), dtype=torch.int32, device=payload.device)
    fill = getattr(border, "value", border)
    _capi.call("be_p4_edges", ctypes.c_void_p(payload.data_ptr()), ctypes.c_void_p(out.data_ptr()),
               n, h, w, int(fill),
               None if scratch is None else ctypes.c_void_p(scratch.data_ptr()), _stream())
    return out


def detect_pbm(data: bytes, border: BorderPolicy = BorderPolicy.WHITE_OUTSIDE,
               raw: bool = True) -> bytes:
    """A PBM file's edge image as a PBM file (CLI `detect`'s data path,
    SPEC.md:388-396): P4 in -> one fused kernel -> P4 out."""
    magic, w, h, off = parse_header(data)
    if magic == "P4" and raw:
        rb = (w + 7) // 8
        out = detect_p4(_payload_tensor(data, off, rb * h), 1, h, w, border)
        return f"P4\n{w} {h}\n".encode() + out.cpu().numpy().tobytes()
    from .edge import detect_edges_mask

    return write_pbm(detect_edges_mask(read_pbm(data), border), raw)


def read_pgm(data: bytes):
    """`imageio.read_pgm`: P2 / P5 with maxval <= 255 -> the
    samples verbatim as a uint8 array [H, W] (the GrayImage the binarize
    functions take); maxval > 255 and short payloads raise ValueError with the
    byte offset.  Host-side parsing: PGM is the photograph entry point, not
    part of the edge path."""
    if len(data) < 2 or data[:1] != b"P" or data[1:2] not in (b"2", b"5"):
        raise ValueError("not a PGM file (magic P2/P5 expected) at offset 0")
    magic = data[1:2]
    pos, vals = 2, []
    while len(vals) < 3:
        while pos < len(data) and (data[pos:pos + 1].isspace() or data[pos:pos + 1] == b"#"):
            if data[pos:pos + 1] == b"#":
                while pos < len(data) and data[pos] not in b"\r\n":
                    pos += 1
            else:
                pos += 1
        start = pos
        while pos < len(data) and data[pos:pos + 1].isdigit():
            pos += 1
        if start == pos:
            raise ValueError(f"malformed PGM header at offset {start}")
        vals.append(int(data[start:pos]))
    w, h, maxval = vals
    if w < 1 or h < 1:
        raise ValueError("image dimensions must be at least 1x1")
    if maxval > 255:
        raise ValueError(f"maxval {maxval} > 255 not supported (offset {pos})")
    pos += 1
    if magic == b"5":
        need = w * h
        if len(data) - pos < need:
            raise ValueError(f"short PGM payload: need {need} bytes at offset {pos}, "
                             f"have {len(data) - pos}")
        return np.frombuffer(data[pos:pos + need], np.uint8).reshape(h, w).copy()
    toks = data[pos:].split()
    if len(toks) < w * h:
        raise ValueError(f"short PGM payload: need {w * h} samples after offset {pos}")
    return np.array([int(t) for t in toks[: w * h]], np.uint8).reshape(h, w)

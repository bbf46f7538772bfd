"""`bitedge.binarize` on the device (the reference ships no
binarize module).  The fixed-threshold rule is the piece SURVEY 8(f) F2 fuses
into the edge kernels; Otsu picks the threshold from a device
histogram.

    threshold(gray, t) -> BitImage      pixel -> White iff sample >= t
    threshold_edges(gray, t, border)    (binarised, edges); batches: cuda.threshold_edges_u8
    otsu_threshold(gray) -> int         between-class-variance maximiser, ties -> smaller t
"""

from __future__ import annotations

import numpy as np

from .bitimage import BitImage, BorderPolicy, _device, _is_tensor, _torch


def _gray_tensor(gray):
    torch = _torch()
    if _is_tensor(gray) and gray.is_cuda:
        g = gray
    else:
        a = np.asarray(gray)
        if a.ndim != 2:
            raise ValueError(f"expected a 2-d array, got shape {a.shape}")
        if a.dtype != np.uint8:
            raise ValueError(f"gray samples must be uint8 (0..255), got {a.dtype}")
        g = torch.from_numpy(np.ascontiguousarray(a)).to(_device())
    if g.dim() != 2 or g.dtype != torch.uint8:
        raise ValueError("gray must be a 2-d uint8 image")
    h, w = g.shape
    if w < 1 or h < 1:
        raise ValueError(f"image dimensions must be at least 1x1, got {w}x{h}")
    return g.contiguous()


def threshold(gray, t: int) -> BitImage:
    """Pixel -> White iff sample >= t."""
    from . import cuda

    g = _gray_tensor(gray)
    h, w = g.shape
    return BitImage._wrap(int(w), int(h), cuda.threshold_u8(g, t, word_bits=64))


def threshold_edges(gray, t: int, border: BorderPolicy = BorderPolicy.WHITE_OUTSIDE):
    """(binarised image, its edge image) as BitImages.  The single-pass fused
    kernel for batches is `cuda.threshold_edges_u8`; this convenience form
    composes threshold() and detect_edges_mask() on the device words."""
    from .edge import detect_edges_mask

    binary = threshold(gray, t)
    return binary, detect_edges_mask(binary, border)


def otsu_threshold(gray: np.ndarray) -> int:
    """Between-class-variance maximiser over the 256-bin histogram; ties go to the
    smaller threshold.  Histogram on the device."""
    torch = _torch()
    g = _gray_tensor(gray).reshape(-1)
    hist = torch.bincount(g.to(torch.int64), minlength=256).to(torch.float64)
    total = hist.sum()
    t = torch.arange(256, dtype=torch.float64, device=g.device)
    w0 = torch.cumsum(hist, 0) - hist             # samples < t  (black class for threshold t)
    m0 = torch.cumsum(hist * t, 0) - hist * t
    w1 = total - w0
    m1 = (hist * t).sum() - m0
    valid = (w0 > 0) & (w1 > 0)
    var = torch.where(valid, w0 * w1 * (m0 / w0.clamp(min=1) - m1 / w1.clamp(min=1)) ** 2,
                      torch.zeros_like(w0))
    best = var.max()
    if best <= 0:
        return 0
    return int(torch.nonzero(var >= best * (1 - 1e-12))[0].item())

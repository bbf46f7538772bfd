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
    smaller threshold.  The histogram is counted on the
    device; the 256 candidates are then compared EXACTLY on the host in integer
    arithmetic: for threshold t (black class = samples < t) with class counts
    w0, w1 and sample sums s0, s1, the variance w0*w1*(s0/w0 - s1/w1)^2 equals
    (s0*w1 - s1*w0)^2 / (w0*w1), and two candidates compare by cross-
    multiplication -- no floating-point near-ties."""
    torch = _torch()
    g = _gray_tensor(gray).reshape(-1)
    hist = [int(v) for v in torch.bincount(g.to(torch.int64), minlength=256).tolist()]
    total = sum(hist)
    total_sum = sum(t * c for t, c in enumerate(hist))
    best_t, best_num, best_den = 0, 0, 1            # variance 0 at t = 0 (w0 = 0)
    w0 = s0 = 0
    for t in range(256):
        # class 0 = samples < t
        if t > 0:
            w0 += hist[t - 1]
            s0 += (t - 1) * hist[t - 1]
        w1, s1 = total - w0, total_sum - s0
        if w0 == 0 or w1 == 0:
            continue
        num = (s0 * w1 - s1 * w0) ** 2
        den = w0 * w1
        if num * best_den > best_num * den:          # strictly larger: ties keep the smaller t
            best_t, best_num, best_den = t, num, den
    return best_t

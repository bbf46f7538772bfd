"""Seeded synthetic inputs for the five BASELINE configs.

The reference's `bench.generate` is absent; these generators
stand in for the paper's glyph/page images, with the shapes, sizes and value
distributions BASELINE.json names.  Every shape is rasterised with integer
arithmetic only, so a generator gives the same bits on the CPU and on a GPU.
Polarity follows the reference: 1 = white background, 0 = black figure.

    C1  1 x 256 x 256 uint8        12 disks + 8 rectangles            seed 1
    C2  4096 x 64 x 64 uint8       1-4 thick polylines per glyph      rng([2, i])
    C3  8192 x 8192 packed uint32  i.i.d. Bernoulli(0.5) bits         seed 3
    C4  65536 x 65536 packed u32   200k disks, r in 4..64             seed 4
    C5  1024 x 2048 x 2048 uint8   text-line rectangles + 0.5% toggles rng([5, i])

C1-C3 are numpy (host).  C2, C4 and C5 rasterise with torch so they can be
built directly in HBM on the GPU box; the rasterisation is never timed.
"""

from __future__ import annotations

import numpy as np

try:  # torch is only needed for the device-side rasterisers
    import torch
except Exception:  # pragma: no cover
    torch = None

# --------------------------------------------------------------------------- C1

C1_SHAPE = (256, 256)


def c1_image(seed: int = 1, size: int = 256, n_disks: int = 12, n_rects: int = 8) -> np.ndarray:
    """256x256 uint8 {0,1}: white canvas, 12 black disks (r 8..40) and 8 black
    rectangles (w, h 4..64), clipped at the raster edge."""
    rng = np.random.default_rng(seed)
    img = np.ones((size, size), dtype=np.uint8)
    yy, xx = np.mgrid[0:size, 0:size]
    for _ in range(n_disks):
        cx, cy = (int(v) for v in rng.integers(0, size, 2))
        r = int(rng.integers(8, 41))
        img[(xx - cx) ** 2 + (yy - cy) ** 2 <= r * r] = 0
    for _ in range(n_rects):
        x0, y0 = (int(v) for v in rng.integers(0, size, 2))
        w, h = (int(v) for v in rng.integers(4, 65, 2))
        img[y0:y0 + h, x0:x0 + w] = 0
    return img


# --------------------------------------------------------------------------- C2

C2_BOX = (12, 52)          # vertex box [lo, hi) tuned for ~15% black (asserted in tests)


def c2_segments(n_images: int, start: int = 0, size: int = 64):
    """Per image i: rng = default_rng([2, i]); k in 1..4 polylines, each with
    3..6 vertices uniform in C2_BOX^2 and thickness t in 3..7.  Returns padded
    int64 arrays ax, ay, bx, by, t4 (= t^2) and a validity mask, shape [N, S]."""
    segs = []
    lo, hi = C2_BOX
    for i in range(start, start + n_images):
        rng = np.random.default_rng([2, i])
        k = int(rng.integers(1, 5))
        s = []
        for _ in range(k):
            n = int(rng.integers(3, 7))
            t = int(rng.integers(3, 8))
            v = rng.integers(lo, hi, (n, 2))
            for j in range(n - 1):
                s.append((v[j, 0], v[j, 1], v[j + 1, 0], v[j + 1, 1], t * t))
        segs.append(s)
    m = max(len(s) for s in segs)
    arr = np.zeros((n_images, m, 5), dtype=np.int64)
    valid = np.zeros((n_images, m), dtype=bool)
    for i, s in enumerate(segs):
        arr[i, : len(s)] = s
        valid[i, : len(s)] = True
    return arr, valid


def _segment_cover(px, py, ax, ay, bx, by, t2):
    """4*dist(P, segment AB)^2 <= t^2, exactly, in int64 (works for numpy and torch)."""
    abx, aby = bx - ax, by - ay
    apx, apy = px - ax, py - ay
    den = abx * abx + aby * aby
    num = apx * abx + apy * aby
    d_a = apx * apx + apy * apy
    bpx, bpy = px - bx, py - by
    d_b = bpx * bpx + bpy * bpy
    cross = apx * aby - apy * abx
    inside = (num > 0) & (num < den)
    # interior: d^2 = cross^2 / den  ->  4 cross^2 <= t^2 den
    cov_in = 4 * cross * cross <= t2 * den
    cov_a = 4 * d_a <= t2
    cov_b = 4 * d_b <= t2
    return (inside & cov_in) | cov_a | cov_b


def c2_images(n_images: int = 4096, start: int = 0, size: int = 64, device="cpu",
              chunk: int = 256) -> "torch.Tensor":
    """uint8 [N, 64, 64] glyph batch as a torch tensor on `device` (exact
    integer rasterisation, so CPU and GPU give identical bits)."""
    arr, valid = c2_segments(n_images, start, size)
    A = torch.as_tensor(arr, device=device)
    V = torch.as_tensor(valid, device=device)
    ys, xs = torch.meshgrid(torch.arange(size, device=device), torch.arange(size, device=device),
                            indexing="ij")
    out = torch.empty((n_images, size, size), dtype=torch.uint8, device=device)
    px = xs.reshape(1, 1, -1)
    py = ys.reshape(1, 1, -1)
    for c0 in range(0, n_images, chunk):
        a = A[c0:c0 + chunk]
        v = V[c0:c0 + chunk]
        ax, ay, bx, by, t2 = (a[..., j:j + 1] for j in range(5))
        cov = _segment_cover(px, py, ax, ay, bx, by, t2) & v[..., None]
        out[c0:c0 + chunk] = (~cov.any(1)).reshape(-1, size, size).to(torch.uint8)
    return out


# --------------------------------------------------------------------------- C3

C3_SHAPE = (8192, 8192)


def c3_words(seed: int = 3, h: int = 8192, w: int = 8192) -> np.ndarray:
    """Pre-packed uint32 [h, w/32], every bit i.i.d. Bernoulli(0.5)."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, 2 ** 32, (h, w // 32), dtype=np.uint32)


# --------------------------------------------------------------------------- C4

C4_SIZE = 65536
C4_DISKS = 200_000


def c4_disks(seed: int = 4, size: int = C4_SIZE, n: int = C4_DISKS, rmin: int = 4, rmax: int = 64):
    """The shared disk list every rank builds: int64 [n, 3] = (cx, cy, r)."""
    rng = np.random.default_rng(seed)
    cx = rng.integers(0, size, n)
    cy = rng.integers(0, size, n)
    r = rng.integers(rmin, rmax + 1, n)
    return np.stack([cx, cy, r], axis=1).astype(np.int64)


def _isqrt_t(v):
    """floor(sqrt(v)) for non-negative int64 torch tensors, exactly."""
    s = torch.sqrt(v.to(torch.float64)).floor().to(torch.int64)
    s = torch.where(s * s > v, s - 1, s)
    s = torch.where((s + 1) * (s + 1) <= v, s + 1, s)
    return s


def pack_bits_rows_t(white: "torch.Tensor") -> "torch.Tensor":
    """bool/uint8 [R, W] (W % 32 == 0, nonzero = white) -> int32 [R, W/32] MSB-first."""
    r, w = white.shape
    b = (white != 0).reshape(r, w // 32, 32).to(torch.int64)
    weights = (1 << torch.arange(31, -1, -1, device=white.device, dtype=torch.int64))
    v = (b * weights).sum(-1)
    return (v - ((v >> 31) << 32)).to(torch.int32)  # wrap into int32 two's complement


def c4_slab(row_lo: int, row_hi: int, disks: np.ndarray, size: int = C4_SIZE, device="cpu",
            chunk_rows: int = 2048) -> "torch.Tensor":
    """Rows [row_lo, row_hi) of the C4 raster as packed int32 words [rows, size/32].
    Only disks touching the slab are rasterised (per-row spans -> coverage)."""
    d = torch.as_tensor(disks, device=device)
    out = torch.empty((row_hi - row_lo, size // 32), dtype=torch.int32, device=device)
    for y0 in range(row_lo, row_hi, chunk_rows):
        y1 = min(row_hi, y0 + chunk_rows)
        cx, cy, r = d[:, 0], d[:, 1], d[:, 2]
        sel = (cy + r >= y0) & (cy - r < y1)
        cx, cy, r = cx[sel], cy[sel], r[sel]
        # one span per (disk, row) with |dy| <= r inside [y0, y1)
        dy = torch.arange(-64, 65, device=device)
        rows = cy[:, None] + dy[None, :]
        ok = (dy[None, :].abs() <= r[:, None]) & (rows >= y0) & (rows < y1)
        half = _isqrt_t((r[:, None] ** 2 - dy[None, :] ** 2).clamp(min=0))
        x0 = (cx[:, None] - half).clamp(min=0)
        x1 = (cx[:, None] + half).clamp(max=size - 1)
        rows, x0, x1 = rows[ok] - y0, x0[ok], x1[ok]
        cov = torch.zeros((y1 - y0) * (size + 1), dtype=torch.int32, device=device)
        ones = torch.ones_like(rows, dtype=torch.int32)
        cov.index_put_((rows * (size + 1) + x0,), ones, accumulate=True)
        cov.index_put_((rows * (size + 1) + x1 + 1,), -ones, accumulate=True)
        cov = cov.view(y1 - y0, size + 1)[:, :size].cumsum(1, dtype=torch.int32)
        out[y0 - row_lo:y1 - row_lo] = pack_bits_rows_t(cov == 0)
        del cov
    return out


# --------------------------------------------------------------------------- C5

C5_SIZE = 2048
C5_LINE_PITCH = 48
C5_BASE0 = 40              # first baseline row; line i has baseline 40 + 48 i
C5_MARGIN = (16, 48)       # left margin drawn from [16, 48)
C5_GAP = (10, 100)          # gap after each rectangle drawn from [10, 60); tuned for ~10% black
C5_TOGGLE = 0.005


def c5_heights(page: int, size: int = C5_SIZE) -> np.ndarray:
    """Column ink heights of one page: uint8 [n_lines, size]; rectangle j of a
    line spans w in 4..30 columns with height h in 10..32, bottom-aligned to
    the baseline, followed by a gap."""
    rng = np.random.default_rng([5, page])
    n_lines = (size - C5_BASE0 + C5_LINE_PITCH - 1) // C5_LINE_PITCH
    H = np.zeros((n_lines, size), dtype=np.uint8)
    cap = size // 14 + 8
    for i in range(n_lines):
        x = int(rng.integers(*C5_MARGIN))
        w = rng.integers(4, 31, cap)
        h = rng.integers(10, 33, cap)
        g = rng.integers(*C5_GAP, cap)
        starts = x + np.concatenate([[0], np.cumsum(w + g)[:-1]])
        for s, ww, hh in zip(starts, w, h):
            if s >= size:
                break
            H[i, s:min(size, s + ww)] = hh
    return H


def c5_toggles(page: int, size: int = C5_SIZE) -> np.ndarray:
    """Sorted unique flat pixel indices whose colour is flipped (0.5% salt)."""
    rng = np.random.default_rng([5, page, 1])
    k = int(rng.binomial(size * size, C5_TOGGLE))
    return np.unique(rng.integers(0, size * size, k))


def c5_pages(n_pages: int = 1024, start: int = 0, size: int = C5_SIZE, device="cpu", out=None):
    """uint8 [n_pages, size, size] page batch (values {0,1})."""
    if out is None:
        out = torch.empty((n_pages, size, size), dtype=torch.uint8, device=device)
    y = torch.arange(size, device=device)
    line = (y // C5_LINE_PITCH).clamp(max=(size - C5_BASE0 - 1) // C5_LINE_PITCH)
    off = C5_BASE0 + C5_LINE_PITCH * line - y                 # baseline - y
    for p in range(n_pages):
        H = torch.as_tensor(c5_heights(start + p, size), device=device)
        Hy = H[line].to(torch.int64)                          # [size(y), size(x)]
        black = (off[:, None] >= 0) & (off[:, None] < Hy)
        img = (~black).to(torch.uint8).view(-1)
        t = torch.as_tensor(c5_toggles(start + p, size), device=device)
        img[t] ^= 1
        out[p] = img.view(size, size)
    return out

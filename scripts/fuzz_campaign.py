"""Time-bounded random parity campaign on the GPU (default dispatch, no knobs):
uint8 batches, packed u32 / u64 rasters and P4 payloads of random shapes --
many of them large enough to reach the flat kernels (K1f, K1p), the TMA ring's
run-time strips and the UNAL variants -- and thresholded grayscale batches,
against the C scanner.
Usage: fuzz_campaign.py [seconds] [seed]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import cscan  # noqa: E402
from oracle import port as P  # noqa: E402
from paper_1401_5245_b200 import cuda as cu  # noqa: E402
from paper_1401_5245_b200 import pbm  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rng = np.random.default_rng(seed)
dev = torch.device("cuda:0")
t0, n_cases, px = time.time(), 0, 0


def shape():
    kind = rng.integers(0, 6)
    if kind == 0:                                    # small
        return int(rng.integers(1, 5)), int(rng.integers(1, 70)), int(rng.integers(1, 400))
    if kind == 1:                                    # batch of medium images
        return int(rng.integers(2, 40)), int(rng.integers(50, 700)), int(rng.integers(100, 2100))
    if kind == 2:                                    # one tall raster, wide rows
        return 1, int(rng.integers(2000, 9000)), int(rng.integers(1000, 9000))
    if kind == 3:                                    # rows near the segment / vector boundaries
        w = int(rng.choice([1024, 1040, 1280, 2048, 4096, 6144, 8000, 8192])) + int(rng.integers(-33, 34))
        return int(rng.integers(1, 4)), int(rng.integers(500, 7000)), max(1, w)
    if kind == 4:                                    # few rows, very wide
        return 1, int(rng.integers(1, 12)), int(rng.integers(5000, 200000))
    return int(rng.integers(1, 3)), int(rng.integers(3000, 16000)), int(rng.integers(200, 2600))


while time.time() - t0 < budget:
    n, h, w = shape()
    if n * h * w > 120_000_000:
        continue
    fill = int(rng.integers(0, 2))
    a = (rng.random((n, h, w)) < rng.choice([0.2, 0.5, 0.8, 0.97])).astype(np.uint8)
    exp = cscan.scan_u8(a, fill)
    tag = (n, h, w, fill)
    # uint8 pixels (contiguous, and a strided view at a byte offset)
    x = torch.from_numpy(a).to(dev)
    got = cu.pack_edges_u8(x, fill).cpu().numpy().view(np.uint32)
    assert (got == exp).all(), ("u8", tag)
    if n * h * w < 40_000_000:
        pad, off = int(rng.integers(0, 37)), int(rng.integers(0, 17))
        buf = torch.zeros(n * h * (w + pad) + off + 64, dtype=torch.uint8, device=dev)
        view = buf[off:off + n * h * (w + pad)].view(n, h, w + pad)[..., :w]
        view.copy_(x)
        got = cu.pack_edges_u8(view, fill).cpu().numpy().view(np.uint32)
        assert (got == exp).all(), ("u8 strided", tag, pad, off)
    # thresholded pack (F2): white iff sample >= t
    if n * h * w < 60_000_000:
        t = int(rng.choice([0, 1, 2, 77, 128, 200, 255]))
        g = rng.integers(0, 256, (n, h, w)).astype(np.uint8)
        got = cu.threshold_edges_u8(torch.from_numpy(g).to(dev), t, fill).cpu().numpy().view(np.uint32)
        assert (got == cscan.scan_u8((g >= t).astype(np.uint8), fill)).all(), ("thr", tag, t)
    # packed u32 and u64 words
    pk = torch.from_numpy(P.pack_u32(a).view(np.int32)).to(dev)
    got = cu.edges_packed(pk, w, fill).cpu().numpy().view(np.uint32)
    assert (got == exp).all(), ("u32", tag)
    es = cu.edges_packed(pk, w, fill, edgeset=True).cpu().numpy().view(np.uint32)
    assert (es == cscan.scan_u8(a, fill, edgeset=True)).all(), ("u32 eset", tag)
    w64 = cu.pack_u8(x, word_bits=64)
    got = P.u64_to_u32_rows(cu.edges_packed(w64, w, fill).cpu().numpy().view(np.uint64).reshape(n * h, -1))
    assert (got[:, : exp.shape[-1]].reshape(exp.shape) == exp).all(), ("u64", tag)
    # P4 payload with garbage padding bits
    rb = (w + 7) // 8
    bits = rng.integers(0, 2, (n, h, rb * 8)).astype(np.uint8)
    bits[..., :w] = a
    payload = torch.from_numpy(np.packbits(1 - bits, axis=-1).reshape(-1).copy()).to(dev)
    out = pbm.detect_p4(payload, n, h, w, fill).cpu().numpy().reshape(n, h, rb)
    assert ((1 - np.unpackbits(out, axis=-1)[..., :w]) == P.unpack_u32(exp, w)).all(), ("p4", tag)
    if w % 8:
        assert not (out[..., -1] & ((1 << (8 - w % 8)) - 1)).any(), ("p4 pad", tag)
    n_cases += 1
    px += n * h * w
print(f"fuzz campaign ok: {n_cases} shapes, {px / 1e9:.2f} Gpx, seed {seed}, {time.time() - t0:.0f} s")

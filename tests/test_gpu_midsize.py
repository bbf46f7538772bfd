"""Mid-size rasters through the DEFAULT dispatch (no knobs): the shapes that pick
K2t2's run-time strip heights (short strips below one wave of resident warps,
wave-fitted strips above), K1f's 31-chunk warps on ragged packed rows, and
K1p / K1f-P4 on P4 payloads with many rows -- each against the C scanner
(oracle/scan.c, per-pixel Edge(p): reference SPEC.md:174-191) on the whole output."""

import numpy as np
import pytest

from oracle import cscan
from oracle import port as P

pytestmark = pytest.mark.gpu


def _pages(h, w, seed):
    rng = np.random.default_rng(seed)
    a = (rng.random((h, w)) < 0.8).astype(np.uint8)
    a[:: max(1, h // 7)] ^= 1                      # whole rows flipped: row-structure mistakes show
    a[:, :: max(1, w // 5)] ^= 1
    return a


@pytest.mark.parametrize("h,w", [(6016, 4096),      # 12 032 row segments: 5-row strips
                                 (2900, 10240),     # 5 segments per row, 5-row strips
                                 (5200, 8192),      # 20 800 row segments: 6-row strips
                                 (8192, 8192),      # 1.15 waves of 8-row strips -> 10-row strips
                                 (7000, 6148),      # ragged rows through the UNAL ring
                                 (12960, 1920),     # 12 frames of 1920 x 1080: one 94 %-full segment
                                 (12000, 1600),     # 78 %-full segments
                                 (12288, 1408),     # the narrowest 32-byte rows the ring takes
                                 (12960, 1900),     # ragged 1900-px rows: UNAL ring under 2048 px
                                 (16000, 1290),     # 63 %-full ragged segments
                                 (14400, 1200),     # 16-byte rows under 1280 px: the ring from 1040 px
                                 (13000, 1100)])    # ragged rows under 1280 px
def test_u8_midsize_default_dispatch(cuda_dev, h, w):
    import torch

    from paper_1401_5245_b200 import cuda as cu

    a = _pages(h, w, h + w)
    x = torch.from_numpy(a).to(cuda_dev)
    for fill in (1, 0):
        got = cu.pack_edges_u8(x, fill).cpu().numpy().view(np.uint32)
        exp = cscan.scan_u8(a, fill)
        assert (got == exp).all(), (h, w, fill, np.argwhere(got != exp)[:4])
    # the drop-in layout (uint64 words, edges + packed input in one launch)
    e64, p64 = cu.pack_and_edges(x, 1, word_bits=64)
    ref = P.from_array(a)
    assert (p64.cpu().numpy().view(np.uint64) == ref.words).all()
    got32 = P.u64_to_u32_rows(e64.cpu().numpy().view(np.uint64))[:, : -(-w // 32)]
    assert (got32 == cscan.scan_u8(a, 1)).all()


@pytest.mark.parametrize("h,w,t", [(8192, 4096, 128), (13000, 1920, 77), (6200, 8192, 200)])
def test_threshold_midsize_default_dispatch(cuda_dev, h, w, t):
    """F2 (threshold fused into the pack, reference SPEC.md:237-245) on rasters that
    take K2t2's 12-row run-time strips: white iff sample >= t."""
    import torch

    from paper_1401_5245_b200 import cuda as cu

    rng = np.random.default_rng(h + w + t)
    g = rng.integers(0, 256, (h, w)).astype(np.uint8)
    g[:: max(1, h // 9)] = 0
    g[:, :: max(1, w // 7)] = 255
    x = torch.from_numpy(g).to(cuda_dev)
    binary = (g >= t).astype(np.uint8)
    for fill in (1, 0):
        got = cu.threshold_edges_u8(x, t, fill).cpu().numpy().view(np.uint32)
        exp = cscan.scan_u8(binary, fill)
        assert (got == exp).all(), (h, w, t, fill, np.argwhere(got != exp)[:4])


def test_u8_rolling_strips_rows_straddling_warps(cuda_dev):
    """K2r (32-row rolling strips; needs >= 303 104 threads) on 640-px rows: 20 words
    per row, so warps straddle rows and lanes 0 / 31 fetch their neighbour bytes."""
    import torch

    from paper_1401_5245_b200 import cuda as cu

    rng = np.random.default_rng(11)
    a = (rng.random((1100, 480, 640)) < 0.7).astype(np.uint8)
    got = cu.pack_edges_u8(torch.from_numpy(a).to(cuda_dev), 1).cpu().numpy().view(np.uint32)
    exp = cscan.scan_u8(a, 1)
    assert (got == exp).all(), np.argwhere(got != exp)[:4]


@pytest.mark.parametrize("h,w,bits", [(8192, 8000, 32), (8192, 8000, 64), (3001, 10016, 32),
                                      (5000, 4100, 64), (2, 8000, 32), (3, 1056, 64)])
def test_packed_ragged_flat(cuda_dev, h, w, bits):
    """K1f (contiguous packed rows that are not vector multiples), whole rasters
    with many row ends per warp and with few rows."""
    import torch

    from paper_1401_5245_b200 import cuda as cu

    a = _pages(h, w, 3 * h + w)
    if bits == 32:
        words = torch.from_numpy(P.pack_u32(a).view(np.int32)).to(cuda_dev)
    else:
        words = torch.from_numpy(P.from_array(a).words.view(np.int64).copy()).to(cuda_dev)
    for fill in (1, 0):
        exp = cscan.scan_u8(a, fill)
        got = cu.edges_packed(words, w, fill).cpu().numpy()
        if bits == 64:
            got = P.u64_to_u32_rows(got.view(np.uint64))[:, : -(-w // 32)]
        else:
            got = got.view(np.uint32)
        assert (got == exp).all(), (h, w, bits, fill, np.argwhere(got != exp)[:4])


@pytest.mark.parametrize("n,h,w", [(1, 3000, 24601),    # 3 076-byte rows: K1p, 32-byte chunks
                                   (2, 2500, 12002),    # 1 501-byte rows: K1p, 16-byte chunks
                                   (3, 700, 4001),      # small payload: inline edge chunks
                                   (1, 4000, 8000),     # 1 000-byte rows: K1f P4
                                   (2, 3000, 7993)])    # 1 000-byte rows with padding bits
def test_p4_midsize(cuda_dev, n, h, w, monkeypatch):
    import torch

    from paper_1401_5245_b200 import pbm

    rng = np.random.default_rng(n * h + w)
    a = np.stack([_pages(h, w, i + w) for i in range(n)])
    rb = (w + 7) // 8
    bits = rng.integers(0, 2, (n, h, rb * 8)).astype(np.uint8)     # garbage padding bits
    bits[..., :w] = a
    payload = torch.from_numpy(np.packbits(1 - bits, axis=-1).reshape(-1).copy()).to(cuda_dev)
    for fill in (1, 0):
        out = pbm.detect_p4(payload, n, h, w, fill).cpu().numpy().reshape(n, h, rb)
        got = 1 - np.unpackbits(out, axis=-1)[..., :w]
        exp = P.unpack_u32(cscan.scan_u8(a, fill), w)
        assert (got == exp).all(), (n, h, w, fill, np.argwhere(got != exp)[:4])
        if w % 8:
            assert not (out[..., -1] & ((1 << (8 - w % 8)) - 1)).any()

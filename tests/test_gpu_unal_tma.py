"""K2t2 UNAL (edge_reg.cuh): uint8 rows >= 2048 px at any byte offset -- rows
whose length is not a 16-byte multiple, views at odd base addresses, strided
rows -- staged by granule-aligned TMA copies and realigned after the pack.
Bit-exact against the per-pixel C oracle for every output the path writes
(edges, EdgeSet, packed words in u32 and the drop-in's u64 layout),
thresholds, both border policies; forced onto small shapes and reached by
dispatch on a large one; and identical to K2 UNAL (BITEDGE_NO_TMA_UNAL)."""

import numpy as np
import pytest

from oracle import cscan
from oracle import port as P

pytestmark = pytest.mark.gpu


def _view(torch, dev, a, base_off, pad):
    """`a` [n,h,w] uint8 copied into a device buffer at byte offset `base_off`
    with `pad` garbage bytes after every row; returns the strided view."""
    n, h, w = a.shape
    rb = w + pad
    rng = np.random.default_rng(base_off * 31 + pad)
    buf = rng.integers(0, 256, base_off + n * h * rb + 64, dtype=np.uint8)
    body = buf[base_off: base_off + n * h * rb].reshape(n, h, rb)
    body[:, :, :w] = a
    t = torch.from_numpy(buf).to(dev)
    return t[base_off: base_off + n * h * rb].view(n, h, rb)[:, :, :w]


@pytest.mark.parametrize("w", [2049, 2050, 2063, 4100, 6001, 8191])
@pytest.mark.parametrize("base_off,pad", [(0, 0), (1, 0), (7, 3), (13, 0), (4, 12)])
@pytest.mark.parametrize("rsl", [None, "5"])
def test_unal_tma_forced(cuda_dev, monkeypatch, w, base_off, pad, rsl):
    import torch

    from paper_1401_5245_b200 import cuda as cu

    monkeypatch.setenv("BITEDGE_FORCE_TMA", "1")
    if rsl:
        monkeypatch.setenv("BITEDGE_TMA2_RSL", rsl)   # run-time strip height
    rng = np.random.default_rng(w + 17 * base_off + pad)
    n, h = 2, 19
    a = (rng.random((n, h, w)) < 0.55).astype(np.uint8) * rng.integers(1, 256, (n, h, w),
                                                                         dtype=np.uint8)
    x = _view(torch, cuda_dev, a, base_off, pad)
    if (w + pad) % 16 == 0 and base_off % 16 == 0:
        pytest.skip("aligned rows take the aligned kernel")
    for fill in (1, 0):
        exp = cscan.scan_u8(a, fill)
        got = cu.pack_edges_u8(x, fill)
        assert (got.cpu().numpy().view(np.uint32) == exp).all(), ("edges", w, base_off, pad, fill)
        es = cu.edges_general(x, border=fill, edges=False, edgeset=True)["edgeset"]
        assert (es.cpu().numpy().view(np.uint32) == cscan.scan_u8(a, fill, edgeset=True)).all()
        pk = torch.empty_like(got)
        cu.pack_edges_u8(x, fill, packed_out=pk)
        assert (pk.cpu().numpy().view(np.uint32) == P.pack_u32((a != 0).astype(np.uint8))).all()
    # the drop-in layout: uint64 words (store column c ^ 1), edges + packed
    e64, p64 = cu.pack_and_edges(x[0], 1, word_bits=64)
    ref = P.from_array(a[0])
    assert (p64.cpu().numpy().view(np.uint64) == ref.words).all()
    assert (e64.cpu().numpy().view(np.uint64) == P.detect_edges_mask(ref, 1).words).all()
    # thresholds (the pack's general >= t compare)
    for t in (2, 128, 255):
        got = cu.threshold_edges_u8(x, t, 1)
        assert (got.cpu().numpy().view(np.uint32) == cscan.scan_u8((a >= t).astype(np.uint8), 1)).all()


def test_unal_tma_dispatch_large(cuda_dev, monkeypatch):
    """Large enough to be chosen without forcing; equal to K2 UNAL."""
    import torch

    from paper_1401_5245_b200 import cuda as cu

    rng = np.random.default_rng(3)
    a = (rng.random((1, 6144, 16100)) < 0.5).astype(np.uint8)
    x = torch.from_numpy(a).to(cuda_dev)
    got = cu.pack_edges_u8(x, 1)
    assert (got.cpu().numpy().view(np.uint32) == cscan.scan_u8(a, 1)).all()
    monkeypatch.setenv("BITEDGE_NO_TMA_UNAL", "1")
    assert torch.equal(cu.pack_edges_u8(x, 1), got)

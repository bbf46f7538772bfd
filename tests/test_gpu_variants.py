"""Every kernel variant the C ABI can dispatch to must agree bit-for-bit with
the per-pixel oracle.  One process exercises them all through the library's
selection knobs:

    default        register-direct kernels (K1 8/4-word items, K2 one-shot
                   strips, K2r rolling strips, K2w warp-per-image)
    tile           one-shot shared-memory tile kernel (the general fallback)
    stream         persistent TMA (cp.async.bulk + mbarrier) pipelined kernel
    cw4, rs8, no_roll, no_warpimg, no_pdl, k2p, no_flat   individual knobs
(the knobs are read once per process; tests/conftest.py re-reads them after
every monkeypatch.setenv)
"""

import numpy as np
import pytest

from oracle import cscan
from oracle import port as P

pytestmark = pytest.mark.gpu

VARIANTS = {
    "default": {},
    "tile": {"BITEDGE_KERNEL": "tile"},
    "stream": {"BITEDGE_KERNEL": "stream"},
    "cw4": {"BITEDGE_CW4": "1"},
    "rs8": {"BITEDGE_RS": "8"},
    "no_roll": {"BITEDGE_NO_ROLL": "1"},
    "no_warpimg": {"BITEDGE_NO_WARPIMG": "1"},
    "no_pdl": {"BITEDGE_PDL": "0"},
    "tma_warp": {"BITEDGE_FORCE_TMA": "1"},
    "tma_warp1k": {"BITEDGE_FORCE_TMA": "1", "BITEDGE_TMA1": "1"},
    "no_tma": {"BITEDGE_NO_TMA": "1"},
    "warpimg_g4": {"BITEDGE_WARPIMG_G4": "1"},
    "pdl_late": {"BITEDGE_PDL_LATE": "1"},
    "tma_warp_rsl32": {"BITEDGE_FORCE_TMA": "1", "BITEDGE_TMA2_RSL32": "1"},
    "tma_warp_rsl3": {"BITEDGE_FORCE_TMA": "1", "BITEDGE_TMA2_RSL": "3"},
    "tma_warp_rsl6": {"BITEDGE_FORCE_TMA": "1", "BITEDGE_TMA2_RSL": "6"},
    "tma_warp_rsl13": {"BITEDGE_FORCE_TMA": "1", "BITEDGE_TMA2_RSL": "13"},
    "k1_generic": {"BITEDGE_K1_GENERIC": "1"},
    "k1_prs2": {"BITEDGE_PRS": "2"},
    "k1_prs8": {"BITEDGE_PRS": "8"},
    "no_unal": {"BITEDGE_NO_UNAL": "1"},
    "unal_chunks": {"BITEDGE_UNAL_CHUNKS": "1"},
    "unal_bytes": {"BITEDGE_UNAL_BYTES": "1"},
    "u64_tma": {"BITEDGE_U64_TMA": "1"},
    "k2p": {"BITEDGE_K2P": "1"},
    "no_h16": {"BITEDGE_NO_H16": "1"},
    "ring": {"BITEDGE_RING": "1"},
    "no_flat": {"BITEDGE_NO_FLAT": "1"},
}

# (n, h, w): glyph batches, wide pages, ragged widths, single rows / columns
SHAPES = [(64, 64, 64), (8, 32, 32), (3, 40, 2048), (2, 70, 4160), (5, 33, 100), (1, 1, 1), (3, 50, 8000), (2, 9, 1000),
          (1, 300, 1), (1, 1, 700), (4, 16, 256), (2, 200, 8192), (1500, 32, 32),
          (600, 16, 64), (333, 64, 128), (2, 37, 4100), (1, 19, 2050), (3, 21, 6001)]


def _t(a, dev):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.fixture(params=list(VARIANTS))
def variant(request, monkeypatch, cuda_dev):
    for k, v in VARIANTS[request.param].items():
        monkeypatch.setenv(k, v)
    return request.param


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_u8_and_packed_paths(variant, shape, cuda_dev):
    from paper_1401_5245_b200 import cuda as cu

    n, h, w = shape
    rng = np.random.default_rng(hash(shape) % 2**32)
    a = (rng.random((n, h, w)) < 0.55).astype(np.uint8) * rng.integers(1, 256, (n, h, w)).astype(
        np.uint8)
    for fill in (1, 0):
        exp = cscan.scan_u8(a, fill)
        got = _u32(cu.pack_edges_u8(_t(a, cuda_dev), fill))
        assert (got == exp).all(), (variant, shape, fill, "u8")
        pk = P.pack_u32(a)
        got32 = _u32(cu.edges_packed(_t(pk.view(np.int32), cuda_dev), w, fill))
        assert (got32 == exp).all(), (variant, shape, fill, "u32")
    # EdgeSet output and the native uint64 layout
    es = _u32(cu.edges_packed(_t(pk.view(np.int32), cuda_dev), w, 1, edgeset=True))
    assert (es == cscan.scan_u8(a, 1, edgeset=True)).all()
    if w > 1:
        w64 = np.stack([P.from_array(x).words for x in a])
        o64 = cu.edges_packed(_t(w64.view(np.int64), cuda_dev), w, 1).cpu().numpy().view(np.uint64)
        exp64 = np.stack([P.detect_edges_mask(P.from_array(x), 1).words for x in a])
        assert (o64 == exp64).all(), (variant, shape, "u64")


def test_row_slabs_each_variant(variant, cuda_dev):
    import torch

    from paper_1401_5245_b200 import cuda as cu

    rng = np.random.default_rng(3)
    H, W = 97, 8192
    a = (rng.random((H, W)) < 0.5).astype(np.uint8)
    pk = torch.from_numpy(P.pack_u32(a).view(np.int32)).to(cuda_dev)
    whole = cu.edges_packed(pk, W, 1)
    cuts = [0, 13, 50, 51, 97]
    parts = []
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        slab = pk[lo:hi].clone()
        above = pk[lo - 1].clone() if lo > 0 else None
        below = pk[hi].clone() if hi < H else None
        parts.append(cu.edges_halo(slab, above, below, W, 1))
    assert torch.equal(torch.cat(parts), whole), variant


@pytest.mark.parametrize("t", [1, 100, 200])
def test_threshold_each_variant(variant, t, cuda_dev):
    """F2 (threshold fused into the pack) through every kernel variant."""
    from paper_1401_5245_b200 import cuda as cu

    rng = np.random.default_rng(t)
    for (n, h, w) in [(16, 64, 64), (2, 40, 2048), (3, 21, 333), (1, 70, 4096)]:
        g = rng.integers(0, 256, (n, h, w), dtype=np.uint8)
        exp = cscan.scan_u8((g >= t).astype(np.uint8), 1)
        assert (_u32(cu.threshold_edges_u8(_t(g, cuda_dev), t, 1)) == exp).all(), (variant, t, w)

"""K1f / K1s (edge_flat.cuh): packed rows whose length is not a multiple of the
vector width, viewed as one flat word array (K1f register-direct, the default;
K1s staged through a per-warp shared-memory ring, opt-in) -- bit-exact against
the per-pixel C
oracle (u32 rows) and the reference composition (the drop-in's uint64 words),
for every realignment phase, 32- and 16-byte buffer alignment, batches, both
border policies and both outputs; and identical to the K1 UNAL kernel it
replaces (BITEDGE_NO_FLAT)."""

import numpy as np
import pytest

from oracle import cscan
from oracle import port as P

pytestmark = pytest.mark.gpu


def _aligned_view(torch, n_words, dtype, dev, offset_words):
    """A contiguous 1-D view starting `offset_words` 32-bit words past a 256-B
    aligned allocation (0: 32-B aligned; 4: only 16-B aligned)."""
    buf = torch.empty(n_words + 64, dtype=torch.int32, device=dev)
    v = buf[offset_words:offset_words + n_words]
    return v if dtype == torch.int32 else v.view(torch.int64)


# widths whose u32 word count hits every phase of the 8- and 4-word grids
U32_WIDTHS = [8000, 7999, 8160, 4100, 520, 600, 1056, 513, 700, 640, 660, 16 * 32 * 3 + 5]


@pytest.fixture(params=["flat", "ring"])
def flat_kernel(request, monkeypatch):
    """K1f (default) or K1s (opt-in, BITEDGE_RING, where it applies)."""
    if request.param == "ring":
        monkeypatch.setenv("BITEDGE_RING", "1")
    return request.param


@pytest.mark.parametrize("w", U32_WIDTHS)
@pytest.mark.parametrize("offset", [0, 4], ids=["a32", "a16"])
def test_flat_u32(cuda_dev, w, offset, flat_kernel):
    import torch

    from paper_1401_5245_b200 import cuda as cu

    rng = np.random.default_rng(w * 7 + offset)
    wp = -(-w // 32)
    for n, h in ((1, 1), (1, 2), (1, 37), (3, 5), (2, 64), (4, 33), (1, 1000), (5, 200)):
        words = rng.integers(0, 2**32, (n, h, wp), dtype=np.uint32)
        src = _aligned_view(torch, n * h * wp, torch.int32, cuda_dev, offset).view(n, h, wp)
        src.copy_(torch.from_numpy(words.view(np.int32)))
        for fill in (1, 0):
            oe = _aligned_view(torch, n * h * wp, torch.int32, cuda_dev, offset).view(n, h, wp)
            os_ = _aligned_view(torch, n * h * wp, torch.int32, cuda_dev, offset).view(n, h, wp)
            cu.edges_packed(src, w, fill, out=oe)
            cu.edges_packed(src, w, fill, out=os_, edgeset=True)
            exp = cscan.scan_p32(words, w, fill)
            exps = cscan.scan_p32(words, w, fill, edgeset=True)
            assert (oe.cpu().numpy().view(np.uint32) == exp).all(), (w, n, h, fill)
            assert (os_.cpu().numpy().view(np.uint32) == exps).all(), (w, n, h, fill)


@pytest.mark.parametrize("w", [8000, 1100, 8100, 1300, 2600, 4100])
@pytest.mark.parametrize("offset", [0, 4], ids=["a32", "a16"])
def test_flat_u64_dropin_words(cuda_dev, w, offset, flat_kernel):
    import torch

    from paper_1401_5245_b200 import cuda as cu

    rng = np.random.default_rng(w + offset)
    wp64 = -(-w // 64)
    for h in (1, 3, 40, 1000):
        a = (rng.random((h, w)) < 0.5).astype(np.uint8)
        ref = P.from_array(a)
        src = _aligned_view(torch, h * wp64 * 2, torch.int64, cuda_dev, offset).view(h, wp64)
        src.copy_(torch.from_numpy(ref.words.view(np.int64)))
        for fill in (1, 0):
            out = _aligned_view(torch, h * wp64 * 2, torch.int64, cuda_dev, offset).view(h, wp64)
            cu.edges_packed(src, w, fill, out=out)
            got = out.cpu().numpy().view(np.uint64)
            assert (got == P.detect_edges_mask(ref, fill).words).all(), (w, h, fill)
            es = cu.edges_packed(src, w, fill, edgeset=True).cpu().numpy().view(np.uint64)
            assert (es == P.edge_set(ref, fill).words).all(), (w, h, fill)


def test_flat_matches_unal_kernel(cuda_dev, monkeypatch):
    """Same words as K1's UNAL items on a larger raster (both dispatches)."""
    import torch

    from paper_1401_5245_b200 import cuda as cu

    g = torch.Generator(device=cuda_dev).manual_seed(5)
    for w, bits in ((8000, 32), (8000, 64), (12345, 32), (30001, 64)):
        wp = -(-w // bits)
        dt = torch.int32 if bits == 32 else torch.int64
        x = torch.randint(-2**31, 2**31 - 1, (3000, wp * bits // 32), generator=g,
                          device=cuda_dev, dtype=torch.int64).to(torch.int32).view(dt)
        a = cu.edges_packed(x, w, 1)
        monkeypatch.setenv("BITEDGE_NO_FLAT", "1")
        b = cu.edges_packed(x, w, 1)
        monkeypatch.delenv("BITEDGE_NO_FLAT")
        assert torch.equal(a, b), (w, bits)

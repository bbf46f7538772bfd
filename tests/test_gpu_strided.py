"""Primitives on strided views (row stride > words per row): every word-op entry
point (invert / and / or / shift / shift_and / scan_edges) must give the same
words as on a contiguous copy, and the output must keep the input's geometry
(outputs were allocated contiguous but written with the input's
stride)."""

import numpy as np
import pytest

from oracle import port as P

pytestmark = pytest.mark.gpu


def _views(cuda_dev, h, wp, extra, seed, n=None):
    import torch

    rng = np.random.default_rng(seed)
    shape = (h, wp + extra) if n is None else (n, h, wp + extra)
    wide = torch.from_numpy(rng.integers(-2**63, 2**63 - 1, shape, dtype=np.int64)).to(cuda_dev)
    view = wide[..., :wp]
    assert view.stride(-2) == wp + extra
    return wide, view, view.contiguous()


@pytest.mark.parametrize("h,width,extra,n", [(7, 130, 3, None), (33, 64, 1, None),
                                             (5, 200, 8, 3), (1, 70, 2, 4)])
def test_primitives_on_strided_views(cuda_dev, h, width, extra, n):
    import torch

    from paper_1401_5245_b200 import cuda as cu

    wp = -(-width // 64)
    _, a, ac = _views(cuda_dev, h, wp, extra, 1, n)
    _, b, bc = _views(cuda_dev, h, wp, extra, 2, n)

    def same(x, y):
        assert x.shape == y.shape
        assert torch.equal(x.contiguous(), y.contiguous())

    same(cu.invert(a, width), cu.invert(ac, width))
    same(cu.and_(a, b, width), cu.and_(ac, bc, width))
    same(cu.or_(a, b, width), cu.or_(ac, bc, width))
    for d in range(4):
        for fill in (0, 1):
            same(cu.shift(a, width, d, fill), cu.shift(ac, width, d, fill))
            same(cu.shift_and(a, b, width, d, fill), cu.shift_and(ac, bc, width, d, fill))
    for fill in (0, 1):
        same(cu.scan_edges(a, width, fill), cu.scan_edges(ac, width, fill))
        same(cu.edges_packed(a, width, fill), cu.edges_packed(ac, width, fill))
    torch.cuda.synchronize()
    # and the contiguous result is the oracle's
    if n is None:
        words = ac.cpu().numpy().view(np.uint64)
        img = P.make(width, h, words)
        got = cu.edges_packed(a, width, 1).cpu().numpy().view(np.uint64)
        assert (got == P.detect_edges_mask(img, 1).words).all()
        got = cu.invert(a, width).cpu().numpy().view(np.uint64)
        assert (got == P.invert(img).words).all()


def test_strided_output_keeps_neighbour_memory(cuda_dev):
    """The padding words past each row of the output view are outside the view;
    writing the primitives' results must not disturb memory after the output."""
    import torch

    from paper_1401_5245_b200 import cuda as cu

    h, width, extra = 16, 192, 5
    wp = 3
    _, a, ac = _views(cuda_dev, h, wp, extra, 3)
    guard = torch.full((1 << 16,), 0x5A5A5A5A, dtype=torch.int32, device=cuda_dev)
    for _ in range(4):
        o = cu.invert(a, width)
        assert o.stride(0) == wp + extra
    torch.cuda.synchronize()
    assert bool((guard == 0x5A5A5A5A).all())
    assert torch.equal(o.contiguous(), cu.invert(ac, width))

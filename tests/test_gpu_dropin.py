"""The drop-in BitImage's deferred pack: `from_array` on a host array uploads
the pixels and defers packing to the first consumer; detect_edges_mask /
edge_set fuse it into their launch (and leave the packed words behind), every
other consumer packs first.  All results word-identical to the reference
composition (oracle/port.py)."""

import numpy as np
import pytest

from oracle import port as P

pytestmark = pytest.mark.gpu


def _img(seed, h=37, w=130):
    rng = np.random.default_rng(seed)
    return (rng.random((h, w)) < 0.5).astype(np.uint8) * rng.integers(1, 256, (h, w)).astype(np.uint8)


@pytest.mark.parametrize("policy", ["WHITE_OUTSIDE", "BLACK_OUTSIDE"])
def test_fused_pack_then_words(policy, cuda_dev):
    from paper_1401_5245_b200.bitimage import BitImage, BorderPolicy
    from paper_1401_5245_b200.edge import detect_edges_mask, edge_set

    b = BorderPolicy[policy]
    for seed, (h, w) in enumerate([(37, 130), (1, 1), (64, 64), (5, 2048), (300, 7)]):
        a = _img(seed, h, w)
        ref = P.from_array(a)
        img = BitImage.from_array(a)
        assert img._pix is not None                          # deferred
        e = detect_edges_mask(img, b)
        assert img._pix is None and img._dev is not None     # packed by the same launch
        assert (e.words == P.detect_edges_mask(ref, b.value).words).all()
        assert (img.words == ref.words).all()
        img2 = BitImage.from_array(a)
        es = edge_set(img2, b)
        assert (es.words == P.edge_set(ref, b.value).words).all()
        assert (img2.words == ref.words).all()


def test_other_consumers_pack_first(cuda_dev):
    from paper_1401_5245_b200.bitimage import BitImage, Direction
    from paper_1401_5245_b200.edge import detect_edges_mask

    a = _img(9, 45, 200)
    ref = P.from_array(a)
    for consume in (lambda i: i.invert(), lambda i: i.shift(Direction.LEFT),
                    lambda i: i.count_black(), lambda i: i.to_array(), lambda i: i.words,
                    lambda i: hash(i), lambda i: i == BitImage.from_array(a)):
        img = BitImage.from_array(a)
        consume(img)
        assert img._pix is None
        assert (img.words == ref.words).all()
        assert (detect_edges_mask(img).words == P.detect_edges_mask(ref).words).all()
    assert BitImage.from_array(a) == BitImage.from_array(a)
    assert BitImage.from_array(a).count_black() == int((a == 0).sum())


def test_consumer_on_another_stream(cuda_dev):
    import torch

    from paper_1401_5245_b200.bitimage import BitImage
    from paper_1401_5245_b200.edge import detect_edges_mask

    a = _img(3, 512, 1024)
    ref = P.from_array(a)
    s = torch.cuda.Stream()
    imgs = [BitImage.from_array(a) for _ in range(4)]        # uploaded on the default stream
    with torch.cuda.stream(s):
        outs = [detect_edges_mask(i) for i in imgs]
        s.synchronize()
    for i, o in zip(imgs, outs):
        assert (o.words == P.detect_edges_mask(ref).words).all()
        assert (i.words == ref.words).all()


def test_device_tensor_input_is_packed_eagerly(cuda_dev):
    """A caller-owned CUDA tensor may change after from_array: packed at once."""
    import torch

    from paper_1401_5245_b200.bitimage import BitImage

    a = _img(4)
    t = torch.from_numpy(a).to(cuda_dev)
    img = BitImage.from_array(t)
    assert img._pix is None
    t.zero_()
    assert (img.words == P.from_array(a).words).all()

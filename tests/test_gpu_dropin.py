"""The drop-in BitImage's deferred pack: `from_array` on a host array keeps a
private copy of the pixels (pageable for small images, page-locked within a
budget for larger ones); detect_edges_mask / edge_set run upload, pack + edges
and the result's download as one call (the larger flow also leaves the packed
words behind), every other consumer uploads and packs first.  All results
word-identical to the reference composition (oracle/port.py)."""

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
        small = w < 1024 and h * w <= (1 << 20)
        e = detect_edges_mask(img, b)
        if small:       # staged one-call flow: nothing left on the device
            assert isinstance(img._pix, np.ndarray) and img._dev is None
        else:
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


def test_threads_share_the_library(cuda_dev):
    """The ABI is reentrant (thread-local error text and launch counter, no other
    state): eight host threads, each on its own stream, mixing kernels, u8/u32
    inputs and invalid calls, get exact results and their own error messages."""
    import threading

    import torch

    from oracle import cscan
    from paper_1401_5245_b200 import cuda as cu

    errors, results = [], {}

    def worker(k):
        try:
            rng = np.random.default_rng(100 + k)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for it in range(20):
                    h, w = int(rng.integers(1, 90)), int(rng.choice([64, 100, 2048, 33]))
                    a = (rng.random((2, h, w)) < 0.5).astype(np.uint8)
                    t = torch.from_numpy(a).to(cuda_dev, non_blocking=False)
                    if it % 2:
                        got = cu.pack_edges_u8(t, 1)
                    else:
                        got = cu.edges_packed(cu.pack_u8(t), w, 1)
                    try:
                        cu.edges_packed(cu.pack_u8(t), w + 1000, 1)   # too few words per row
                    except ValueError as e:
                        assert "words per row" in str(e)
                    s.synchronize()
                    results[(k, it)] = (got.cpu().numpy().view(np.uint32), cscan.scan_u8(a, 1))
        except Exception as e:      # pragma: no cover - reported below
            errors.append((k, repr(e)))

    th = [threading.Thread(target=worker, args=(k,)) for k in range(8)]
    for t_ in th:
        t_.start()
    for t_ in th:
        t_.join()
    assert not errors, errors
    assert len(results) == 160
    for key, (got, exp) in results.items():
        assert (got == exp).all(), key


@pytest.mark.parametrize("w", [1024, 1056, 1100, 2048, 2080, 3000, 4096, 100])
def test_u8_to_u64_words(w, cuda_dev):
    """uint8 pixels -> uint64 words (the BitImage layout) through K2t2's swapped
    stores (w >= 1024) or the tile kernel: pack, fused pack+edges, every output,
    BLACK_OUTSIDE, a threshold; padding words included (odd uint32 counts)."""
    import torch

    from paper_1401_5245_b200 import cuda as cu

    rng = np.random.default_rng(w)
    for n, h in [(1, 37), (3, 9)]:
        a = (rng.random((n, h, w)) < 0.5).astype(np.uint8)
        g = torch.from_numpy(a * rng.integers(1, 256, a.shape).astype(np.uint8)).to(cuda_dev)
        refs = [P.from_array(x) for x in a]
        pk = cu.pack_u8(g, word_bits=64).cpu().numpy().view(np.uint64)
        assert (pk == np.stack([r.words for r in refs])).all(), (w, n, h)
        for fill in (1, 0):
            e, p2 = cu.pack_and_edges(g, fill, word_bits=64)
            exp = np.stack([P.detect_edges_mask(r, fill).words for r in refs])
            assert (e.cpu().numpy().view(np.uint64) == exp).all(), (w, n, h, fill)
            assert (p2.cpu().numpy().view(np.uint64) == np.stack([r.words for r in refs])).all()
        res = cu.edges_general(g, None, 1, word_bits=64, edgeset=True, sides=True, packed=True)
        for k, d in (("left", P.LEFT), ("right", P.RIGHT), ("up", P.UP), ("down", P.DOWN)):
            exp = np.stack([P.fundamental_edge(r, P.build_mask(r), d, 1).words for r in refs])
            assert (res[k].cpu().numpy().view(np.uint64) == exp).all(), (w, k)
        exp = np.stack([P.edge_set(r, 1).words for r in refs])
        assert (res["edgeset"].cpu().numpy().view(np.uint64) == exp).all()
        # a threshold: gray >= 200 is white
        gray = torch.from_numpy(rng.integers(0, 256, (n, h, w)).astype(np.uint8)).to(cuda_dev)
        th = cu.threshold_u8(gray, 200, word_bits=64).cpu().numpy().view(np.uint64)
        expt = np.stack([P.from_array((x >= 200).astype(np.uint8)).words
                         for x in gray.cpu().numpy()])
        assert (th == expt).all(), (w, "threshold")


@pytest.mark.parametrize("policy", ["WHITE_OUTSIDE", "BLACK_OUTSIDE"])
def test_host_flow_one_call(policy, cuda_dev):
    """from_array of a host array keeps a private page-locked copy; the first
    detect_edges_mask / edge_set uploads, packs + detects and downloads in one
    native call (be_host_detect_u64): host words ready, device words equal, the
    input keeps its packed words, and later mutation of the caller's array does
    not leak in."""
    import torch

    from paper_1401_5245_b200.bitimage import BitImage, BorderPolicy
    from paper_1401_5245_b200.edge import detect_edges_mask, edge_set

    b = BorderPolicy[policy]
    for seed, (h, w) in enumerate([(1, 1), (256, 256), (37, 130), (3, 1100), (70, 4160),
                                   (2, 3000), (500, 1)]):
        a = _img(100 + seed, h, w)
        ref = P.from_array(a)
        exp = P.detect_edges_mask(ref, b.value).words
        src = a.copy()
        img = BitImage.from_array(src)
        src[...] = 0                                        # the image owns its pixels
        assert img._pix is not None and not getattr(img._pix, "is_cuda", False)
        e = detect_edges_mask(img, b)
        assert e._words is not None                         # downloaded by the same call
        assert (e.words == exp).all()
        assert (e.device_words().cpu().numpy().view(np.uint64) == exp).all()
        assert (img.words == ref.words).all()               # packed input kept
        # the result chains on the device like any other image
        assert (detect_edges_mask(e, b).words ==
                P.detect_edges_mask(P.make(w, h, exp.copy()), b.value).words).all()
        es = edge_set(BitImage.from_array(a), b)
        assert (es.words == P.edge_set(ref, b.value).words).all()
    torch.cuda.synchronize()


def test_host_flow_input_dtypes(cuda_dev):
    """Nonzero = white for every input dtype (bitimage.py:124,133)."""
    from paper_1401_5245_b200.bitimage import BitImage
    from paper_1401_5245_b200.edge import detect_edges_mask

    rng = np.random.default_rng(7)
    base = (rng.random((33, 77)) < 0.5)
    exp = P.detect_edges_mask(P.from_array(base.astype(np.uint8))).words
    for a in (base, base.astype(np.int8) * -3, base.astype(np.uint8) * 200,
              base.astype(np.int32) * 5, base.astype(np.float32) * 0.5, base.astype(np.int64) - 0,
              np.asfortranarray(base.astype(np.uint8)), base.astype(np.uint8)[:, ::-1][:, ::-1]):
        assert (detect_edges_mask(BitImage.from_array(a)).words == exp).all(), a.dtype


@pytest.mark.parametrize("zero_copy", [True, False])
def test_host_detect_copy_modes(zero_copy, cuda_dev):
    """be_host_detect_u64 with device staging (H2D / kernel / D2H) and with the
    kernel reading and writing page-locked host memory itself: same words."""
    import torch

    from paper_1401_5245_b200 import cuda as cu

    for seed, (h, w) in enumerate([(1, 1), (64, 64), (256, 256), (9, 1000), (130, 63)]):
        a = _img(200 + seed, h, w)
        hp = torch.empty((h, w), dtype=torch.uint8, pin_memory=True)
        hp.numpy()[...] = a
        ref = P.from_array(a)
        for fill in (1, 0):
            for es in (False, True):
                out, packed, words = cu.host_detect(hp, fill, edgeset=es, zero_copy=zero_copy)
                exp = (P.edge_set if es else P.detect_edges_mask)(ref, fill).words
                assert (words == exp).all(), (h, w, fill, es)
                assert (packed.cpu().numpy().view(np.uint64) == ref.words).all()
                if out is not None:
                    assert (out.cpu().numpy().view(np.uint64) == exp).all()
    if zero_copy:
        hp = torch.empty((2, 1024), dtype=torch.uint8, pin_memory=True)
        with pytest.raises(ValueError, match="zero-copy"):
            cu.host_detect(hp, 1, zero_copy=True)


def test_large_host_array_packed_at_once(cuda_dev, monkeypatch):
    """Above the page-locked copy limit from_array uploads and packs at once
    (same words, same edges)."""
    from paper_1401_5245_b200 import bitimage as B
    from paper_1401_5245_b200.edge import detect_edges_mask

    monkeypatch.setattr(B, "_PINNED_MAX", 1000)
    # wider than the small-image flow's 1023 px: the page-locked path's limit applies
    for a in (_img(7, 40, 1030), _img(8, 40, 1030).astype(np.int32)):
        img = B.BitImage.from_array(a)
        assert img._pix is None and img._dev is not None
        ref = P.from_array(a)
        assert (img.words == ref.words).all()
        assert (detect_edges_mask(img).words == P.detect_edges_mask(ref).words).all()


def test_host_detect_refuses_pageable_zero_copy(cuda_dev):
    """be_host_detect_u64's zero-copy mode checks that both host buffers are
    page-locked instead of letting the kernel fault."""
    import torch

    from paper_1401_5245_b200 import _capi

    h, w = 8, 40
    pix = np.ones((h, w), np.uint8)                      # pageable
    out = np.empty((h, 1), np.uint64)
    pk = torch.empty((h, 1), dtype=torch.int64, device=cuda_dev)
    rc = _capi.fn("be_host_detect_u64")(pix.ctypes.data, h, w, 1, 0, None, pk.data_ptr(), None,
                                        out.ctypes.data, None)
    assert rc < 0 and b"page-locked" in _capi.load().be_last_error()
    torch.cuda.synchronize()                             # the context is still healthy
    hp = torch.ones((h, w), dtype=torch.uint8, pin_memory=True)
    rc = _capi.fn("be_host_detect_u64")(hp.data_ptr(), h, w, 1, 0, None, pk.data_ptr(), None,
                                        out.ctypes.data, None)
    assert rc < 0


def test_small_flow_input_forms(cuda_dev):
    """The staged small-image flow on non-contiguous, reversed, bool and int
    arrays, and the caller mutating its array after from_array."""
    from paper_1401_5245_b200.bitimage import BitImage
    from paper_1401_5245_b200.edge import detect_edges_mask, edge_set

    base = _img(11, 80, 300)
    for a in (base[:, ::-1], base[::2, 5:250], base.astype(bool), base.astype(np.int32) * -3,
              np.asfortranarray(base), base[::-1]):
        ref = P.from_array(a)
        img = BitImage.from_array(a)
        assert (detect_edges_mask(img).words == P.detect_edges_mask(ref).words).all()
        assert (edge_set(img).words == P.edge_set(ref).words).all()
        assert (img.words == ref.words).all()
    a = base.copy()
    img = BitImage.from_array(a)
    a[:] = 0                                                  # private copy: unaffected
    ref = P.from_array(base)
    assert (detect_edges_mask(img).words == P.detect_edges_mask(ref).words).all()


def test_pinned_budget_bounds_pending_copies(cuda_dev, monkeypatch):
    """Pending page-locked copies never exceed the budget: past it, from_array
    uploads and packs at once; the held bytes return to zero as images go."""
    import gc

    from paper_1401_5245_b200 import bitimage as B
    from paper_1401_5245_b200.edge import detect_edges_mask

    monkeypatch.setattr(B, "_PINNED_BUDGET", 3 * 1200 * 1100)
    gc.collect()
    held0 = B._pinned_held[0]
    a = _img(12, 1200, 1100)                  # > 1 Mpx: the page-locked flow
    ref = P.from_array(a)
    imgs = [B.BitImage.from_array(a) for _ in range(5)]
    pending = [i for i in imgs if i._pix is not None]
    assert len(pending) == 3 and all(i._dev is not None for i in imgs[3:])
    assert B._pinned_held[0] - held0 == 3 * 1200 * 1100
    for i in imgs:
        assert (detect_edges_mask(i).words == P.detect_edges_mask(ref).words).all()
        assert (i.words == ref.words).all()
    del imgs, pending, i
    gc.collect()
    assert B._pinned_held[0] == held0


def test_small_flow_from_threads(cuda_dev):
    """Per-thread staging: eight threads running the one-call flow at once."""
    import threading

    from paper_1401_5245_b200.bitimage import BitImage
    from paper_1401_5245_b200.edge import detect_edges_mask

    errors = []

    def worker(k):
        try:
            for it in range(40):
                a = _img(1000 * k + it, 20 + it, 64 + 7 * k)
                got = detect_edges_mask(BitImage.from_array(a)).words
                assert (got == P.detect_edges_mask(P.from_array(a)).words).all()
        except Exception as e:  # pragma: no cover
            errors.append(repr(e))

    th = [threading.Thread(target=worker, args=(k,)) for k in range(8)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors

"""Out-of-bounds checks by sentinels (compute-sanitizer is not available on the
GPU pool): every output is a view into a larger buffer whose guard words
before and after the view, whose row-stride padding and whose rows outside
[row_lo, row_hi) hold a sentinel that no kernel may overwrite; every input
carries garbage in its row padding (and in the bytes around it) that no
output may depend on.  Runs over every kernel-selection knob."""

import numpy as np
import pytest

from oracle import cscan
from oracle import port as P

pytestmark = pytest.mark.gpu

KNOBS = [{}, {"BITEDGE_KERNEL": "tile"}, {"BITEDGE_KERNEL": "stream"}, {"BITEDGE_CW4": "1"},
         {"BITEDGE_NO_ROLL": "1"}, {"BITEDGE_NO_WARPIMG": "1"}, {"BITEDGE_FORCE_TMA": "1"},
         {"BITEDGE_FORCE_TMA": "1", "BITEDGE_TMA1": "1"}, {"BITEDGE_RS": "8"},
         {"BITEDGE_FORCE_TMA": "1", "BITEDGE_TMA2_RSL32": "1"}, {"BITEDGE_FORCE_TMA": "1", "BITEDGE_TMA2_RSL": "5"}, {"BITEDGE_FORCE_TMA": "1", "BITEDGE_TMA2_RSL": "11"}, {"BITEDGE_K1_GENERIC": "1"}, {"BITEDGE_NO_UNAL": "1"}, {"BITEDGE_NO_TMA": "1"}]
SHAPES = [(3, 64, 64), (1, 37, 2048), (2, 19, 1000), (1, 5, 4096), (4, 9, 33), (1, 70, 3000)]
SENT = 0x5A5A5A5A
GUARD = 96                                   # words before and after each output view


def _guarded(dev, n, h, wp, pad, wb):
    """An [n, h, wp] output view with `pad` extra words per row and GUARD words
    either side, all set to the sentinel.  Returns (buffer, view)."""
    import torch

    dt = torch.int64 if wb == 64 else torch.int32
    per = 2 if wb == 64 else 1
    total = GUARD * 2 + n * h * (wp + pad) * per
    buf = torch.full((total // per + 1,), 0, dtype=dt, device=dev)
    buf.view(torch.int32).fill_(SENT)
    view = buf[GUARD // per: GUARD // per + n * h * (wp + pad)].view(n, h, wp + pad)[..., :wp]
    return buf, view


def _mask(n, h, wp, pad, wb, lo, hi):
    """Boolean mask over the buffer's int32 words: True where the kernel may write."""
    per = 2 if wb == 64 else 1
    m = np.zeros(n * h * (wp + pad) * per, bool)
    rows = m.reshape(n * h, (wp + pad) * per)
    rows[lo:hi, : wp * per] = True
    full = np.zeros(GUARD * 2 + m.size + per, bool)
    full[GUARD: GUARD + m.size] = m
    return full


def _input(dev, a, kind, rng):
    """`a` (uint8 0/1 [n,h,w]) as uint8 / u32 / u64 rows in a larger buffer with
    garbage in the row padding, a garbage byte/word region after the last row
    and garbage in the padding bits of the last word of every row."""
    import torch

    n, h, w = a.shape
    if kind == "u8":
        g = a * rng.integers(1, 256, a.shape).astype(np.uint8)
        pad = int(rng.integers(1, 48))
        buf = rng.integers(0, 256, n * h * (w + pad) + 256).astype(np.uint8)
        t = torch.from_numpy(buf).to(dev)
        view = t[: n * h * (w + pad)].view(n, h, w + pad)[..., :w]
        view.copy_(torch.from_numpy(g).to(dev))
        return view, 32
    if kind == "u32":
        words = P.pack_u32(a)
        wp = words.shape[2]
        junk = np.uint32(0xFFFFFFFF) >> np.uint32(w % 32) if w % 32 else np.uint32(0)
        words[..., -1] ^= junk & rng.integers(0, 2 ** 32, (n, h), dtype=np.uint64).astype(np.uint32)
        pad = int(rng.integers(1, 6))
        buf = rng.integers(-2 ** 31, 2 ** 31, n * h * (wp + pad) + 64).astype(np.int32)
        t = torch.from_numpy(buf).to(dev)
        view = t[: n * h * (wp + pad)].view(n, h, wp + pad)[..., :wp]
        view.copy_(torch.from_numpy(words.view(np.int32)).to(dev))
        return view, 32
    words = np.stack([P.from_array(x).words for x in a])       # u64, padding = 1
    wp = words.shape[2]
    if w % 64:
        junk = np.uint64(0xFFFFFFFFFFFFFFFF) >> np.uint64(w % 64)
        # the drop-in layout keeps padding at 1; the kernel must not read it anyway
        words[..., -1] ^= junk & rng.integers(0, 2 ** 63, (n, h), dtype=np.uint64)
    pad = int(rng.integers(1, 4))
    buf = rng.integers(-2 ** 62, 2 ** 62, n * h * (wp + pad) + 32).astype(np.int64)
    t = torch.from_numpy(buf).to(dev)
    view = t[: n * h * (wp + pad)].view(n, h, wp + pad)[..., :wp]
    view.copy_(torch.from_numpy(words.view(np.int64)).to(dev))
    return view, 64


@pytest.mark.parametrize("knob", KNOBS, ids=lambda k: ",".join(f"{a}={b}" for a, b in k.items()) or "default")
def test_guards(knob, cuda_dev, monkeypatch):
    from paper_1401_5245_b200 import cuda as cu

    for k, v in knob.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(77)
    for (n, h, w) in SHAPES:
        a = (rng.random((n, h, w)) < 0.5).astype(np.uint8)
        exp = cscan.scan_u8(a, 1)                               # [n, h, wp32] u32 rows
        for kind in ("u8", "u32", "u64"):
            inp, wb = _input(cuda_dev, a, kind, rng)
            wp = cu.words_per_row(w, wb)
            pad = int(rng.integers(1, 5))
            lo = int(rng.integers(0, n * h))
            hi = int(rng.integers(lo + 1, n * h + 1))
            bufs, outs = {}, {}
            for name in ("edges", "edgeset", "left", "down"):
                bufs[name], outs[name] = _guarded(cuda_dev, n, h, wp, pad, wb)
            cu.edges_general(inp, None if kind == "u8" else w, 1, word_bits=wb, edgeset=True,
                             sides=False, row_lo=lo, row_hi=hi, outs=outs)
            allowed = _mask(n, h, wp, pad, wb, lo, hi)
            for name, buf in bufs.items():
                words = buf.view(-1).cpu().numpy().view(np.uint32)[: allowed.size]
                bad = np.flatnonzero((words != np.uint32(SENT)) & ~allowed[: words.size])
                assert bad.size == 0, (knob, kind, n, h, w, name, lo, hi, bad[:8])
            got = outs["edges"].cpu().numpy().reshape(n * h, -1)[lo:hi]
            if wb == 64:
                got = P.u64_to_u32_rows(got.view(np.uint64))[:, : -(-w // 32)]
            else:
                got = got.view(np.uint32)
            assert (got == exp.reshape(n * h, -1)[lo:hi]).all(), (knob, kind, n, h, w, lo, hi)


@pytest.mark.parametrize("knob", KNOBS[:1] + KNOBS[6:8], ids=["default", "tma2", "tma1"])
def test_input_garbage_does_not_leak(knob, cuda_dev, monkeypatch):
    """Same image, different garbage around it -> identical words."""
    from paper_1401_5245_b200 import cuda as cu

    for k, v in knob.items():
        monkeypatch.setenv(k, v)
    for (n, h, w) in SHAPES:
        a = (np.random.default_rng(w).random((n, h, w)) < 0.3).astype(np.uint8)
        for kind in ("u8", "u32", "u64"):
            res = []
            for seed in (1, 2):
                inp, wb = _input(cuda_dev, a, kind, np.random.default_rng(seed))
                r = cu.edges_general(inp, None if kind == "u8" else w, 1, word_bits=wb,
                                     edgeset=True, sides=True)
                res.append({k: v.cpu().numpy() for k, v in r.items()})
            for k in res[0]:
                assert (res[0][k] == res[1][k]).all(), (knob, kind, n, h, w, k)


@pytest.mark.parametrize("G", [256, 259], ids=["aligned", "misaligned"])
@pytest.mark.parametrize("w", [128, 2048, 4096, 96, 8000, 32, 100, 1000, 7])
def test_p4_guards(w, G, cuda_dev):
    """be_p4_edges (K1 for 16-byte or 4-byte rows, the byte kernel otherwise)
    writes exactly n*h*ceil(w/8) bytes; the payload's unused trailing bits are
    zero (PBM convention)."""
    import ctypes

    import torch

    from paper_1401_5245_b200 import _capi

    rng = np.random.default_rng(w)
    n, h = 3, 21
    rb = (w + 7) // 8
    a = (rng.random((n, h, w)) < 0.5).astype(np.uint8)
    bits = np.ones((n, h, rb * 8), np.uint8)
    bits[..., :w] = a
    payload = np.packbits(1 - bits, axis=-1).reshape(-1)
    src = torch.from_numpy(np.concatenate([payload, rng.integers(0, 256, 512).astype(np.uint8)]))
    src = src.to(cuda_dev)
    buf = torch.full((G + n * h * rb + G,), 0xA5, dtype=torch.uint8, device=cuda_dev)
    scratch = torch.empty(2 * n * h * ((w + 31) // 32), dtype=torch.int32, device=cuda_dev)
    _capi.call("be_p4_edges", ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(buf.data_ptr() + G),
               n, h, w, 1, ctypes.c_void_p(scratch.data_ptr()),
               ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    host = buf.cpu().numpy()
    assert (host[:G] == 0xA5).all() and (host[G + n * h * rb:] == 0xA5).all()
    out = host[G: G + n * h * rb].reshape(n, h, rb)
    got = 1 - np.unpackbits(out, axis=-1)[..., :w]
    assert (got == P.unpack_u32(cscan.scan_u8(a, 1), w)).all()


@pytest.mark.parametrize("n,h,w", [(8, 64, 64), (9, 64, 64), (100, 32, 32), (333, 64, 128),
                                   (1183, 64, 64), (1185, 48, 64), (4096, 64, 64),
                                   (5000, 32, 64), (700, 224, 32)])
def test_k2p_guarded_batches(cuda_dev, n, h, w, monkeypatch):
    """K2p (opt-in, BITEDGE_K2P: whole glyph batch requested by TMA at kernel
    start, one CTA per SM):
    image counts that are not multiples of the warp count, mbarrier header and
    image buffers side by side in shared memory -- output bit-exact, nothing
    written past the batch (guard words), EdgeSet too."""
    import torch

    from paper_1401_5245_b200 import cuda as cu

    monkeypatch.setenv("BITEDGE_K2P", "1")
    rng = np.random.default_rng(n * 7 + h)
    a = (rng.random((n, h, w)) < 0.6).astype(np.uint8)
    # garbage bytes after the last image (a warp reading a nonexistent image
    # would pick them up and write their edges into the guard words)
    src = torch.from_numpy(np.concatenate([a.reshape(-1), rng.integers(0, 256, 64 * 1024,
                                                                        dtype=np.uint8)]))
    x = src.to(cuda_dev)[: a.size].view(n, h, w)
    wp = -(-w // 32)
    for fill in (1, 0):
        for eset in (False, True):
            buf = torch.full((n * h * wp + 2 * GUARD,), SENT, dtype=torch.int32, device=cuda_dev)
            view = buf[GUARD: GUARD + n * h * wp].view(n, h, wp)
            if eset:
                cu.edges_general(x, w, fill, edges=False, edgeset=True, outs={"edgeset": view})
            else:
                cu.pack_edges_u8(x, fill, out=view)
            torch.cuda.synchronize()
            b = buf.cpu().numpy()
            assert (b[:GUARD] == SENT).all() and (b[GUARD + n * h * wp:] == SENT).all()
            exp = cscan.scan_u8(a, fill, edgeset=eset)
            assert (view.cpu().numpy().view(np.uint32) == exp).all(), (n, h, w, fill, eset)


@pytest.mark.parametrize("k2p", ["0", "1"])
def test_glyph_batches_concurrent_streams(cuda_dev, k2p, monkeypatch):
    """The bench's schedule (K2w by default, K2p opt-in): C2 batches on three parallel streams (CUDA graph
    replay, PDL between consecutive launches of a stream), distinct outputs,
    every output bit-exact."""
    import torch

    from paper_1401_5245_b200 import cuda as cu
    from paper_1401_5245_b200 import synth

    if k2p == "1":
        monkeypatch.setenv("BITEDGE_K2P", "1")
    imgs = synth.c2_images(4096)
    exp = cscan.scan_u8(imgs.numpy(), 1)
    x = imgs.to(cuda_dev)
    outs = [torch.empty((4096, 64, 2), dtype=torch.int32, device=cuda_dev) for _ in range(24)]
    side = [torch.cuda.Stream(cuda_dev) for _ in range(3)]
    g = torch.cuda.CUDAGraph()
    cur = torch.cuda.current_stream(cuda_dev)
    for s_ in side:
        s_.wait_stream(cur)
    with torch.cuda.stream(side[0]):
        cu.pack_edges_u8(x, 1, out=outs[0])             # warm-up outside the capture
    cur.wait_stream(side[0])
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        c = torch.cuda.current_stream(cuda_dev)
        for s_ in side:
            s_.wait_stream(c)
        for i in range(len(outs)):
            with torch.cuda.stream(side[i % 3]):
                cu.pack_edges_u8(x, 1, out=outs[i])
        for s_ in side:
            c.wait_stream(s_)
    for _ in range(20):
        for o in outs:
            o.fill_(0)
        g.replay()
        torch.cuda.synchronize()
        for o in outs:
            assert (o.cpu().numpy().view(np.uint32) == exp).all()

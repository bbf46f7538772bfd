"""GPU parity: the sm_100a kernels (through the C ABI) against the oracle and
the golden vectors the real reference produced.  Bit-exact on every word,
padding included.  Run with `pytest -m gpu` on a B200."""

import hashlib

import numpy as np
import pytest

from conftest import encode_bits, exhaustive_images, golden, split_corpus
from oracle import cscan
from oracle import port as P

pytestmark = pytest.mark.gpu

POL = {"WHITE_OUTSIDE": 1, "BLACK_OUTSIDE": 0}


def _t(a, dev):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


def _u64(t):
    return t.cpu().numpy().view(np.uint64)


# ---------------------------------------------------------------- exhaustive (SPEC acceptance 1)

@pytest.mark.parametrize("n", [3, 4])
@pytest.mark.parametrize("pol", list(POL))
def test_exhaustive_batch_u8(cuda_dev, n, pol):
    """All 2^(n*n) rasters as ONE batch through the fused pack+edge kernel."""
    from paper_1401_5245_b200 import cuda as cu

    g = golden("exhaustive.npz")
    imgs = exhaustive_images(n)
    fill = POL[pol]
    out = cu.pack_edges_u8(_t(imgs, cuda_dev), fill)
    bits = P.unpack_u32(_u32(out), n)
    assert (encode_bits(bits) == g[f"out{n}_{pol}"]).all()
    # padding of every output word is 1
    assert ((_u32(out) & np.uint32((1 << (32 - n)) - 1)) == (1 << (32 - n)) - 1).all()
    # packed-input path (K1, u32 and u64 words) and the EdgeSet
    packed32 = _t(P.pack_u32(imgs).view(np.int32), cuda_dev)
    assert (_u32(cu.edges_packed(packed32, n, fill)) == _u32(out)).all()
    es = cu.edges_packed(packed32, n, fill, edgeset=True)
    assert (encode_bits(P.unpack_u32(_u32(es), n)) == g[f"eset{n}_{pol}"]).all()
    packed64 = cu.pack_u8(_t(imgs, cuda_dev), word_bits=64)
    o64 = cu.edges_packed(packed64, n, fill)
    w64 = _u64(o64)                                   # [K, n, 1] native u64 words
    bits64 = np.unpackbits(w64.astype(">u8").view(np.uint8).reshape(len(imgs), n, 8),
                           axis=-1)[..., :n]
    assert (encode_bits(bits64) == g[f"out{n}_{pol}"]).all()      # every raster
    pad64 = np.uint64((1 << (64 - n)) - 1)
    assert ((w64 & pad64) == pad64).all()
    exp64 = np.stack([P.detect_edges_mask(P.from_array(imgs[i]), fill).words
                      for i in range(0, len(imgs), 257)])
    assert (w64[::257] == exp64).all()


# ---------------------------------------------------------------- random corpus (acceptance 1c)

def _corpus():
    g = golden("random.npz")
    pix, packed = split_corpus(g["shapes"], g["pixels"], g["packed"])
    return g, pix, packed


def test_random_corpus_bitimage_api(cuda_dev):
    """The drop-in API (BitImage + edge module) vs reference words, per image."""
    from paper_1401_5245_b200 import edge as E
    from paper_1401_5245_b200.bitimage import BitImage, BorderPolicy, Direction, first_difference

    g, pix, packed = _corpus()
    outs = {p: split_corpus(g["shapes"], g["pixels"], g[f"out_{p}"])[1] for p in POL}
    esets = {p: split_corpus(g["shapes"], g["pixels"], g[f"eset_{p}"])[1] for p in POL}
    funds = {(s, p): split_corpus(g["shapes"], g["pixels"], g[f"fund_{s}_{p}"])[1]
             for s in ("LEFT", "RIGHT", "UP", "DOWN") for p in POL}
    for i, a in enumerate(pix):
        img = BitImage.from_array(a)
        assert (img.words == packed[i]).all(), i
        for pol in POL:
            b = BorderPolicy[pol]
            out = E.detect_edges_mask(img, b)
            assert (out.words == outs[pol][i]).all(), (i, pol)
            if i % 7 == 0:
                assert (E.edge_set(img, b).words == esets[pol][i]).all()
                assert (E.detect_edges_scan(img, b).words == outs[pol][i]).all()
                m = E.build_mask(img)
                for s in ("LEFT", "RIGHT", "UP", "DOWN"):
                    fe = E.fundamental_edge(img, m, Direction[s], b)
                    assert (fe.words == funds[(s, pol)][i]).all(), (i, s, pol)
                fes = E.fundamental_edges(img, b)
                for s in ("LEFT", "RIGHT", "UP", "DOWN"):
                    assert (fes[Direction[s]].words == funds[(s, pol)][i]).all()
                assert (fes["edges"].words == outs[pol][i]).all()
                assert first_difference(out, E.detect_edges_scan(img, b)) is None
        if i % 50 == 0:
            assert (img.to_array() == (a != 0)).all()


def test_random_corpus_batched_u32(cuda_dev):
    """Same corpus through the tensor API: u8 -> fused pack+edge and packed u32."""
    from paper_1401_5245_b200 import cuda as cu

    g, pix, _ = _corpus()
    outs = {p: split_corpus(g["shapes"], g["pixels"], g[f"out_{p}"])[1] for p in POL}
    for i, a in enumerate(pix):
        w = a.shape[1]
        for pol, fill in POL.items():
            exp = P.u64_to_u32_rows(outs[pol][i])[:, : -(-w // 32)]
            got = _u32(cu.pack_edges_u8(_t(a, cuda_dev), fill))
            assert (got == exp).all(), (i, pol)
            if i % 5 == 0:
                pk = _t(P.pack_u32(a).view(np.int32), cuda_dev)
                assert (_u32(cu.edges_packed(pk, w, fill)) == exp).all()


def test_first_difference_and_queries(cuda_dev):
    from paper_1401_5245_b200.bitimage import BitImage, PixelColor, first_difference

    a = BitImage.from_array(np.ones((5, 70), np.uint8))
    b = a.set(66, 3, PixelColor.BLACK)
    assert first_difference(a, b) == (66, 3)
    assert b.count_black() == 1 and a.count_black() == 0
    assert repr(b) == "BitImage(70x5, black=1)"
    assert a != b and a == BitImage.filled(70, 5, PixelColor.WHITE)
    assert b.to_text().splitlines()[3][66] == "#"


# ---------------------------------------------------------------- primitives (acceptance 3)

def test_primitives_vs_reference(cuda_dev):
    from paper_1401_5245_b200.bitimage import BitImage, BorderPolicy, Direction

    g = golden("shift.npz")
    pix, _ = split_corpus(g["shapes"], g["pixels"])
    exp = {k: split_corpus(g["shapes"], g["pixels"], g[k])[1] for k in g.files
           if k.startswith("shift_") or k in ("invert", "and_rot", "or_rot")}
    W, B = BorderPolicy.WHITE_OUTSIDE, BorderPolicy.BLACK_OUTSIDE
    for i, a in enumerate(pix):
        img = BitImage.from_array(a)
        for s in ("LEFT", "RIGHT", "UP", "DOWN"):
            for pol in POL:
                got = img.shift(Direction[s], BorderPolicy[pol]).words
                assert (got == exp[f"shift_{s}_{pol}"][i]).all(), (i, s, pol)
        assert ((~img).words == exp["invert"][i]).all()
        assert ((img & img.shift(Direction.RIGHT, W)).words == exp["and_rot"][i]).all()
        assert ((img | img.shift(Direction.DOWN, B)).words == exp["or_rot"][i]).all()
        assert img.count_black() == g["count_black"][i]


def test_pack_rule_nonzero_bytes(cuda_dev):
    import torch

    from paper_1401_5245_b200 import cuda as cu
    from paper_1401_5245_b200.bitimage import BitImage

    a = np.array([[0, 1, 2, 255, 0, 17, 128, 0]] * 3, dtype=np.uint8)
    img = BitImage.from_array(a)
    assert img.to_array().tolist() == [[0, 1, 1, 1, 0, 1, 1, 0]] * 3
    assert BitImage.from_array(a.astype(np.int8)) == img
    assert BitImage.from_array(a.astype(np.float32) * 0.5) == img
    assert BitImage.from_array(a.astype(bool)) == img
    t = torch.from_numpy(a).cuda()
    assert (_u32(cu.pack_u8(t)) == P.pack_u32(a)).all()
    assert (cu.unpack_u8(cu.pack_u8(t), 8).cpu().numpy() == (a != 0)).all()


# ---------------------------------------------------------------- layouts / strides / alignment

def test_strided_and_unaligned_inputs(cuda_dev):
    import torch

    from paper_1401_5245_b200 import cuda as cu

    rng = np.random.default_rng(11)
    for (n, h, w) in [(3, 17, 45), (2, 9, 200), (1, 40, 1000), (5, 1, 33), (4, 33, 1)]:
        a = (rng.random((n, h, w)) < 0.55).astype(np.uint8) * rng.integers(1, 256, (n, h, w)).astype(np.uint8)
        exp = cscan.scan_u8(a, 1)
        # contiguous, unaligned row stride (byte path)
        assert (_u32(cu.pack_edges_u8(_t(a, cuda_dev), 1)) == exp).all(), (n, h, w)
        # padded row stride (vector path) via a view into a wider buffer
        wide = torch.zeros((n, h, (w + 15) // 16 * 16 + 16), dtype=torch.uint8, device=cuda_dev)
        wide[..., :w] = _t(a, cuda_dev)
        assert (_u32(cu.pack_edges_u8(wide[..., :w], 1)) == exp).all()
        # packed words with a padded stride (scalar + vector paths)
        pk = P.pack_u32(a)
        for extra in (0, 1, 3, 4):
            buf = np.full((n, h, pk.shape[2] + extra), 0xA5A5A5A5, dtype=np.uint32)
            buf[..., : pk.shape[2]] = pk
            t = _t(buf.view(np.int32), cuda_dev)[..., : pk.shape[2]]
            assert (_u32(cu.edges_packed(t, w, 1)) == exp).all(), (n, h, w, extra)


def test_garbage_padding_bits_ignored(cuda_dev):
    """Inputs with padding bits 0 (or random) give the same output as pad = 1."""
    from paper_1401_5245_b200 import cuda as cu

    rng = np.random.default_rng(5)
    for w in (1, 5, 31, 33, 63, 65, 100, 129):
        a = (rng.random((2, 7, w)) < 0.5).astype(np.uint8)
        pk = P.pack_u32(a)
        exp = cscan.scan_u8(a, 1)
        noisy = pk ^ (rng.integers(0, 2**32, pk.shape, dtype=np.uint32)
                      & np.uint32(P.u32_pad_mask(w) or 0))
        noisy[..., :-1] = pk[..., :-1]
        assert (_u32(cu.edges_packed(_t(noisy.view(np.int32), cuda_dev), w, 1)) == exp).all()
        cleared = pk.copy()
        cleared[..., -1] &= ~np.uint32(P.u32_pad_mask(w))
        got = _u32(cu.edges_packed(_t(cleared.view(np.int32), cuda_dev), w, 0))
        exp0 = cscan.scan_u8(a, 0)
        bad = np.argwhere(got != exp0)
        assert bad.size == 0, (w, bad[:4].tolist(), [hex(int(got[tuple(b)])) for b in bad[:4]],
                               [hex(int(exp0[tuple(b)])) for b in bad[:4]],
                               [hex(int(cleared[tuple(b)])) for b in bad[:4]])


# ---------------------------------------------------------------- BASELINE configs

def test_config_c1(cuda_dev):
    from paper_1401_5245_b200 import cuda as cu
    from paper_1401_5245_b200 import synth
    from paper_1401_5245_b200.bitimage import BitImage, BorderPolicy
    from paper_1401_5245_b200.edge import detect_edges_mask

    g = golden("configs.npz")
    c1 = synth.c1_image()
    img = BitImage.from_array(c1)
    assert (img.words == g["c1_input_packed"]).all()
    for pol in POL:
        assert (detect_edges_mask(img, BorderPolicy[pol]).words == g[f"c1_out_{pol}"]).all()
    got = _u32(cu.pack_edges_u8(_t(c1, cuda_dev), 1))
    assert (got == P.u64_to_u32_rows(g["c1_out_WHITE_OUTSIDE"])).all()


def test_config_c2_full(cuda_dev):
    """4096 glyphs generated on the device; output digest == the reference's."""
    from paper_1401_5245_b200 import cuda as cu
    from paper_1401_5245_b200 import synth

    g = golden("configs.npz")
    imgs = synth.c2_images(4096, device=cuda_dev)
    assert hashlib.sha256(imgs.cpu().numpy().tobytes()).digest() == g["c2_in_sha256"].tobytes()
    packed = torch_empty_like_words(imgs)
    out = cu.pack_edges_u8(imgs, 1, packed_out=packed)
    o = _u32(out)
    assert hashlib.sha256(o.tobytes()).digest() == g["c2_out_sha256"].tobytes()
    assert (o[:8] == P.u64_to_u32_rows(g["c2_head_out"].reshape(-1, 1)).reshape(8, 64, 2)).all()
    assert (_u32(packed) == P.pack_u32(imgs.cpu().numpy())).all()
    # K1 on the packed side output gives the same edges
    assert (_u32(cu.edges_packed(packed, 64, 1)) == o).all()


def torch_empty_like_words(imgs):
    import torch

    n, h, w = imgs.shape
    return torch.empty((n, h, -(-w // 32)), dtype=torch.int32, device=imgs.device)


def test_config_c3_full(cuda_dev):
    from paper_1401_5245_b200 import cuda as cu
    from paper_1401_5245_b200 import synth

    g = golden("configs.npz")
    c3 = synth.c3_words()
    out = _u32(cu.edges_packed(_t(c3.view(np.int32), cuda_dev), 8192, 1))
    assert hashlib.sha256(out.tobytes()).digest() == g["c3_out_sha256"].tobytes()
    # the same raster as the reference's native u64 words
    w64 = _t(P.u32_rows_to_u64(c3).view(np.int64), cuda_dev)
    o64 = _u64(cu.edges_packed(w64, 8192, 1))
    assert (P.u64_to_u32_rows(o64) == out).all()


@pytest.mark.slow
def test_config_c4_full(cuda_dev):
    """65536^2 (4 Gpx, 512 MiB packed): kernel vs the C per-pixel scanner, full size."""
    from paper_1401_5245_b200 import cuda as cu
    from paper_1401_5245_b200 import synth

    disks = synth.c4_disks()
    slab = synth.c4_slab(0, synth.C4_SIZE, disks, device=cuda_dev)
    out = cu.edges_packed(slab, synth.C4_SIZE, 1)
    host_in = _u32(slab)
    black = np.unpackbits(host_in[:2048].view(np.uint8)).mean()
    assert 0.7 < black < 0.9            # ~19% black in the sample
    exp = cscan.scan_p32(host_in, synth.C4_SIZE, 1)
    assert (_u32(out) == exp).all()
    # size-independent property: edges subset of figure (black out => black in)
    assert not (~_u32(out) & host_in).any()


@pytest.mark.slow
def test_config_c5_full(cuda_dev):
    """The WHOLE 1024 x 2048^2 batch (4 Gpx, 4 GiB uint8, fused pack + edges in
    one launch) vs the threaded C per-pixel scanner on every page, plus
    size-independent properties (edges subset of figure; mask method equals the
    per-pixel scan kernel; unfused pack -> K1 equals the fused kernel)."""
    import torch

    from paper_1401_5245_b200 import cuda as cu
    from paper_1401_5245_b200 import synth

    pages = synth.c5_pages(1024, device=cuda_dev)
    out = cu.pack_edges_u8(pages, 1)
    host = pages.cpu().numpy()
    black = 1.0 - host[:16].mean()
    assert 0.05 < black < 0.2            # ~10% black
    exp = cscan.scan_u8(host, 1)
    got = _u32(out)
    bad = np.nonzero((got != exp).any(axis=(1, 2)))[0]
    assert bad.size == 0, f"pages differing from the oracle: {bad[:16].tolist()}"
    del host, exp
    packed = cu.pack_u8(pages)
    assert torch.equal(cu.edges_packed(packed, 2048, 1), out)
    assert torch.equal(cu.scan_edges(packed, 2048, 1), out)
    assert int(((~out) & packed).count_nonzero()) == 0


@pytest.mark.slow
@pytest.mark.parametrize("knob", [{}, {"BITEDGE_NO_TMA": "1"}, {"BITEDGE_KERNEL": "tile"}],
                         ids=["default", "no_tma", "tile"])
def test_beyond_4gib_offsets(knob, cuda_dev, monkeypatch):
    """A uint8 raster of 4.4 GB (> 2^32 bytes, 2^32 pixels) and its packed form:
    64-bit offsets everywhere.  Oracle on bands at the start, across the 2^31
    and 2^32 byte marks and at the end (each band with its 1-row halos)."""
    import torch

    from paper_1401_5245_b200 import cuda as cu

    for k, v in knob.items():
        monkeypatch.setenv(k, v)
    h, w = 40000, 110016
    g = torch.Generator(device=cuda_dev).manual_seed(11)
    pix = (torch.rand((h, w), device=cuda_dev, generator=g) < 0.5).to(torch.uint8)
    out = cu.pack_edges_u8(pix, 1)
    packed = cu.pack_u8(pix)
    assert torch.equal(cu.edges_packed(packed, w, 1), out)
    for r in (0, (1 << 31) // w, (1 << 32) // w, h - 6):
        lo, hi = max(0, r - 1), min(h, r + 7)
        band = pix[lo:hi].cpu().numpy()[None]
        exp = cscan.scan_u8(band, 1)[0]
        got = _u32(out[lo:hi])
        # interior rows of the band (its first/last row saw the band border)
        a = 0 if lo == 0 else 1
        b = hi - lo if hi == h else hi - lo - 1
        assert (got[a:b] == exp[a:b]).all(), (knob, r)
    del pix, out, packed
    torch.cuda.empty_cache()


@pytest.mark.slow
@pytest.mark.parametrize("wb", [32, 64])
def test_beyond_4gib_packed(wb, cuda_dev):
    """A packed raster of 5.2 GB (40000 rows of 2^20 pixels) through K1."""
    import torch

    from paper_1401_5245_b200 import cuda as cu

    h, w = 40000, 1 << 20
    dt = torch.int32 if wb == 32 else torch.int64
    words = torch.randint(-2 ** 31, 2 ** 31 - 1, (h, w // 32), dtype=torch.int32,
                          device=cuda_dev, generator=torch.Generator(device=cuda_dev).manual_seed(5))
    inp = words if wb == 32 else words.view(torch.int64)
    out = cu.edges_packed(inp, w, 1)
    for r in (0, (1 << 31) // (w // 8), (1 << 32) // (w // 8), h - 6):
        lo, hi = max(0, r - 1), min(h, r + 7)
        band = words[lo:hi].cpu().numpy().view(np.uint32)
        o = out[lo:hi].cpu().numpy()
        if wb == 32:
            band_px, got = band, o.view(np.uint32)
        else:       # u64 words: pixel word p sits at u32 index p ^ 1
            band_px = P.u64_to_u32_rows(band.view(np.uint64))
            got = P.u64_to_u32_rows(o.view(np.uint64))
        exp = cscan.scan_p32(band_px, w, 1)
        a = 0 if lo == 0 else 1
        b = hi - lo if hi == h else hi - lo - 1
        assert (got[a:b] == exp[a:b]).all(), (wb, r)
    del words, inp, out
    torch.cuda.empty_cache()


# ---------------------------------------------------------------- row sharding (K3)

@pytest.mark.parametrize("W", [2048 + 96, 2048, 8192])   # ragged, and K1's tail-free (w % 256 == 0) kernels
@pytest.mark.parametrize("G", [2, 3, 4, 8])
@pytest.mark.parametrize("prs", ["", "4"])    # K1 strip height: size-chosen, or forced 4 rows
def test_row_slabs_with_halos_equal_whole(cuda_dev, G, W, prs, monkeypatch):
    import torch

    if prs:
        monkeypatch.setenv("BITEDGE_PRS", prs)

    from paper_1401_5245_b200 import cuda as cu

    rng = np.random.default_rng(G)
    H = 301
    a = (rng.random((H, W)) < 0.5).astype(np.uint8)
    whole = cu.pack_edges_u8(_t(a, cuda_dev), 1)
    pk = torch.from_numpy(P.pack_u32(a).view(np.int32)).to(cuda_dev)
    edges = np.linspace(0, H, G + 1).astype(int)
    for fill in (1, 0):
        whole = cu.pack_edges_u8(_t(a, cuda_dev), fill)
        parts = []
        for r in range(G):
            lo, hi = edges[r], edges[r + 1]
            slab = pk[lo:hi].clone()
            above = pk[lo - 1].clone() if lo > 0 else None
            below = pk[hi].clone() if hi < H else None
            out = torch.empty_like(slab)
            # interior first, then the two boundary rows (the overlapped schedule)
            if hi - lo > 2:
                cu.edges_halo(slab, None, None, W, fill, out=out, row_lo=1, row_hi=hi - lo - 1)
            cu.edges_halo(slab, above, below, W, fill, out=out, row_lo=0, row_hi=1)
            cu.edges_halo(slab, above, below, W, fill, out=out, row_lo=hi - lo - 1, row_hi=hi - lo)
            parts.append(out)
        assert torch.equal(torch.cat(parts), whole), (G, fill)


@pytest.mark.parametrize("W", [1, 31, 32, 33, 100, 1000, 8192, 65536])
@pytest.mark.parametrize("G", [2, 3, 8])
def test_row_slabs_halo_ends_kernel(cuda_dev, G, W):
    """RowShardedEdges' schedule: K3 on the interior rows [1, n-1), then K3e
    (rows 0 and n-1, one launch) with the received halos -- equal to the whole
    raster; K3e writes nothing but those two rows (sentinel), n = 1 and 2
    included."""
    import torch

    from paper_1401_5245_b200 import cuda as cu

    rng = np.random.default_rng(W + G)
    H = 2 * G + 3 if W > 8192 else 61
    a = (rng.random((H, W)) < 0.5).astype(np.uint8)
    pk = torch.from_numpy(P.pack_u32(a).view(np.int32)).to(cuda_dev)
    cuts = [0, 1, 3] + list(np.linspace(4, H, G - 1).astype(int)) if G >= 3 else [0, 1, H]
    cuts = sorted(set(int(c) for c in cuts))
    for fill in (1, 0):
        whole = cu.pack_edges_u8(_t(a, cuda_dev), fill)
        parts = []
        for r in range(len(cuts) - 1):
            lo, hi = cuts[r], cuts[r + 1]
            n = hi - lo
            slab = pk[lo:hi].clone()
            above = pk[lo - 1].clone() if lo > 0 else None
            below = pk[hi].clone() if hi < H else None
            out = torch.full_like(slab, 0x5A5A5A5A)
            cu.edges_halo_ends(slab, above, below, W, fill, out=out)
            if n > 2:
                assert (out[1:n - 1] == 0x5A5A5A5A).all(), "K3e wrote an interior row"
                cu.edges_halo(slab, None, None, W, fill, out=out, row_lo=1, row_hi=n - 1)
            parts.append(out)
        assert torch.equal(torch.cat(parts), whole), (G, W, fill, cuts)


@pytest.mark.parametrize("zc", [False, True, None])     # staged copies / kernel over host memory / auto
def test_host_pipeline_e2e(cuda_dev, zc):
    from paper_1401_5245_b200 import synth
    from paper_1401_5245_b200.host import HostBatchEdges

    imgs = synth.c2_images(512)
    pipe = HostBatchEdges(imgs.shape, kind="u8", chunk_images=100, zero_copy=zc)
    assert pipe.zero_copy == (zc is not False)
    hin, hout = pipe.new_host_buffers()
    hin.copy_(imgs)
    pipe(hin, hout)
    assert (hout.numpy().view(np.uint32) == cscan.scan_u8(imgs.numpy(), 1)).all()
    c3 = synth.c3_words(h=512)
    pipe2 = HostBatchEdges((1, 512, 256), kind="packed", width=8192, chunk_images=1, zero_copy=zc)
    import torch

    hin2 = torch.from_numpy(c3.view(np.int32)).reshape(1, 512, 256).pin_memory()
    out2 = pipe2(hin2)
    assert (out2.numpy().view(np.uint32)[0] == cscan.scan_p32(c3, 8192)).all()
    # pageable buffers always take the staged path (the kernel cannot map them)
    out3 = torch.empty(pipe.out_shape, dtype=torch.int32)
    pipe(imgs.clone(), out3)
    assert (out3.numpy().view(np.uint32) == cscan.scan_u8(imgs.numpy(), 1)).all()
    # ragged uint8 rows and a single C1-sized image, both border fills
    rng = np.random.default_rng(5)
    for (n, h, w) in ((1, 256, 256), (3, 37, 130), (1, 1, 1)):
        a = (rng.random((n, h, w)) < 0.5).astype(np.uint8) * 7
        for fill in (1, 0):
            p3 = HostBatchEdges((n, h, w), kind="u8", border=fill, zero_copy=zc)
            hi, ho = p3.new_host_buffers()
            hi.copy_(torch.from_numpy(a))
            got = p3.submit(hi, ho).synchronize().numpy().view(np.uint32)
            assert (got == cscan.scan_u8(a, fill)).all(), (n, h, w, fill, zc)


def test_host_pipeline_zero_copy_limits(cuda_dev):
    from paper_1401_5245_b200.host import HostBatchEdges

    assert not HostBatchEdges((4096, 64, 64), kind="u8").zero_copy          # 16 MiB: copy engines
    assert HostBatchEdges((1, 256, 256), kind="u8").zero_copy
    assert not HostBatchEdges((1, 64, 1024), kind="u8").zero_copy            # TMA kernels
    with pytest.raises(ValueError, match="zero_copy"):
        HostBatchEdges((1, 64, 2048), kind="u8", zero_copy=True)


@pytest.mark.parametrize("zc", [False, None])
def test_host_pipeline_submit(cuda_dev, zc):
    """HostBatchEdges.submit: several batches in flight over two host output
    buffers (the bench's e2e loop), each result exact when its handle syncs."""
    import torch

    from paper_1401_5245_b200 import synth
    from paper_1401_5245_b200.host import HostBatchEdges

    batches = [synth.c2_images(300, start=300 * k) for k in range(3)]   # distinct images
    pipe = HostBatchEdges(tuple(batches[0].shape), kind="u8", chunk_images=64, zero_copy=zc)
    hins = [torch.empty(tuple(b.shape), dtype=torch.uint8, pin_memory=True) for b in batches]
    for h_, b in zip(hins, batches):
        h_.copy_(b)
    houts = [torch.empty(pipe.out_shape, dtype=torch.int32, pin_memory=True) for _ in range(2)]
    pend = [None, None]
    for i in range(9):
        pend[i & 1] = pipe.submit(hins[i % 3], houts[i & 1])
        if i > 0:
            j = i - 1
            got = pend[j & 1].synchronize().numpy().view(np.uint32)
            assert (got == cscan.scan_u8(batches[j % 3].numpy(), 1)).all(), j
    got = pend[8 & 1].synchronize().numpy().view(np.uint32)
    assert (got == cscan.scan_u8(batches[8 % 3].numpy(), 1)).all()
    assert pend[0].query() and pend[1].query()


@pytest.mark.parametrize("kind", ["u8", "packed"])
@pytest.mark.parametrize("fill", [1, 0])
def test_host_pipeline_rows(kind, fill, cuda_dev):
    """A single host image chunked by rows (be_host_edges_rows): chunk sizes that
    do and do not divide the height, 1-row chunks, and the automatic choice."""
    import torch

    from paper_1401_5245_b200 import synth
    from paper_1401_5245_b200.host import HostBatchEdges

    rng = np.random.default_rng(fill + (kind == "u8"))
    for h, w in [(101, 2048), (37, 100), (64, 8192), (5, 33)]:
        a = (rng.random((1, h, w)) < 0.5).astype(np.uint8)
        exp = cscan.scan_u8(a, fill)
        if kind == "u8":
            host = torch.from_numpy(a * rng.integers(1, 256, a.shape).astype(np.uint8))
        else:
            host = torch.from_numpy(P.pack_u32(a).view(np.int32))
        for cr in (1, 7, 16, h, None):
            pipe = HostBatchEdges(tuple(host.shape), kind=kind, width=w, border=fill,
                                  chunk_rows=cr)
            hin, hout = pipe.new_host_buffers()
            hin.copy_(host)
            got = pipe(hin, hout).numpy().view(np.uint32)
            assert (got == exp).all(), (kind, fill, h, w, cr)
            assert pipe.rows_mode == (cr is not None)
    # row slabs of one raster with host halo rows (multi-GPU row shards)
    a = (rng.random((1, 90, 300)) < 0.5).astype(np.uint8)
    exp = cscan.scan_u8(a, fill)[0]
    full = torch.from_numpy(a * 7) if kind == "u8" else torch.from_numpy(P.pack_u32(a).view(np.int32))
    for lo, hi in [(0, 30), (30, 61), (61, 90), (0, 90), (45, 46)]:
        ha, hb = lo > 0, hi < 90
        pipe = HostBatchEdges((1, hi - lo, full.shape[2]), kind=kind, width=300, border=fill,
                              halo_rows=(ha, hb), chunk_rows=7)
        hin, hout = pipe.new_host_buffers()
        hin.copy_(full[:, lo - ha:hi + hb])
        got = pipe(hin, hout).numpy().view(np.uint32)[0]
        assert (got == exp[lo:hi]).all(), (kind, fill, lo, hi)
    big = synth.c3_words(h=4096)                                     # 4 MiB: automatic rows mode
    pipe = HostBatchEdges((1, 4096, 256), kind="packed", width=8192, border=fill)
    assert pipe.rows_mode
    hin = torch.from_numpy(big.view(np.int32)).reshape(1, 4096, 256).pin_memory()
    assert (pipe(hin).numpy().view(np.uint32)[0] == cscan.scan_p32(big, 8192, fill)).all()


def test_fill_policies_on_border_touching_figure(cuda_dev):
    """Interior invariance: pixels >= 2 from the border do not depend
    on the policy; border pixels do."""
    from paper_1401_5245_b200 import cuda as cu

    a = np.zeros((1, 20, 70), np.uint8)
    a[0, 5:9, 30:40] = 1
    t = _t(a, cuda_dev)
    w = P.unpack_u32(_u32(cu.pack_edges_u8(t, 1)), 70)[0]
    b = P.unpack_u32(_u32(cu.pack_edges_u8(t, 0)), 70)[0]
    assert (w[2:-2, 2:-2] == b[2:-2, 2:-2]).all()
    assert (w[0] == 0).all() and (b[0] == 1).all()


# ---------------------------------------------------------------- F2: threshold fused into the pack

@pytest.mark.parametrize("t", [0, 1, 2, 77, 127, 128, 129, 200, 255])
def test_threshold_edges_fused(cuda_dev, t):
    """binarize.threshold (sample >= t -> white) + edges in one
    kernel == threshold on the host followed by the oracle scan."""
    from paper_1401_5245_b200 import cuda as cu

    rng = np.random.default_rng(t)
    for (n, h, w) in [(3, 45, 2048), (2, 33, 100), (64, 64, 64), (1, 1, 7)]:
        g = rng.integers(0, 256, (n, h, w), dtype=np.uint8)
        binary = (g >= t).astype(np.uint8)
        exp = cscan.scan_u8(binary, 1)
        bo = torch_empty_like_words(_t(g, cuda_dev))
        got = _u32(cu.threshold_edges_u8(_t(g, cuda_dev), t, 1, binary_out=bo))
        assert (got == exp).all(), (t, n, h, w)
        assert (_u32(bo) == P.pack_u32(binary)).all(), (t, n, h, w)
        assert (_u32(cu.threshold_u8(_t(g, cuda_dev), t)) == P.pack_u32(binary)).all()


def test_threshold_spec_examples(cuda_dev):
    from paper_1401_5245_b200.binarize import threshold, threshold_edges
    from paper_1401_5245_b200.edge import detect_edges_mask

    g = np.array([[0, 127, 128, 255]], dtype=np.uint8)
    assert threshold(g, 128).to_array().tolist() == [[0, 0, 1, 1]]
    assert threshold(g, 0).to_array().tolist() == [[1, 1, 1, 1]]
    assert threshold(np.full((2, 3), 254, np.uint8), 255).count_black() == 6
    b, e = threshold_edges(g, 128)
    assert e == detect_edges_mask(b)


# ---------------------------------------------------------------- F1: PBM P4 at the kernel boundary

def test_pbm_spec_examples(cuda_dev):
    from paper_1401_5245_b200.pbm import read_pbm, write_pbm

    assert read_pbm(b"P1\n3 1\n1 0 1\n").to_array().tolist() == [[0, 1, 0]]
    assert read_pbm(b"P4\n3 1\n\xa0").to_array().tolist() == [[0, 1, 0]]
    f = b"P4\n3 1\n\xa0"
    assert write_pbm(read_pbm(f), raw=True) == f
    with pytest.raises(ValueError, match="offset"):
        read_pbm(b"P4\n16 2\n\x00\x00\x00")                                  # short payload


def test_pbm_roundtrip_and_detect(cuda_dev):
    """read∘write identity on random rasters (acceptance 8) and the
    fused P4 -> edges -> P4 path against the oracle, aligned and unaligned rows."""
    from paper_1401_5245_b200.bitimage import BitImage
    from paper_1401_5245_b200.pbm import detect_pbm, read_pbm, write_pbm

    rng = np.random.default_rng(4)
    for (h, w) in [(5, 3), (17, 100), (9, 128), (33, 1024), (3, 250), (64, 2048), (2, 8192), (7, 1),
                   (40, 96), (11, 8000), (6, 7993), (300, 32)]:
        a = (rng.random((h, w)) < 0.5).astype(np.uint8)
        img = BitImage.from_array(a)
        for raw in (True, False):
            data = write_pbm(img, raw)
            assert read_pbm(data) == img, (h, w, raw)
        p4 = write_pbm(img, True)
        exp = P.to_array(P.detect_edges_mask(P.from_array(a), 1))
        import os

        # default dispatch (K1 on 16-byte or 4-byte rows, else the byte kernel),
        # the byte kernel forced, and decode -> K1 -> encode
        from paper_1401_5245_b200 import _capi

        for knob in (None, "BITEDGE_P4_BYTES", "BITEDGE_P4_UNFUSED"):
            if knob:
                os.environ[knob] = "1"
                _capi.reload_knobs()
            try:
                got = read_pbm(detect_pbm(p4)).to_array()
            finally:
                if knob:
                    os.environ.pop(knob, None)
                    _capi.reload_knobs()
            assert (got == exp).all(), (h, w, knob)
        # P4 padding bits of the output are zero
        if w % 8:
            out = detect_pbm(p4)
            payload = np.frombuffer(out[-((w + 7) // 8) * h:], np.uint8).reshape(h, -1)
            assert not (payload[:, -1] & ((1 << (8 - w % 8)) - 1)).any()


# ---------------------------------------------------------------- extremes

def test_empty_batch_and_extreme_shapes(cuda_dev):
    """n = 0 is a no-op; one very long row, one very tall column and a wide
    3-row strip agree with the oracle (grid-size and tail handling)."""
    import torch

    from paper_1401_5245_b200 import cuda as cu

    empty = torch.zeros((0, 5, 40), dtype=torch.uint8, device=cuda_dev)
    assert cu.pack_edges_u8(empty).shape == (0, 5, 2)
    assert cu.edges_packed(torch.zeros((0, 5, 2), dtype=torch.int32, device=cuda_dev), 40).shape[0] == 0
    rng = np.random.default_rng(9)
    for (n, h, w) in [(1, 1, 1 << 20), (1, 1 << 18, 1), (1, 3, 100003), (2, 1 << 12, 33)]:
        a = (rng.random((n, h, w)) < 0.5).astype(np.uint8)
        exp = cscan.scan_u8(a, 1)
        assert (_u32(cu.pack_edges_u8(_t(a, cuda_dev), 1)) == exp).all(), (n, h, w)
        pk = _t(P.pack_u32(a).view(np.int32), cuda_dev)
        assert (_u32(cu.edges_packed(pk, w, 0)) == cscan.scan_u8(a, 0)).all(), (n, h, w)

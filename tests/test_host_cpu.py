"""CPU-only checks of the product's host side: the C-ABI library loads and
exports every symbol include/bitedge.h declares, argument validation maps to
the reference's exceptions without touching a GPU, the drop-in BitImage
mirrors the reference's constructor/enum/accessor semantics, and the
generators have the BASELINE shapes and densities."""

import ctypes

import numpy as np
import pytest

from paper_1401_5245_b200 import _capi
from paper_1401_5245_b200.bitimage import (BitImage, BorderPolicy, Direction, PixelColor,
                                           WORD_BITS)


def test_library_exports_every_header_symbol():
    lib = _capi.load()
    syms = _capi.header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) <= set(_capi._SIGNATURES), "ctypes signatures missing for some symbols"
    assert lib.be_abi_version() == 1


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("args,msg", [
    ((None, None, 1, 0, 5, 1, 1, 0, None), "at least 1x1"),
    ((None, None, 1, 5, 5, 1, 2, 0, None), "fill_bit"),
    ((ctypes.c_void_p(16), ctypes.c_void_p(32), 1, 5, 100, 1, 1, 0, None), "row stride"),
    ((None, None, 1, 5, 5, 1, 1, 0, None), "NULL"),
    ((None, None, 1 << 40, 1 << 40, 5, 1, 1, 0, None), "too large"),   # n * h would overflow
    ((None, None, 1, 5, 1 << 40, 1 << 35, 1, 0, None), "too large"),
])
def test_abi_validation_errors(args, msg):
    """Invalid arguments fail before any launch with a negative code -> ValueError."""
    lib = _capi.load()
    rc = lib.be_edge_packed_u32(*args)
    assert rc < 0
    assert msg in lib.be_last_error().decode()
    with pytest.raises(ValueError, match=msg):
        _capi.check(rc)


def test_abi_rejects_misaligned_and_bad_enums():
    lib = _capi.load()
    assert lib.be_shift(ctypes.c_void_p(8), ctypes.c_void_p(16), 32, 1, 1, 5, 1, 7, 1, None) < 0
    assert lib.be_bitop(9, ctypes.c_void_p(8), None, ctypes.c_void_p(16), 32, 1, 1, 5, 1, None) < 0
    assert lib.be_shift(ctypes.c_void_p(4), ctypes.c_void_p(16), 64, 1, 1, 5, 1, 0, 1, None) \
        == -2  # BE_EALIGN: 64-bit words need 8-byte alignment
    assert lib.be_edge_packed_u32(ctypes.c_void_p(16), ctypes.c_void_p(16), 1, 2, 32, 1, 1, 0,
                                  None) < 0  # output aliases input
    halo = lib.be_edges_general(ctypes.c_void_p(16), 0, 1, ctypes.c_void_p(32), None,
                                ctypes.byref(_capi.be_outputs(edges=64)), 32, 1, 2, 3, 32, 1, 0, 6,
                                None)
    assert halo < 0 and "single slab" in lib.be_last_error().decode()


def test_cuda_api_refuses_cpu_tensors():
    import torch

    from paper_1401_5245_b200 import cuda as cu

    with pytest.raises(ValueError, match="CUDA tensor"):
        cu.edges_packed(torch.zeros((4, 1), dtype=torch.int32), 32)
    with pytest.raises(ValueError, match="CUDA tensor"):
        cu.pack_edges_u8(torch.zeros((4, 8), dtype=torch.uint8))


# ---------------------------------------------------------------- drop-in BitImage (host side)

def test_enums_match_reference():
    assert PixelColor.BLACK == 0 and PixelColor.WHITE == 1
    assert Direction.LEFT.value == (-1, 0) and Direction.DOWN.dy == 1
    assert Direction.LEFT.opposite is Direction.RIGHT and Direction.UP.opposite is Direction.DOWN
    assert BorderPolicy.WHITE_OUTSIDE.fill_bit == 1
    assert BorderPolicy.BLACK_OUTSIDE.fill_color is PixelColor.BLACK
    assert WORD_BITS == 64


def test_constructor_errors_mirror_reference():
    w = np.zeros((2, 1), np.uint64)
    with pytest.raises(TypeError):
        BitImage(np.int64(3), 2, w)           # numpy ints rejected (bitimage.py:87-88)
    with pytest.raises(ValueError, match="at least 1x1"):
        BitImage(0, 2, w)
    with pytest.raises(ValueError, match="uint64 with shape"):
        BitImage(3, 2, np.zeros((2, 1), np.int64))
    with pytest.raises(ValueError, match="uint64 with shape"):
        BitImage(3, 2, np.zeros((2, 2), np.uint64))
    with pytest.raises(ValueError, match="at least 1x1"):
        BitImage.filled(0, 3, PixelColor.WHITE)
    with pytest.raises(ValueError, match="2-d"):
        BitImage.from_array(np.zeros(5, np.uint8))
    with pytest.raises(ValueError, match="at least 1x1"):
        BitImage.from_array(np.zeros((3, 0), np.uint8))


def test_constructor_forces_padding_and_freezes():
    w = np.zeros((2, 1), np.uint64)
    img = BitImage(3, 2, w)
    assert int(img.words[0, 0]) == (1 << 61) - 1
    assert not img.words.flags.writeable
    assert img.words is w                    # takes ownership, like the reference
    ro = np.zeros((1, 2), np.uint64)
    ro.setflags(write=False)
    img2 = BitImage(70, 1, ro)
    assert img2.words is not ro and int(img2.words[0, 1]) == (1 << 58) - 1


def test_get_set_host_semantics():
    img = BitImage.filled(3, 3, PixelColor.WHITE)
    b = img.set(1, 1, PixelColor.BLACK)
    assert b.get(1, 1) == PixelColor.BLACK and img.get(1, 1) == PixelColor.WHITE
    with pytest.raises(IndexError):
        img.get(3, 0)
    with pytest.raises(IndexError):
        img.set(0, -1, PixelColor.BLACK)
    assert b == b.set(1, 1, PixelColor.BLACK)
    assert b != img and hash(b) == hash(img.set(1, 1, PixelColor.BLACK))
    assert (img == 5) is False or (img.__eq__(5) is NotImplemented)
    assert img.__and__(3) is NotImplemented and img.__or__("x") is NotImplemented
    assert img.words_per_row == 1


def test_compute_ops_fail_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    img = BitImage.filled(3, 3, PixelColor.WHITE)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        img.invert()
    from paper_1401_5245_b200 import edge

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        edge.detect_edges_mask(img)


def test_shape_mismatch_message():
    a = BitImage.filled(3, 3, PixelColor.WHITE)
    b = BitImage.filled(4, 3, PixelColor.WHITE)
    with pytest.raises(ValueError, match="AND needs identical dimensions: 3x3 vs 4x3"):
        a & b
    with pytest.raises(ValueError, match="OR needs identical dimensions"):
        a | b


def test_drop_in_import_names():
    import bitedge.bitimage as bb
    import bitedge.edge as be

    assert bb.BitImage is BitImage
    for name in ("build_mask", "fundamental_edge", "detect_edges_mask", "edge_set",
                 "is_edge_point", "detect_edges_scan", "at_most_one_black_8neighbor"):
        assert callable(getattr(be, name))


def test_product_never_imports_oracle():
    import pathlib

    root = pathlib.Path(__file__).resolve().parents[1]
    for p in list((root / "paper_1401_5245_b200").rglob("*.py")) + list((root / "bitedge").rglob("*.py")):
        text = p.read_text()
        assert "import oracle" not in text and "from oracle" not in text, p


# ---------------------------------------------------------------- generators

def test_generators_shapes_and_density():
    from paper_1401_5245_b200 import synth

    c1 = synth.c1_image()
    assert c1.shape == (256, 256) and set(np.unique(c1)) <= {0, 1}
    assert 0.2 < 1 - c1.mean() < 0.6
    c2 = synth.c2_images(256).numpy()
    assert c2.shape == (256, 64, 64)
    assert 0.12 < 1 - c2.mean() < 0.19          # ~15% black
    assert (synth.c2_images(8, start=3).numpy() == c2[3:11]).all()   # per-image seeds
    c3 = synth.c3_words(h=64, w=8192)
    assert c3.dtype == np.uint32 and abs(np.unpackbits(c3.view(np.uint8)).mean() - 0.5) < 0.01
    pages = synth.c5_pages(2).numpy()
    assert pages.shape == (2, 2048, 2048)
    assert 0.07 < 1 - pages.mean() < 0.13       # ~10% black


def test_c4_slab_rasteriser_matches_bruteforce():
    import torch

    from paper_1401_5245_b200 import synth
    from oracle import port as P

    size = 512
    disks = synth.c4_disks(seed=9, size=size, n=60)
    yy, xx = np.mgrid[0:size, 0:size]
    ref = np.ones((size, size), np.uint8)
    for cx, cy, r in disks:
        ref[(xx - cx) ** 2 + (yy - cy) ** 2 <= r * r] = 0
    got = synth.c4_slab(0, size, disks, size=size, chunk_rows=100).numpy().view(np.uint32)
    assert (got == P.pack_u32(ref)).all()
    part = synth.c4_slab(100, 300, disks, size=size).numpy().view(np.uint32)
    assert (part == got[100:300]).all()


# ---------------------------------------------------------------- PBM header (F1 host side)

def test_pbm_header_parsing():
    from paper_1401_5245_b200.pbm import parse_header

    assert parse_header(b"P1\n3 1\n1 0 1\n") == ("P1", 3, 1, 7)
    assert parse_header(b"P4\n3 1\n\xa0") == ("P4", 3, 1, 7)
    assert parse_header(b"P4 # comment\n  12\t7\n") == ("P4", 12, 7, 20)
    with pytest.raises(ValueError, match="offset 0"):
        parse_header(b"P5\n1 1\n")
    with pytest.raises(ValueError, match="offset"):
        parse_header(b"P4\n3 \n")
    with pytest.raises(ValueError, match="at least 1x1"):
        parse_header(b"P4\n0 3\n")

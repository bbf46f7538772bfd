"""numpy restatement of the reference hot path -- TEST INFRASTRUCTURE ONLY.

Pinned against the real reference by `tests/golden/*.npz` (written by
`oracle/make_golden.py`, which imports `/root/reference/pkg/src/bitedge/
bitimage.py` by path).  See `oracle/__init__.py` for who may import this.

Representation (bitimage.py:1-11): a raster is (width, height, words) with
`words` a C-contiguous uint64 array of shape (height, ceil(width/64)); the MSB
of a word is its leftmost pixel; 1 = white, 0 = black; padding bits (pixel
positions >= width in the last word of each row) are 1 after every operation
(bitimage.py:101-104).

The edge composition below is SPEC.md's (the reference ships no `edge`
module): build_mask = NOT, fundamental_edge = shift(opposite
side) AND mask, detect_edges_mask = NOT(OR of four) (SPEC:165-
168).  It is deliberately op-for-op the reference's composition (13 full-
raster passes) so that timing it is timing the reference's CPU path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

WORD = 64
_U1 = np.uint64(1)
_U63 = np.uint64(63)
_TOP = np.uint64(1 << 63)
_FULL = np.uint64(0xFFFFFFFFFFFFFFFF)

# Direction values as (dx, dy), y grows downwards (bitimage.py:35-41).
LEFT, RIGHT, UP, DOWN = (-1, 0), (1, 0), (0, -1), (0, 1)
SIDES = (LEFT, RIGHT, UP, DOWN)
WHITE_OUTSIDE, BLACK_OUTSIDE = 1, 0          # BorderPolicy.fill_bit (bitimage.py:56-64)


def words_per_row(width: int) -> int:
    return -(-width // WORD)


def pad_mask(width: int) -> np.uint64:
    """Bits of the last row word that lie beyond pixel width-1 (bitimage.py:101-102)."""
    rem = width % WORD
    return np.uint64(0) if rem == 0 else np.uint64((1 << (WORD - rem)) - 1)


@dataclass(frozen=True)
class Raster:
    width: int
    height: int
    words: np.ndarray   # uint64 (height, words_per_row), padding normalised to 1

    def __eq__(self, other):  # word equality is pixel equality (bitimage.py:251-257)
        return (self.width, self.height) == (other.width, other.height) and bool(
            np.array_equal(self.words, other.words))

    __hash__ = None


def make(width: int, height: int, words: np.ndarray) -> Raster:
    """Normalise padding to 1 and freeze (bitimage.py:82-109)."""
    w = np.array(words, dtype=np.uint64, copy=True, order="C")
    assert w.shape == (height, words_per_row(width)), (w.shape, width, height)
    pm = pad_mask(width)
    if pm:
        w[:, -1] |= pm
    w.setflags(write=False)
    return Raster(width, height, w)


def from_array(a) -> Raster:
    """Pack: nonzero -> white(1), MSB-first, padded with 1s (bitimage.py:122-136)."""
    a = np.asarray(a)
    h, w = a.shape
    wp = words_per_row(w)
    bits = np.ones((h, wp * WORD), dtype=np.uint8)
    bits[:, :w] = a != 0
    by = np.packbits(bits, axis=1)                          # MSB-first within each byte
    words = by.view(">u8").astype(np.uint64)                 # 8 bytes big-endian -> one word
    return make(w, h, words)


def to_array(r: Raster) -> np.ndarray:
    """Unpack to uint8 bits (bitimage.py:149-153)."""
    by = r.words.astype(">u8").view(np.uint8).reshape(r.height, -1)
    return np.unpackbits(by, axis=1)[:, : r.width]


def filled(width: int, height: int, white: bool) -> Raster:
    fill = _FULL if white else np.uint64(0)
    return make(width, height, np.full((height, words_per_row(width)), fill, dtype=np.uint64))


# ---- word-parallel primitives ------------------------------------------------

def invert(r: Raster) -> Raster:                      # bitimage.py:181-183
    return make(r.width, r.height, ~r.words)


def and_(a: Raster, b: Raster) -> Raster:             # bitimage.py:195-199
    return make(a.width, a.height, a.words & b.words)


def or_(a: Raster, b: Raster) -> Raster:              # bitimage.py:201-205
    return make(a.width, a.height, a.words | b.words)


def shift(r: Raster, direction, fill: int = WHITE_OUTSIDE) -> Raster:
    """out(x, y) = in(x - dx, y - dy); outside pixels take `fill` (bitimage.py:207-240)."""
    src = r.words
    fw = _FULL if fill else np.uint64(0)
    if direction == DOWN:                  # row y <- row y-1, row 0 <- fill  (:216-219)
        out = np.vstack([np.full((1, src.shape[1]), fw, np.uint64), src[:-1]])
    elif direction == UP:                  # row y <- row y+1, last row <- fill (:220-223)
        out = np.vstack([src[1:], np.full((1, src.shape[1]), fw, np.uint64)])
    elif direction == RIGHT:               # pixel x <- pixel x-1, with word carry (:224-229)
        out = src >> _U1
        out[:, 1:] |= src[:, :-1] << _U63
        if fill:
            out[:, 0] |= _TOP
    elif direction == LEFT:                # pixel x <- pixel x+1; pixel W-1 <- fill (:230-239)
        out = src << _U1
        out[:, :-1] |= src[:, 1:] >> _U63
        last = _U1 << np.uint64(WORD - 1 - (r.width - 1) % WORD)
        if fill:
            out[:, -1] |= last
        else:
            out[:, -1] &= ~last
    else:
        raise ValueError(direction)
    return make(r.width, r.height, out)


def count_black(r: Raster) -> int:                     # bitimage.py:244-249
    ones = int(np.bitwise_count(r.words).sum(dtype=np.int64))
    pad = r.words.shape[1] * WORD - r.width
    return r.width * r.height - (ones - r.height * pad)


# ---- SPEC `edge` composition --------------------------------

def opposite(d):
    return (-d[0], -d[1])


def build_mask(img: Raster) -> Raster:
    return invert(img)


def fundamental_edge(img: Raster, mask: Raster, side, fill: int = WHITE_OUTSIDE) -> Raster:
    """shift(img, opposite(side)) AND mask; 1 marks black pixels whose `side`
    neighbour is white (side L -> shift RIGHT etc.)."""
    return and_(shift(img, opposite(side), fill), mask)


def edge_set(img: Raster, fill: int = WHITE_OUTSIDE) -> Raster:
    """Pre-inversion OR of the four fundamental edges."""
    mask = build_mask(img)
    e = [fundamental_edge(img, mask, s, fill) for s in SIDES]
    return or_(or_(or_(e[0], e[1]), e[2]), e[3])


def detect_edges_mask(img: Raster, fill: int = WHITE_OUTSIDE) -> Raster:
    """invert(OR of four fundamental edges); edges black on white."""
    return invert(edge_set(img, fill))


# ---- the paper's per-pixel scanner ----------------

def is_edge_point_bits(bits: np.ndarray, x: int, y: int, fill: int) -> bool:
    """Edge(p) = p' and (n2 or n4 or n6 or n8) on an unpacked uint8 raster."""
    h, w = bits.shape

    def px(xx, yy):
        return fill if not (0 <= xx < w and 0 <= yy < h) else int(bits[yy, xx])

    if px(x, y):
        return False
    return bool(px(x, y - 1) or px(x - 1, y) or px(x, y + 1) or px(x + 1, y))


def detect_edges_scan_loop(img: Raster, fill: int = WHITE_OUTSIDE) -> Raster:
    """Literal per-pixel scan; small rasters only (~2 us/px)."""
    bits = to_array(img)
    out = np.ones_like(bits)
    for y in range(img.height):
        for x in range(img.width):
            if is_edge_point_bits(bits, x, y, fill):
                out[y, x] = 0
    return from_array(out)


def edge_bits_vectorised(bits: np.ndarray, fill: int = WHITE_OUTSIDE) -> np.ndarray:
    """Independent vectorised Edge(p) over an unpacked raster (output 0 = edge)."""
    b = np.asarray(bits) != 0
    p = np.pad(b, 1, constant_values=bool(fill))
    any_white = p[:-2, 1:-1] | p[2:, 1:-1] | p[1:-1, :-2] | p[1:-1, 2:]
    edge = ~b & any_white
    return (~edge).astype(np.uint8)


def detect_edges_scan(img: Raster, fill: int = WHITE_OUTSIDE) -> Raster:
    return from_array(edge_bits_vectorised(to_array(img), fill))


# ---- layout conversions between the reference u64 words and BASELINE's u32 rows ----

def u64_to_u32_rows(words: np.ndarray) -> np.ndarray:
    """Native-u64 MSB-first words -> MSB-first uint32 row words."""
    return np.ascontiguousarray(words.astype(">u8").view(">u4").astype(np.uint32))


def u32_rows_to_u64(u32: np.ndarray) -> np.ndarray:
    """Inverse of u64_to_u32_rows; the u32 row length must be even."""
    u = np.ascontiguousarray(u32)
    return np.ascontiguousarray(u.astype(">u4").view(">u8").astype(np.uint64))


def u32_words_per_row(width: int) -> int:
    return -(-width // 32)


def u32_pad_mask(width: int) -> np.uint32:
    rem = width % 32
    return np.uint32(0) if rem == 0 else np.uint32((1 << (32 - rem)) - 1)


def pack_u32(a: np.ndarray) -> np.ndarray:
    """uint8 [.., H, W] (nonzero = white) -> uint32 [.., H, ceil(W/32)] MSB-first, pad = 1."""
    a = np.asarray(a)
    *lead, h, w = a.shape
    wp = u32_words_per_row(w)
    bits = np.ones((*lead, h, wp * 32), dtype=np.uint8)
    bits[..., :w] = a != 0
    by = np.packbits(bits, axis=-1)
    return np.ascontiguousarray(by.view(">u4").astype(np.uint32))


def unpack_u32(words: np.ndarray, width: int) -> np.ndarray:
    by = np.ascontiguousarray(words).astype(">u4").view(np.uint8)
    return np.unpackbits(by, axis=-1)[..., :width]


def edge_u32_rows(words: np.ndarray, width: int, fill: int = WHITE_OUTSIDE,
                  edgeset: bool = False) -> np.ndarray:
    """Mask-method output in BASELINE's u32 row format for one [H, Wp32] raster
    or a batch [N, H, Wp32], via the u64 composition above (odd Wp32 is padded
    to an even count with all-ones words, which are padding in u64 form)."""
    words = np.asarray(words, dtype=np.uint32)
    if words.ndim == 3:
        return np.stack([edge_u32_rows(x, width, fill, edgeset) for x in words])
    h, wp = words.shape
    ev = wp + (wp & 1)
    buf = np.full((h, ev), 0xFFFFFFFF, dtype=np.uint32)
    buf[:, :wp] = words
    img = make(width, h, u32_rows_to_u64(buf))
    res = edge_set(img, fill) if edgeset else detect_edges_mask(img, fill)
    out = u64_to_u32_rows(res.words)[:, :wp]
    return np.ascontiguousarray(out)

"""Drop-in `bitedge.edge`: the paper's method of masks on the B200.

The reference package names this module but does not ship
it; names, signatures, defaults and output conventions follow SPEC.md:

    build_mask(img)                              SPEC:147-155   PAPER sec. 3
    fundamental_edge(img, mask, side, border)    SPEC:156-164   PAPER sec. 4
    detect_edges_mask(img, border)               SPEC:165-173   PAPER sec. 5
    edge_set(img, border)                        SPEC:141-144, 212 (EdgeSet accessor)
    fundamental_edges(img, border)               all four sides + EdgeSet in one pass (F3)
    is_edge_point(img, x, y, border)             SPEC:174-182   PAPER sec. 1
    detect_edges_scan(img, border)               SPEC:183-191   PAPER sec. 1
    at_most_one_black_8neighbor(img, x, y, b)
    Neighborhood / neighborhood(img, x, y, b)    SPEC:137-140 (Fig. 1 numbering)

`detect_edges_mask` is ONE fused kernel (mask, four shifts, four ANDs, OR,
NOT) over the image's device words instead of the reference composition's
13 full-raster passes; `detect_edges_scan` is a separate per-pixel kernel
(the paper's "traditional scanning").  Edges are black (0) on white (1);
the default border is WHITE_OUTSIDE.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .bitimage import BitImage, BorderPolicy, Direction, PixelColor

_WHITE = BorderPolicy.WHITE_OUTSIDE


_CU = None


def _cuda():
    global _CU
    if _CU is None:
        from . import cuda

        _CU = cuda
    return _CU


def build_mask(img: BitImage) -> BitImage:
    """The negative image: mask bit 1 exactly at black pixels."""
    return img.invert()


def fundamental_edge(img: BitImage, mask: BitImage, side: Direction,
                     border: BorderPolicy = _WHITE) -> BitImage:
    """EdgeSet of black pixels whose `side` neighbour is white:
    and(shift(img, opposite(side), border), mask), as one fused
    shift+AND kernel.  Side Left -> shift Right, Right -> Left, Up -> Down,
    Down -> Up."""
    if not isinstance(mask, BitImage):
        raise TypeError("mask must be a BitImage")
    img._require_same_shape(mask, "AND")
    return BitImage._wrap(img.width, img.height,
                          _cuda().shift_and(img.device_words(), mask.device_words(), img.width,
                                            side.code, border.fill_bit))


def _edges(img: BitImage, border: BorderPolicy, edgeset: bool) -> BitImage:
    pix = img._take_pixels()
    if type(pix) is np.ndarray:
        # small host image, nothing uploaded yet: pack + edges in one kernel over
        # the thread's page-locked staging pair, words back, in one native call;
        # the result holds host words (uploaded on demand), the input keeps its
        # pixels (packed on demand)
        res = BitImage._wrap(img.width, img.height, None)
        res._words = _cuda().host_detect_small(pix, border.fill_bit, edgeset=edgeset)
        return res
    if pix is not None:
        # from_array of a larger host array, nothing uploaded yet: upload, pack +
        # edges (one launch) and the result's download in one native call; the
        # result holds its words on the host (and in HBM when the call staged them
        # there), the input keeps its packed words in HBM
        out, packed, host = _cuda().host_detect(pix.t, border.fill_bit, edgeset=edgeset)
        img._adopt_packed(packed)
        res = BitImage._wrap(img.width, img.height, out)   # out None: uploaded on demand
        res._words = host
        return res
    out = _cuda().edges_packed(img.device_words(), img.width, border.fill_bit, edgeset=edgeset)
    return BitImage._wrap(img.width, img.height, out)


def detect_edges_mask(img: BitImage, border: BorderPolicy = _WHITE) -> BitImage:
    """invert(OR of the four fundamental EdgeSets): edge pixels black (0), all
    others white (1), padding 1.  One kernel launch -- which
    also packs the image when it came from `from_array` of a host array and was
    not packed yet (then upload, kernel and the result's download are one call)."""
    return _edges(img, border, False)


def edge_set(img: BitImage, border: BorderPolicy = _WHITE) -> BitImage:
    """The pre-inversion marker raster: 1 = edge pixel."""
    return _edges(img, border, True)


def fundamental_edges(img: BitImage, border: BorderPolicy = _WHITE) -> dict:
    """All four fundamental EdgeSets plus their OR and the edge image from a
    single read of the image: {Direction: BitImage, 'edgeset': ..., 'edges': ...}."""
    res = _cuda().edges_general(img.device_words(), img.width, border.fill_bit, word_bits=64,
                                edges=True, edgeset=True, sides=True)
    out = {}
    for d, k in ((Direction.LEFT, "left"), (Direction.RIGHT, "right"), (Direction.UP, "up"),
                 (Direction.DOWN, "down")):
        out[d] = BitImage._wrap(img.width, img.height, res[k][0])
    out["edgeset"] = BitImage._wrap(img.width, img.height, res["edgeset"][0])
    out["edges"] = BitImage._wrap(img.width, img.height, res["edges"][0])
    return out


# ---- the paper's per-pixel definitions (sec. 1) ------------------------------

# Fig. 1 numbering: row above [3, 2, 1], middle [4, P, 8],
# row below [5, 6, 7]; index -> (dx, dy) with y growing downwards.
NEIGHBOR_OFFSETS = {1: (1, -1), 2: (0, -1), 3: (-1, -1), 4: (-1, 0),
                    5: (-1, 1), 6: (0, 1), 7: (1, 1), 8: (1, 0)}
FOUR_NEIGHBORS = (2, 4, 6, 8)


@dataclass(frozen=True)
class Neighborhood:
    """The 8 neighbour samples of a pixel, numbered per Fig. 1;
    out-of-raster neighbours are materialised via the border policy."""

    samples: tuple  # samples[i - 1] is neighbour i

    def __getitem__(self, i: int) -> PixelColor:
        if not 1 <= i <= 8:
            raise IndexError(f"neighbour index must be 1..8, got {i}")
        return self.samples[i - 1]


def neighborhood(img: BitImage, x: int, y: int, border: BorderPolicy = _WHITE) -> Neighborhood:
    img._check_coords(x, y)
    fill = border.fill_color
    s = []
    for i in range(1, 9):
        dx, dy = NEIGHBOR_OFFSETS[i]
        xx, yy = x + dx, y + dy
        inside = 0 <= xx < img.width and 0 <= yy < img.height
        s.append(img.get(xx, yy) if inside else fill)
    return Neighborhood(tuple(s))


def is_edge_point(img: BitImage, x: int, y: int, border: BorderPolicy = _WHITE) -> bool:
    """Edge(p) = (p)' and (2 or 4 or 6 or 8)."""
    img._check_coords(x, y)
    if img.get(x, y) == PixelColor.WHITE:
        return False
    nb = neighborhood(img, x, y, border)
    return any(nb[i] == PixelColor.WHITE for i in FOUR_NEIGHBORS)


def detect_edges_scan(img: BitImage, border: BorderPolicy = _WHITE) -> BitImage:
    """is_edge_point at every pixel, same output convention as
    detect_edges_mask; a per-pixel device kernel."""
    return BitImage._wrap(img.width, img.height,
                          _cuda().scan_edges(img.device_words(), img.width, border.fill_bit))


def at_most_one_black_8neighbor(img: BitImage, x: int, y: int,
                                border: BorderPolicy = _WHITE) -> bool:
    """True iff <= 1 of the 8 Fig. 1 neighbours is black;
    a property-check helper, not part of detection."""
    img._check_coords(x, y)
    if img.get(x, y) == PixelColor.WHITE:
        raise ValueError(f"pixel ({x}, {y}) is white; the helper is defined for black pixels")
    nb = neighborhood(img, x, y, border)
    return sum(1 for i in range(1, 9) if nb[i] == PixelColor.BLACK) <= 1

"""SPEC.md's invariants and properties, on the device through the drop-in API:
BitImage, edge and binarize.
Seeded random rasters across word boundaries, both border policies."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rasters(seed, count=24):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        h, w = int(rng.integers(1, 40)), int(rng.integers(1, 200))
        d = float(rng.choice([0.1, 0.5, 0.9]))
        out.append((rng.random((h, w)) >= d).astype(np.uint8))
    return out


def _pad_ok(img):
    from paper_1401_5245_b200.bitimage import WORD_BITS

    pad = img.words_per_row * WORD_BITS - img.width
    if pad == 0:
        return True
    mask = np.uint64((1 << pad) - 1)
    return bool((img.words[:, -1] & mask == mask).all())


def test_bitimage_properties(cuda_dev):
    from paper_1401_5245_b200.bitimage import BitImage, BorderPolicy, Direction

    for a in _rasters(1):
        img = BitImage.from_array(a)
        other = BitImage.from_array(np.random.default_rng(a.size).integers(0, 2, a.shape))
        h, w = a.shape
        ops = [img.invert(), img & other, img | other]
        for d in Direction:
            for b in BorderPolicy:
                s = img.shift(d, b)
                ops.append(s)
                # shift inverse on the interior
                back = s.shift(d.opposite, b).to_array()
                if h > 2 and w > 2:
                    assert (back[1:-1, 1:-1] == a[1:-1, 1:-1]).all(), (d, b)
        assert all(_pad_ok(x) for x in ops)                     # padding hygiene
        # De Morgan, commutativity, associativity, idempotence
        third = BitImage.from_array(np.random.default_rng(w).integers(0, 2, a.shape))
        assert ~(img | other) == (~img & ~other)
        assert (img & other) == (other & img) and (img | other) == (other | img)
        assert ((img & other) & third) == (img & (other & third))
        assert ((img | other) | third) == (img | (other | third))
        assert (img & img) == img and (img | img) == img
        assert ~~img == img


def test_edge_properties(cuda_dev):
    from paper_1401_5245_b200.bitimage import BitImage, BorderPolicy, Direction, PixelColor
    from paper_1401_5245_b200.edge import (at_most_one_black_8neighbor, build_mask,
                                           detect_edges_mask, detect_edges_scan, edge_set,
                                           fundamental_edge, is_edge_point)

    for k, a in enumerate(_rasters(2)):
        img = BitImage.from_array(a)
        h, w = a.shape
        for b in BorderPolicy:
            e = detect_edges_mask(img, b)
            assert e == detect_edges_scan(img, b)
            ea = e.to_array()
            assert not ((ea == 0) & (a == 1)).any()                     # edge ⊆ figure
            es = edge_set(img, b)
            assert es == ~e                                            # OR == invert(edges)
            mask = build_mask(img)
            for side in Direction:
                fe = fundamental_edge(img, mask, side, b)
                assert (fe | es) == es                                 # each ⊆ OR
            assert _pad_ok(e) and _pad_ok(es)
        ew = detect_edges_mask(img, BorderPolicy.WHITE_OUTSIDE).to_array()
        eb = detect_edges_mask(img, BorderPolicy.BLACK_OUTSIDE).to_array()
        if h > 4 and w > 4:
            assert (ew[2:-2, 2:-2] == eb[2:-2, 2:-2]).all()
        if k < 6:                                                      # subsumption
            for y in range(h):
                for x in range(w):
                    if img.get(x, y) == PixelColor.BLACK and at_most_one_black_8neighbor(img, x, y):
                        assert is_edge_point(img, x, y)


def test_thin_figure_fixed_point(cuda_dev):
    """One-pixel-wide strokes: every black pixel is an edge point, so
    detect_edges_mask(img) == img."""
    from paper_1401_5245_b200.bitimage import BitImage, BorderPolicy
    from paper_1401_5245_b200.edge import detect_edges_mask

    rng = np.random.default_rng(3)
    for it in range(12):
        h, w = int(rng.integers(3, 50)), int(rng.integers(3, 150))
        a = np.ones((h, w), np.uint8)
        rows = sorted(set(int(r) for r in rng.integers(0, h, 6)))
        for r in rows:
            if all(abs(r - q) >= 2 for q in rows if q != r):    # no two strokes touch
                lo = int(rng.integers(0, w))
                a[r, lo:int(rng.integers(lo, w)) + 1] = 0       # a horizontal run
        if it % 2:
            a = np.ascontiguousarray(a.T)                        # vertical strokes
        for b in BorderPolicy:
            img = BitImage.from_array(a)
            if b == BorderPolicy.BLACK_OUTSIDE and (a[0] == 0).any() | (a[-1] == 0).any() | \
                    (a[:, 0] == 0).any() | (a[:, -1] == 0).any():
                continue        # border-touching strokes are suppressed by BLACK_OUTSIDE
            assert detect_edges_mask(img, b) == img, (it, b)


def test_binarize_properties(cuda_dev):
    from paper_1401_5245_b200.binarize import otsu_threshold, threshold

    rng = np.random.default_rng(4)
    g = rng.integers(0, 256, (37, 101)).astype(np.uint8)
    prev = None
    for t in range(0, 257, 16):
        t = min(t, 255)
        black = threshold(g, t).to_array() == 0
        if prev is not None:
            assert not (prev & ~black).any()                 # monotone in t
        prev = black
    assert (threshold(g, 0).to_array() == 1).all()
    assert (threshold(np.full((5, 7), 254, np.uint8), 255).to_array() == 0).all()
    # Otsu attains the maximum between-class variance (exhaustive re-check)
    for img in (g, np.concatenate([np.full(50, 10), np.full(50, 200)]).astype(np.uint8)[None],
                np.array([[0, 255]], np.uint8), np.full((4, 4), 77, np.uint8)):
        t = otsu_threshold(img)
        x = img.reshape(-1).astype(np.float64)

        def var(t_):
            lo, hi = x[x < t_], x[x >= t_]
            if lo.size == 0 or hi.size == 0:
                return 0.0
            return lo.size * hi.size * (lo.mean() - hi.mean()) ** 2

        best = max(var(u) for u in range(256))
        assert abs(var(t) - best) <= 1e-9 * max(1.0, best), (t, var(t), best)
        if best > 0:
            assert t == min(u for u in range(256) if abs(var(u) - best) <= 1e-9 * best)
        else:
            assert t == 0


def _otsu_exact(img):
    """Brute force with exact rationals: the smallest t attaining the maximum
    between-class variance w0*w1*(mean0 - mean1)^2."""
    from fractions import Fraction

    x = [int(v) for v in np.asarray(img).reshape(-1)]
    best, arg = Fraction(0), 0
    for t in range(256):
        lo = [v for v in x if v < t]
        hi = [v for v in x if v >= t]
        if not lo or not hi:
            continue
        v = len(lo) * len(hi) * (Fraction(sum(lo), len(lo)) - Fraction(sum(hi), len(hi))) ** 2
        if v > best:
            best, arg = v, t
    return arg


def test_otsu_exact_ties(cuda_dev):
    """Exact tie-breaking (a float tolerance could pick a smaller,
    non-maximal t): symmetric histograms with exact ties, and random images."""
    from paper_1401_5245_b200.binarize import otsu_threshold

    rng = np.random.default_rng(11)
    cases = [np.array([[0, 255]], np.uint8),
             np.array([[10, 10, 200, 200]], np.uint8),
             np.array([[0, 100, 155, 255]], np.uint8),                 # symmetric: ties
             np.array([[3, 4, 250, 251, 3, 251]], np.uint8),
             np.full((3, 3), 0, np.uint8), np.full((3, 3), 255, np.uint8)]
    for _ in range(12):
        k = int(rng.integers(2, 6))
        vals = rng.choice(256, k, replace=False)
        cases.append(rng.choice(vals, (int(rng.integers(1, 40)), 3)).astype(np.uint8))
    for img in cases:
        assert otsu_threshold(img) == _otsu_exact(img), img.reshape(-1)[:12]

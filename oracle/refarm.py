"""The reference arm's CPU executor -- BENCH INFRASTRUCTURE ONLY (see oracle/__init__.py).

`bench.py --impl reference` and bench.py's `cpu_baseline` leg time the
reference's own CPU implementation of the path with this module:

* kind "reference": the UNMODIFIED reference `bitedge/bitimage.py`, installed
  by `pip install --target baseline/_ref /root/reference/pkg` (DESIGN.md
  section 8; `baseline/_ref` is git-ignored but travels to the GPU box), loaded
  by file path -- this repository's own `bitedge` package would shadow it --
  with SPEC.md's `edge` composition built from its primitives, exactly as
  oracle/make_golden.py builds the golden vectors:

      build_mask(img)                = img.invert()
      fundamental_edge(img, m, side) = img.shift(side.opposite) & m
      detect_edges_mask(img)         = ~(eL | eR | eU | eD)

* kind "port": oracle/port.py (the same composition restated on numpy, pinned
  to the reference by tests/golden) when baseline/_ref is absent.

Work is split into independent UNITS (whole images, or row bands of one raster
with a 1-row overlap on each side whose output rows are discarded) that worker
processes generate once and then recompute every step.
"""

from __future__ import annotations

import importlib.util
import os
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(_HERE)
REF_BITIMAGE = os.path.join(ROOT, "baseline", "_ref", "bitedge", "bitimage.py")

_impl = None


class _Ref:
    """SPEC's edge composition over the reference BitImage (bitimage.py:181-240)."""

    kind = "reference"

    def __init__(self, mod):
        self.R = mod
        D = mod.Direction
        self.sides = (D.LEFT, D.RIGHT, D.UP, D.DOWN)
        self.white = mod.BorderPolicy.WHITE_OUTSIDE

    def detect(self, img):
        m = img.invert()
        e = [img.shift(s.opposite, self.white) & m for s in self.sides]
        return ~(e[0] | e[1] | e[2] | e[3])

    def from_array(self, a):
        return self.R.BitImage.from_array(a)                       # bitimage.py:122-136

    def from_words(self, width, height, words_u64):
        return self.R.BitImage(width, height, words_u64)           # bitimage.py:82-109


class _Port:
    kind = "port"

    def __init__(self):
        from oracle import port

        self.P = port

    def detect(self, img):
        return self.P.detect_edges_mask(img, 1)

    def from_array(self, a):
        return self.P.from_array(a)

    def from_words(self, width, height, words_u64):
        return self.P.make(width, height, words_u64)


def impl():
    """The reference (baseline/_ref) when installed, else the port."""
    global _impl
    if _impl is None:
        if os.path.exists(REF_BITIMAGE) and not os.environ.get("BITEDGE_REFARM_PORT"):
            spec = importlib.util.spec_from_file_location("_ref_bitimage", REF_BITIMAGE)
            mod = importlib.util.module_from_spec(spec)
            sys.modules["_ref_bitimage"] = mod
            spec.loader.exec_module(mod)
            _impl = _Ref(mod)
        else:
            _impl = _Port()
    return _impl


def describe() -> str:
    k = impl().kind
    if k == "reference":
        return ("unmodified reference bitimage.py from baseline/_ref (pip install --target) "
                "+ SPEC.md:147-168 edge composition")
    return "oracle/port.py (numpy restatement of the reference BitImage composition)"


# ----------------------------------------------------------------------------- units

def units(cfg: str, n: int, h: int, w: int, target_px: int = 1 << 24, min_units: int = 1):
    """Independent work units covering the WHOLE config: ("img", i0, i1) image
    ranges or ("rows", lo, hi) row bands of one raster; at most `target_px`
    pixels per unit and, where the config divides, at least `min_units` units."""
    per_img = h * w
    if n > 1 or per_img <= target_px:
        k = max(1, min(n, target_px // per_img, -(-n // max(1, min_units))))
        return [("img", i, min(n, i + k)) for i in range(0, n, k)]
    rows = max(2, min(target_px // w, -(-h // max(1, min_units))))
    return [("rows", r, min(h, r + rows)) for r in range(0, h, rows)]


def make_unit(cfg: str, unit, h: int, w: int):
    """Generate one unit's input (untimed) in the form the reference consumes:
    ("u8", [H, W] arrays) or ("packed", (BitImage of the band, drop_top, keep))."""
    import torch

    from paper_1401_5245_b200 import synth

    kind, a, b = unit
    if cfg == "c1":
        return ("u8", [synth.c1_image()])
    if cfg == "c2":
        return ("u8", list(synth.c2_images(b - a, start=a).numpy()))
    if cfg == "c5":
        return ("u8", list(synth.c5_pages(b - a, start=a).numpy()))
    if cfg == "c3":
        full = synth.c3_words()
        lo, hi = max(0, a - 1), min(h, b + 1)
        u32 = full[lo:hi]
    elif cfg == "c4":
        lo, hi = max(0, a - 1), min(h, b + 1)
        u32 = synth.c4_slab(lo, hi, synth.c4_disks(), device="cpu").numpy().view(np.uint32)
    else:
        raise ValueError(cfg)
    del torch
    # u32 row words -> the reference's native u64 words, wrapped in its BitImage
    # once (neither is timed: SURVEY 8(d) starts C3/C4 from a uint64 BitImage)
    u64 = np.ascontiguousarray(np.ascontiguousarray(u32).astype(">u4").view(">u8")
                               .astype(np.uint64))
    return ("packed", (impl().from_words(w, hi - lo, u64), a - lo, b - a))


def run_unit(data) -> int:
    """One unit of the reference CPU path; returns a word of the result so the
    work cannot be skipped."""
    R = impl()
    kind, payload = data
    if kind == "u8":
        acc = 0
        for a in payload:
            acc ^= int(R.detect(R.from_array(a)).words[0, 0])     # from_array + detect
        return acc
    img, top, keep = payload
    out = R.detect(img).words[top:top + keep]
    return int(out[0, 0])

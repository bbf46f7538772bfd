"""Generate tests/golden/*.npz from the REAL reference -- TEST INFRASTRUCTURE ONLY.

Runs in the build container only (it reads /root/reference, which does not
exist on the GPU box).  It loads `/root/reference/pkg/src/bitedge/bitimage.py`
by file path (a package named `bitedge` in this repo would shadow it;
SURVEY.md 0.3 item 9) and composes SPEC.md's `edge` functions from the
reference's own BitImage primitives:

    build_mask(img)                  = img.invert()
    fundamental_edge(img, m, side)   = img.shift(side.opposite) & m
    edge_set(img)                    = eL | eR | eU | eD
    detect_edges_mask(img)           = ~edge_set(img)

Usage:  python oracle/make_golden.py      (rewrites tests/golden/)
"""

from __future__ import annotations

import hashlib
import importlib.util
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src/bitedge/bitimage.py"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "tests", "golden")


def load_reference():
    spec = importlib.util.spec_from_file_location("_ref_bitimage", REF)
    mod = importlib.util.module_from_spec(spec)
    sys.modules["_ref_bitimage"] = mod
    spec.loader.exec_module(mod)
    return mod


R = load_reference()
BI, D, BP = R.BitImage, R.Direction, R.BorderPolicy
SIDES = (D.LEFT, D.RIGHT, D.UP, D.DOWN)
POLICIES = (BP.WHITE_OUTSIDE, BP.BLACK_OUTSIDE)


def fundamental(img, mask, side, border):
    return img.shift(side.opposite, border) & mask


def edge_set(img, border):
    m = img.invert()
    e = [fundamental(img, m, s, border) for s in SIDES]
    return e[0] | e[1] | e[2] | e[3]


def detect(img, border):
    return ~edge_set(img, border)


def bits_index(arr: np.ndarray) -> int:
    v = 0
    for i, b in enumerate(arr.reshape(-1)):
        v |= int(b) << i
    return v


def exhaustive(n: int):
    """All 2^(n*n) n x n rasters; image i has pixel (x, y) = bit (y*n + x) of i.
    Returns visible output bits in the same encoding, per policy."""
    total = 1 << (n * n)
    idx = np.arange(total, dtype=np.int64)
    shifts = np.arange(n * n, dtype=np.int64)
    imgs = ((idx[:, None] >> shifts[None, :]) & 1).astype(np.uint8).reshape(total, n, n)
    res = {}
    for pol in POLICIES:
        outs = np.empty(total, dtype=np.uint16)
        eset = np.empty(total, dtype=np.uint16)
        for i in range(total):
            img = BI.from_array(imgs[i])
            o = detect(img, pol).to_array()
            e = edge_set(img, pol).to_array()
            outs[i] = bits_index(o)
            eset[i] = bits_index(e)
        res[pol.name] = (outs, eset)
    return res


def concat_words(imgs):
    words = np.concatenate([im.words.reshape(-1) for im in imgs]) if imgs else np.zeros(0, np.uint64)
    return words


def random_set(seed=1401, count=1000):
    """>=1000 seeded rasters, h, w in 1..64, densities {0.1, 0.5, 0.9},
    plus ragged larger shapes; inputs may hold any nonzero byte for white."""
    rng = np.random.default_rng(seed)
    shapes, arrays = [], []
    for i in range(count):
        h, w = int(rng.integers(1, 65)), int(rng.integers(1, 65))
        dens = (0.1, 0.5, 0.9)[i % 3]
        black = rng.random((h, w)) < dens
        vals = rng.integers(1, 256, (h, w)).astype(np.uint8)    # any nonzero = white
        arrays.append(np.where(black, 0, vals).astype(np.uint8))
        shapes.append((h, w))
    for h, w in [(1, 1), (1, 500), (500, 1), (7, 130), (199, 200), (3, 192), (64, 65), (33, 127)]:
        black = rng.random((h, w)) < 0.4
        arrays.append(np.where(black, 0, 1).astype(np.uint8))
        shapes.append((h, w))
    return shapes, arrays


def main():
    os.makedirs(OUT, exist_ok=True)

    # 1. exhaustive 3x3 / 4x4 (SPEC acceptance 1a/1b)
    ex = {}
    for n in (3, 4):
        r = exhaustive(n)
        for pol, (o, e) in r.items():
            ex[f"out{n}_{pol}"] = o
            ex[f"eset{n}_{pol}"] = e
    np.savez_compressed(os.path.join(OUT, "exhaustive.npz"), **ex)

    # 2. random + ragged corpus: inputs (uint8 flattened), reference words out
    shapes, arrays = random_set()
    data = {"shapes": np.array(shapes, dtype=np.int64),
            "pixels": np.concatenate([a.reshape(-1) for a in arrays])}
    imgs = [BI.from_array(a) for a in arrays]
    data["packed"] = concat_words(imgs)                          # from_array pin (A3)
    for pol in POLICIES:
        data[f"out_{pol.name}"] = concat_words([detect(im, pol) for im in imgs])
        data[f"eset_{pol.name}"] = concat_words([edge_set(im, pol) for im in imgs])
        for s in SIDES:
            m = [im.invert() for im in imgs]
            data[f"fund_{s.name}_{pol.name}"] = concat_words(
                [fundamental(im, mm, s, pol) for im, mm in zip(imgs, m)])
    np.savez_compressed(os.path.join(OUT, "random.npz"), **data)

    # 3. shifts at every bit alignment: widths 1..192, heights 1..3 (SPEC acceptance 3)
    rng = np.random.default_rng(444)
    sh_shapes, sh_pix = [], []
    for w in range(1, 193):
        for h in (1, 2, 3):
            sh_shapes.append((h, w))
            sh_pix.append((rng.random((h, w)) < 0.5).astype(np.uint8))
    simgs = [BI.from_array(a) for a in sh_pix]
    sd = {"shapes": np.array(sh_shapes, dtype=np.int64),
          "pixels": np.concatenate([a.reshape(-1) for a in sh_pix])}
    for d in SIDES:
        for pol in POLICIES:
            sd[f"shift_{d.name}_{pol.name}"] = concat_words([im.shift(d, pol) for im in simgs])
    sd["invert"] = concat_words([~im for im in simgs])
    # binary ops between consecutive images of equal shape (rows i, i+1 share no shape; use self-rotations)
    sd["and_rot"] = concat_words([im & im.shift(D.RIGHT) for im in simgs])
    sd["or_rot"] = concat_words([im | im.shift(D.DOWN, BP.BLACK_OUTSIDE) for im in simgs])
    sd["count_black"] = np.array([im.count_black() for im in simgs], dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "shift.npz"), **sd)

    # 4. BASELINE config C1 in full, C2 / C3 pinned by digest (the generators are in-repo)
    sys.path.insert(0, ROOT)
    from paper_1401_5245_b200 import synth
    c1 = synth.c1_image()
    img = BI.from_array(c1)
    cfg = {"c1_input_packed": img.words,
           "c1_out_WHITE_OUTSIDE": detect(img, BP.WHITE_OUTSIDE).words,
           "c1_out_BLACK_OUTSIDE": detect(img, BP.BLACK_OUTSIDE).words,
           "c1_eset_WHITE_OUTSIDE": edge_set(img, BP.WHITE_OUTSIDE).words}
    c3 = synth.c3_words()
    c3_img = BI(8192, 8192, c3.astype(">u4").view(">u8").astype(np.uint64))
    c3_out = detect(c3_img, BP.WHITE_OUTSIDE)
    c3_u32 = c3_out.words.astype(">u8").view(">u4").astype(np.uint32)
    cfg["c3_out_sha256"] = np.frombuffer(hashlib.sha256(c3_u32.tobytes()).digest(), np.uint8)
    cfg["c3_out_count_black"] = np.int64(c3_out.count_black())
    cfg["c3_in_sha256"] = np.frombuffer(hashlib.sha256(c3.tobytes()).digest(), np.uint8)
    n2 = 4096
    c2 = synth.c2_images(n2).numpy()
    h2 = hashlib.sha256()
    hin = hashlib.sha256(c2.tobytes())
    blacks = 0
    for i in range(n2):
        o = detect(BI.from_array(c2[i]), BP.WHITE_OUTSIDE)
        h2.update(o.words.astype(">u8").view(">u4").astype(np.uint32).tobytes())
        blacks += o.count_black()
    cfg["c2_in_sha256"] = np.frombuffer(hin.digest(), np.uint8)
    cfg["c2_out_sha256"] = np.frombuffer(h2.digest(), np.uint8)
    cfg["c2_out_count_black"] = np.int64(blacks)
    # the first 8 glyphs in full, for readable diffs
    cfg["c2_head_out"] = np.stack([detect(BI.from_array(c2[i]), BP.WHITE_OUTSIDE).words
                                   for i in range(8)])
    np.savez_compressed(os.path.join(OUT, "configs.npz"), **cfg)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()

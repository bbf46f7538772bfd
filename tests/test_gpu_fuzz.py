"""Seeded fuzzing of the whole dispatch surface against the per-pixel C oracle:
random batch shapes (including 1-pixel rows/columns), row-stride padding,
byte offsets that break alignment, border policy, threshold, uint8 / packed
u32 / packed u64 / P4 inputs and every kernel-selection knob.  Bit-exact."""

import os

import numpy as np
import pytest

from oracle import cscan
from oracle import port as P

pytestmark = pytest.mark.gpu

KNOBS = [{}, {"BITEDGE_KERNEL": "tile"}, {"BITEDGE_KERNEL": "stream"}, {"BITEDGE_CW4": "1"},
         {"BITEDGE_NO_ROLL": "1"}, {"BITEDGE_NO_WARPIMG": "1"}, {"BITEDGE_FORCE_TMA": "1"},
         {"BITEDGE_FORCE_TMA": "1", "BITEDGE_TMA1": "1"}, {"BITEDGE_PDL": "0"},
         {"BITEDGE_RS": "8"}, {"BITEDGE_WARPIMG_G4": "1"}, {"BITEDGE_PDL_LATE": "1"},
         {"BITEDGE_FORCE_TMA": "1", "BITEDGE_TMA2_RSL32": "1"}, {"BITEDGE_FORCE_TMA": "1", "BITEDGE_TMA2_RSL": "5"}, {"BITEDGE_FORCE_TMA": "1", "BITEDGE_TMA2_RSL": "11"}, {"BITEDGE_K1_GENERIC": "1"}, {"BITEDGE_NO_UNAL": "1"}, {"BITEDGE_UNAL_CHUNKS": "1"}, {"BITEDGE_UNAL_BYTES": "1"}, {"BITEDGE_U64_TMA": "1"}]


def _shape(rng):
    kind = rng.integers(0, 5)
    if kind == 0:
        return int(rng.integers(1, 9)), int(rng.integers(1, 70)), int(rng.integers(1, 200))
    if kind == 1:
        return int(rng.integers(1, 40)), 64, 64
    if kind == 2:
        return 1, int(rng.integers(1, 130)), int(rng.choice([1024, 1056, 2048, 2080, 4096, 3000]))
    if kind == 3:
        return int(rng.integers(1, 4)), int(rng.integers(1, 5)), int(rng.integers(1, 9000))
    return int(rng.integers(1, 300)), 1, int(rng.integers(1, 70))


@pytest.mark.parametrize("seed", range(12))
def test_fuzz(seed, cuda_dev, monkeypatch):
    import torch

    from paper_1401_5245_b200 import cuda as cu

    rng = np.random.default_rng(1000 + seed)
    for knob in KNOBS:
        for k, v in knob.items():
            monkeypatch.setenv(k, v)
        for _ in range(3):
            n, h, w = _shape(rng)
            fill = int(rng.integers(0, 2))
            t = int(rng.choice([1, 1, 1, 0, 2, 100, 128, 255]))
            g = rng.integers(0, 256, (n, h, w)).astype(np.uint8)
            g[rng.random((n, h, w)) < 0.4] = 0
            binary = (g >= t).astype(np.uint8)
            exp = cscan.scan_u8(binary, fill)
            # uint8 input, padded row stride and a byte offset that may break alignment
            pad, off = int(rng.integers(0, 40)), int(rng.integers(0, 3))
            buf = torch.zeros(n * h * (w + pad) + off + 64, dtype=torch.uint8, device=cuda_dev)
            view = buf[off:off + n * h * (w + pad)].view(n, h, w + pad)[..., :w]
            view.copy_(torch.from_numpy(g).to(cuda_dev))
            got = cu.threshold_edges_u8(view, t, fill).cpu().numpy().view(np.uint32)
            assert (got == exp).all(), (knob, n, h, w, pad, off, fill, t)
            # packed u32 with stride padding; packed u64 through the drop-in layout
            pk = P.pack_u32(binary)
            spad = int(rng.integers(0, 6))
            wb = torch.full((n, h, pk.shape[2] + spad), -1, dtype=torch.int32, device=cuda_dev)
            wb[..., : pk.shape[2]] = torch.from_numpy(pk.view(np.int32)).to(cuda_dev)
            got32 = cu.edges_packed(wb[..., : pk.shape[2]], w, fill).cpu().numpy().view(np.uint32)
            assert (got32 == exp).all(), (knob, n, h, w, spad, "u32")
            w64 = np.stack([P.from_array(x).words for x in binary]).view(np.int64)
            o64 = cu.edges_packed(torch.from_numpy(w64).to(cuda_dev), w, fill)
            e64 = np.stack([P.detect_edges_mask(P.from_array(x), fill).words for x in binary])
            assert (o64.cpu().numpy().view(np.uint64) == e64).all(), (knob, n, h, w, "u64")
        for k in knob:
            monkeypatch.delenv(k, raising=False)


@pytest.mark.parametrize("knob", [None, "BITEDGE_P4_BYTES", "BITEDGE_P4_UNFUSED",
                                  "BITEDGE_P4_NO_FLAT"])
@pytest.mark.parametrize("seed", range(4))
def test_fuzz_p4(seed, knob, cuda_dev, monkeypatch):
    import torch

    from paper_1401_5245_b200 import pbm

    if knob:
        monkeypatch.setenv(knob, "1")
    rng = np.random.default_rng(2000 + seed)
    for _ in range(8):
        n = int(rng.integers(1, 4))
        h = int(rng.integers(1, 50))
        w = int(rng.choice([int(rng.integers(1, 300)), 128, 1024, 2040, 4096, 96, 8000,
                            32 * int(rng.integers(1, 40)) - int(rng.integers(0, 8))]))
        fill = int(rng.integers(0, 2))
        a = (rng.random((n, h, w)) < 0.5).astype(np.uint8)
        rb = (w + 7) // 8
        bits = rng.integers(0, 2, (n, h, rb * 8)).astype(np.uint8)   # garbage padding bits
        bits[..., :w] = a
        payload = np.packbits(1 - bits, axis=-1)                     # P4: 1 = black
        out = pbm.detect_p4(torch.from_numpy(payload.reshape(-1).copy()).to(cuda_dev), n, h, w,
                            fill).cpu().numpy().reshape(n, h, rb)
        got = 1 - np.unpackbits(out, axis=-1)[..., :w]
        exp = P.unpack_u32(cscan.scan_u8(a, fill), w)
        assert (got == exp).all(), (n, h, w, fill)
        if w % 8:
            assert not (out[..., -1] & ((1 << (8 - w % 8)) - 1)).any()


@pytest.mark.parametrize("knob", KNOBS, ids=lambda k: ",".join(f"{a}={b}" for a, b in k.items()) or "default")
def test_fuzz_halo_slabs_all_inputs(knob, cuda_dev, monkeypatch):
    """Row slabs with halo rows through be_edges_general for uint8 pixels, u32
    words and u64 words: slab results concatenated == whole-image oracle."""
    import torch

    from paper_1401_5245_b200 import cuda as cu

    for k, v in knob.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(len(knob) * 7 + 1)
    for (H, W) in [(41, 2048), (23, 100), (37, 4096), (9, 64)]:
        a = (rng.random((H, W)) < 0.5).astype(np.uint8) * rng.integers(1, 256, (H, W)).astype(np.uint8)
        exp = cscan.scan_u8(a, 1)
        cuts = sorted({0, H, *rng.integers(1, H, 3).tolist()})
        views = {
            "u8": (torch.from_numpy(a).to(cuda_dev), 32),
            "u8_to_u64": (torch.from_numpy(a).to(cuda_dev), 64),
            "u32": (torch.from_numpy(P.pack_u32(a).view(np.int32)).to(cuda_dev), 32),
            "u64": (torch.from_numpy(P.from_array(a).words.view(np.int64).copy()).to(cuda_dev), 64),
        }
        img = P.from_array(a)
        mask = P.build_mask(img)
        exp_all = {"edges": exp}
        for k, d in (("left", P.LEFT), ("right", P.RIGHT), ("up", P.UP), ("down", P.DOWN)):
            exp_all[k] = P.u64_to_u32_rows(P.fundamental_edge(img, mask, d, 1).words)[:, : -(-W // 32)]
        for name, (full, wb) in views.items():
            parts = {k: [] for k in exp_all}
            for lo, hi in zip(cuts[:-1], cuts[1:]):
                slab = full[lo:hi].clone()
                above = full[lo - 1].clone() if lo > 0 else None
                below = full[hi].clone() if hi < H else None
                res = cu.edges_general(slab.unsqueeze(0), W, 1, word_bits=wb, above=above,
                                       below=below, sides=True)
                for k in parts:
                    parts[k].append(res[k][0])
            for k, ex in exp_all.items():
                got = torch.cat(parts[k]).cpu().numpy()
                if wb == 64:
                    got = P.u64_to_u32_rows(got.view(np.uint64))[:, : -(-W // 32)]
                else:
                    got = got.view(np.uint32)
                assert (got == ex).all(), (knob, name, k, H, W, cuts)


@pytest.mark.parametrize("w", [25, 31, 33, 57, 100, 127, 129, 250, 255, 257, 1000, 1001, 2047,
                               4100, 8001, 32002,
                               539, 544, 1180, 1216, 8000, 31993, 32032])   # rows of whole words: K1f P4
def test_p4_flat_widths(w, cuda_dev, monkeypatch):
    """K1p (P4 payloads viewed as one flat byte array) for every row-length
    phase mod 16 bytes, and K1f's P4 variant for rows of whole 4-byte words that
    are not vector multiples; batches whose images start mid-word, h = 1 / 2 /
    many, both borders -- against the oracle and against the byte kernel."""
    import torch

    from paper_1401_5245_b200 import pbm

    rng = np.random.default_rng(w)
    rb = (w + 7) // 8
    for n, h in ((1, 1), (1, 2), (3, 7), (2, 40)) if w < 8000 else ((1, 3), (2, 9)):
        a = (rng.random((n, h, w)) < 0.5).astype(np.uint8)
        bits = rng.integers(0, 2, (n, h, rb * 8)).astype(np.uint8)   # garbage padding bits
        bits[..., :w] = a
        payload = torch.from_numpy(np.packbits(1 - bits, axis=-1).reshape(-1).copy()).to(cuda_dev)
        for fill in (1, 0):
            out = pbm.detect_p4(payload, n, h, w, fill).cpu().numpy().reshape(n, h, rb)
            got = 1 - np.unpackbits(out, axis=-1)[..., :w]
            exp = P.unpack_u32(cscan.scan_u8(a, fill), w)
            assert (got == exp).all(), (n, h, w, fill)
            if w % 8:
                assert not (out[..., -1] & ((1 << (8 - w % 8)) - 1)).any()
            monkeypatch.setenv("BITEDGE_P4_BYTES", "1")
            ref = pbm.detect_p4(payload, n, h, w, fill).cpu().numpy().reshape(n, h, rb)
            monkeypatch.delenv("BITEDGE_P4_BYTES")
            assert (ref == out).all(), (n, h, w, fill)
            # 16- / 32-byte chunks by knob, and 16 because a buffer is only 16-byte aligned
            for kn in ("BITEDGE_P4_FLAT16", "BITEDGE_P4_FLAT32"):
                monkeypatch.setenv(kn, "1")
                ok = pbm.detect_p4(payload, n, h, w, fill).cpu().numpy().reshape(n, h, rb)
                monkeypatch.delenv(kn)
                assert (ref == ok).all(), (n, h, w, fill, kn)
            nb = payload.numel()
            src = torch.zeros(nb + 48, dtype=torch.uint8, device=cuda_dev)
            dst = torch.full((nb + 48,), 0xA5, dtype=torch.uint8, device=cuda_dev)
            src[16:16 + nb] = payload
            pbm.detect_p4(src[16:16 + nb], n, h, w, fill, out=dst[16:16 + nb])
            assert (dst[16:16 + nb].cpu().numpy().reshape(n, h, rb) == ref).all(), (n, h, w, fill, "+16")
            assert (dst[:16] == 0xA5).all() and (dst[16 + nb:] == 0xA5).all(), (n, h, w, "guard")

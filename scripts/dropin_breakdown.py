"""Where the drop-in API's per-call time goes for a small image (256^2):
each piece timed alone with a device sync, median of reps (wall clock)."""

import statistics
import sys
import time
import os

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def med_us(fn, reps=300):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e6)
    return statistics.median(ts)


def main():
    import ctypes

    import torch

    from paper_1401_5245_b200 import _capi
    from paper_1401_5245_b200 import cuda as cu
    from paper_1401_5245_b200.bitimage import BitImage
    from paper_1401_5245_b200.cli import generate
    from paper_1401_5245_b200.edge import detect_edges_mask

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    a = generate("glyph", n, 0.5)
    dev = torch.device("cuda:0")
    img = BitImage.from_array(a)
    dw = img.device_words()
    out = torch.empty_like(dw)
    t8 = torch.from_numpy(a).to(dev)
    lib = _capi.load()
    s = torch.cuda.current_stream().cuda_stream
    sync = torch.cuda.synchronize
    rows = {
        "sync (idle)": lambda: sync(),
        "current_stream()": lambda: torch.cuda.current_stream().cuda_stream,
        "torch.empty_like": lambda: torch.empty_like(dw),
        "raw ctypes K1 + sync": lambda: (lib.be_edge_packed_u64(ctypes.c_void_p(dw.data_ptr()), ctypes.c_void_p(out.data_ptr()), 1, n, n, dw.shape[1], 1, 0, ctypes.c_void_p(s)), sync()),
        "raw ctypes K1 x10 (no sync) /10": None,
        "cu.edges_packed + sync": lambda: (cu.edges_packed(dw, n, 1), sync()),
        "detect_edges_mask(dev img) + sync": lambda: (detect_edges_mask(img), sync()),
        "np->dev .to(dev) (pageable)": lambda: torch.from_numpy(a).to(dev),
        "cu.pack_u8 + sync": lambda: (cu.pack_u8(t8, word_bits=64), sync()),
        "BitImage.from_array(np)": lambda: BitImage.from_array(a),
        "dev->host .cpu() 8KB": lambda: dw.cpu(),
        "full host flow": lambda: detect_edges_mask(BitImage.from_array(a)).words,
    }

    def ten():
        for _ in range(10):
            lib.be_edge_packed_u64(ctypes.c_void_p(dw.data_ptr()), ctypes.c_void_p(out.data_ptr()), 1, n, n, dw.shape[1], 1, 0, ctypes.c_void_p(s))
        sync()
    for k, fn in rows.items():
        if fn is None:
            print(f"{k:40s} {med_us(ten, 100) / 10:8.1f} us")
        else:
            print(f"{k:40s} {med_us(fn):8.1f} us")


if __name__ == "__main__":
    main()

"""Fused pack + edges on uint8 pixels across row lengths (16-byte multiples go to
K2 / K2r / K2t2, others to the tile kernel): kernel time per step by CUDA-graph
replay over a rotating pool > 3x L2, 3 streams and serial; u32 and u64 output."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_5245_b200 import cuda as cu  # noqa: E402

dev = torch.device("cuda:0")


sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from u8_widths_lib import timed  # noqa: E402


for (n, h, w) in ((1, 16384, 16384), (1, 16384, 16100), (1, 16384, 16001), (1, 4096, 4096), (1, 4096, 4100), (1, 4096, 4000), (16, 1024, 1024), (16, 1024, 1000),
                  (64, 256, 256), (64, 256, 250)):
    nbytes = n * h * w
    pool = max(2, min(48, (3 * 126 << 20) // nbytes + 1))
    ins = [torch.randint(0, 2, (n, h, w), dtype=torch.uint8, device=dev) for _ in range(pool)]
    for wb in (32, 64, "pack"):
        def step(i):
            if wb == 32:
                cu.pack_edges_u8(ins[i % pool], 1)
            elif wb == 64:
                cu.pack_and_edges(ins[i % pool], 1, word_bits=64)
            else:
                cu.pack_u8(ins[i % pool], word_bits=64)
        k = pool * max(1, 96 // pool)
        us3, us1 = timed(step, k, 3), timed(step, k, 1)
        alg = nbytes * 1.125 if wb != 64 else nbytes * 1.25
        print(f"u8->{wb} {n}x{h}x{w}: {us3:7.2f} us ({alg / us3 / 1e3 / 6540.5:.3f}), serial {us1:7.2f} us "
              f"({alg / us1 / 1e3 / 6540.5:.3f})", flush=True)

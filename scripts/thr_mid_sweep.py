"""Thresholded (F2) fused pack + edges on mid-size grayscale rasters under dispatch
knobs given on the command line (K=V,K=V ...): protocol of u8_widths.py."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_1401_5245_b200 import _capi  # noqa: E402
from paper_1401_5245_b200 import cuda as cu  # noqa: E402
from u8_widths_lib import timed  # noqa: E402

dev = torch.device("cuda:0")
KNOBS = [{}]
for a in sys.argv[1:]:
    KNOBS.append(dict(kv.split("=") for kv in a.split(",")))
for (n, h, w) in ((1, 4096, 4096), (1, 5000, 5008), (1, 8192, 8192), (1, 12288, 12288), (64, 1080, 1920), (256, 480, 640)):
    nbytes = n * h * w
    pool = max(2, min(48, (3 * 126 << 20) // nbytes + 1))
    ins = [torch.randint(0, 256, (n, h, w), dtype=torch.uint8, device=dev) for _ in range(pool)]
    for kn in KNOBS:
        for k_, v_ in kn.items():
            os.environ[k_] = v_
        _capi.reload_knobs()

        def step(i):
            cu.threshold_edges_u8(ins[i % pool], 128, 1)
        k = pool * max(1, 96 // pool)
        us3, us1 = timed(step, k, 3), timed(step, k, 1)
        alg = nbytes * 1.125
        print(f"t=128 {n}x{h}x{w} {','.join(f'{a[8:]}={b}' for a, b in kn.items()) or 'default':28s}: {us3:7.2f} us "
              f"({alg / us3 / 1e3 / 6540.5:.3f}), serial {us1:7.2f} us ({alg / us1 / 1e3 / 6540.5:.3f})", flush=True)
        for k_ in kn:
            os.environ.pop(k_, None)

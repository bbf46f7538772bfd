"""Batches of small / medium uint8 images (between C2's 64^2 glyphs and C5's 2048^2
pages): which kernel owns them and how close to the copy peak.  Protocol of
u8_widths.py."""
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
SHAPES = ((16384, 64, 64), (4096, 128, 128), (1024, 256, 256), (256, 512, 512), (64, 1024, 1024),
          (1024, 256, 250), (1024, 200, 320), (256, 480, 640), (64, 1080, 1920), (16, 2048, 2048))
if os.environ.get("U8B_SHAPES"):       # e.g. U8B_SHAPES=64x1080x1920,32x1200x1600
    SHAPES = tuple(tuple(int(v) for v in t.split("x")) for t in os.environ["U8B_SHAPES"].split(","))
for (n, h, w) in SHAPES:
    nbytes = n * h * w
    pool = max(2, min(48, (3 * 126 << 20) // nbytes + 1))
    ins = [torch.randint(0, 2, (n, h, w), dtype=torch.uint8, device=dev) for _ in range(pool)]
    outs = [torch.empty((n, h, (w + 31) // 32), dtype=torch.int32, device=dev) for _ in range(pool)]
    for kn in KNOBS:
        for k_, v_ in kn.items():
            os.environ[k_] = v_
        _capi.reload_knobs()

        def step(i):
            cu.pack_edges_u8(ins[i % pool], 1, out=outs[i % pool])
        k = pool * max(1, 96 // pool)
        us3, us1 = timed(step, k, 3), timed(step, k, 1)
        alg = nbytes * 1.125
        print(f"{n}x{h}x{w} {','.join(f'{a[8:]}={b}' for a, b in kn.items()) or 'default':24s}: {us3:7.2f} us "
              f"({alg / us3 / 1e3 / 6540.5:.3f}), serial {us1:7.2f} us ({alg / us1 / 1e3 / 6540.5:.3f})", flush=True)
        for k_ in kn:
            os.environ.pop(k_, None)

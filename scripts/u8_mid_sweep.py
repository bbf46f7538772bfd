"""Mid-size uint8 rasters (4-64 MB) under the K2-family dispatch knobs: which
kernel should own them?  Same protocol as u8_widths.py."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_5245_b200 import _capi  # noqa: E402
from paper_1401_5245_b200 import cuda as cu  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from u8_widths_lib import timed  # noqa: E402

dev = torch.device("cuda:0")
KNOBS = [{}, {"BITEDGE_NO_TMA": "1"}] + [{"BITEDGE_TMA2_MIN": "0", "BITEDGE_TMA2_RSL": str(r)} for r in (4, 5, 6, 8, 10, 12, 16, 24)]
if len(sys.argv) > 1 and sys.argv[1] == "final":    # the dispatch as shipped against K2 alone
    KNOBS = [{}, {"BITEDGE_NO_TMA": "1"}]
for (n, h, w) in ((1, 4096, 4096), (4, 2048, 2048), (1, 3000, 5008), (1, 5000, 5008), (1, 6000, 6016), (1, 6000, 8000), (1, 8192, 8192),
                  (1, 12288, 12288), (1, 16384, 16384), (1, 8192, 8100)):
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
        print(f"{n}x{h}x{w} {','.join(f'{a[8:]}={b}' for a, b in kn.items()) or 'default':28s}: {us3:7.2f} us ({alg / us3 / 1e3 / 6540.5:.3f}), serial {us1:7.2f} us "
              f"({alg / us1 / 1e3 / 6540.5:.3f})", flush=True)
        for k_ in kn:
            os.environ.pop(k_, None)

"""Per-phase host time of the staged small-image flow (BITEDGE_TRACE_STAGED=1
prints memcpy_in / launch / sync / memcpy_out averages from the library), and
the wall time per call, for C2- / C1-sized and larger images; plus the floor of
any launch + stream sync on this box."""
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1401_5245_b200 import cuda as cu, synth  # noqa: E402
from paper_1401_5245_b200.cli import generate  # noqa: E402

tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("BITEDGE_"))
for name, a in (("64x64", synth.c2_images(1).numpy()[0]), ("256x256", synth.c1_image()),
                ("512x512", generate("glyph", 512, 0.5))):
    for _ in range(2000):
        cu.host_detect_small(a, 1)
    ts = []
    for _ in range(2000):
        t = time.perf_counter()
        cu.host_detect_small(a, 1)
        ts.append(time.perf_counter() - t)
    print(f"{tag} {name} host_detect_small median {statistics.median(ts) * 1e6:.2f} us", flush=True)
x = torch.zeros((1, 1), dtype=torch.int32, device="cuda")
o = torch.empty_like(x)
f = cu._capi.fn("be_edge_packed_u32")
s = torch.cuda.current_stream().cuda_stream
ts = []
for i in range(3000):
    t = time.perf_counter()
    f(x.data_ptr(), o.data_ptr(), 1, 1, 32, 1, 1, 0, s)
    torch.cuda.current_stream().synchronize()
    ts.append(time.perf_counter() - t)
print(f"{tag} floor: tiny device kernel launch + stream sync {statistics.median(ts) * 1e6:.2f} us")

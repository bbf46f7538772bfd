"""C2 e2e stability: ten consecutive 119-step windows of the bench's pipelined
host loop in one process (is a slow e2e transient or per-process?)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1401_5245_b200 import synth  # noqa: E402
from paper_1401_5245_b200.host import HostBatchEdges  # noqa: E402

imgs = synth.c2_images(4096)
pipe = HostBatchEdges(tuple(imgs.shape), kind="u8")
hin, hout = pipe.new_host_buffers()
hin.copy_(imgs)
houts = [hout, torch.empty_like(hout, pin_memory=True)]
pend = [None, None]
rates = []
for win in range(10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(119):
        pend[i & 1] = pipe.submit(hin, houts[i & 1])
        if i > 0:
            _ = int(pend[(i - 1) & 1].synchronize()[0, 0, 0])
    _ = int(pend[118 & 1].synchronize()[0, 0, 0])
    dt = (time.perf_counter() - t0) / 119
    rates.append(round(4096 * 4096 / dt / 1e9, 1))
print("Gpx/s per window:", rates)

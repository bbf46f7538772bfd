"""Row-chunk size sweep of the single-image host path (be_host_edges_rows) for
C3 (8 MiB packed) and C4 (512 MiB packed): ms per step, pipelined submits."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1401_5245_b200 import synth  # noqa: E402
from paper_1401_5245_b200.host import HostBatchEdges  # noqa: E402


def sweep(host, h, width, chunks, steps):
    for cr in chunks:
        pipe = HostBatchEdges(tuple(host.shape), kind="packed", width=width, chunk_rows=cr,
                              lanes=int(os.environ.get("LANES", "2")))
        hin, hout = pipe.new_host_buffers()
        hin.copy_(host)
        houts = [hout, torch.empty_like(hout, pin_memory=True)]
        pend = [None, None]

        def run(n):
            for i in range(n):
                pend[i & 1] = pipe.submit(hin, houts[i & 1])
                if i > 0:
                    _ = int(pend[(i - 1) & 1].synchronize()[0, 0, 0])
            _ = int(pend[(n - 1) & 1].synchronize()[0, 0, 0])
        run(max(3, steps // 5))
        t = time.perf_counter()
        run(steps)
        dt = (time.perf_counter() - t) / steps
        print(h, cr, pipe.chunk, f"{dt * 1e3:.4f} ms", f"{h * width / dt / 1e9:.1f} Gpx/s", flush=True)


w = synth.c3_words()
sweep(torch.from_numpy(w.view(np.int32)).reshape(1, 8192, 256), 8192, 8192,
      (1024, 2048, 4096, 8192, None), 1000)
slab = synth.c4_slab(0, 65536, synth.c4_disks(), device="cuda").cpu().unsqueeze(0)
if not os.environ.get("C3_ONLY"):
    sweep(slab, 65536, 65536, (1024, 2048, 4096, 8192, 16384, None), 20)

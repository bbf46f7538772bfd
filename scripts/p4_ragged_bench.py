"""F1 on rows that are not 16-byte multiples: the byte-granular single-pass P4
kernel against the 3-pass reference path (decode -> K1 -> encode), kernel-only
time per step (CUDA events over back-to-back launches, input > L2 rotating)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_5245_b200 import _capi  # noqa: E402
from paper_1401_5245_b200 import pbm  # noqa: E402

dev = torch.device("cuda:0")
for (h, w) in ((32000, 32000), (32000, 31993), (32000, 32002), (16000, 16002), (12000, 12002), (8000, 8001), (8000, 8000), (8000, 7993), (2000, 2000), (256, 250)):
    rb = (w + 7) // 8
    nbytes = h * rb
    pool = max(2, min(32, (3 * 126 << 20) // (2 * nbytes) + 1))
    ins = [torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=dev) for _ in range(pool)]
    outs = [torch.empty_like(x) for x in ins]
    res = {}
    for mode in ("fused", "unfused"):
        if mode == "unfused":
            os.environ["BITEDGE_P4_UNFUSED"] = "1"
        else:
            os.environ.pop("BITEDGE_P4_UNFUSED", None)
        _capi.reload_knobs()                       # knobs are read once per process
        for i in range(3):
            pbm.detect_p4(ins[i % pool], 1, h, w, out=outs[i % pool])
        torch.cuda.synchronize()
        k = pool * max(1, 200 // pool)
        g = torch.cuda.CUDAGraph()                 # replay: no per-call host overhead
        with torch.cuda.graph(g):
            for i in range(k):
                pbm.detect_p4(ins[i % pool], 1, h, w, out=outs[i % pool])
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / k
        res[mode] = outs[0].clone()
        print(f"{h}x{w} (row {rb} B) {mode:8s} {us:9.2f} us/step  {h * w / us / 1e3:9.1f} Gpx/s  "
              f"{2 * nbytes / us / 1e3:8.1f} GB/s", flush=True)
    os.environ.pop("BITEDGE_P4_UNFUSED", None)
    print("   fused == unfused:", bool(torch.equal(res["fused"], res["unfused"])), flush=True)

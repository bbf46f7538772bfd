"""K1p (flat P4 kernel, 32- / 16-byte chunks) against the byte kernel on
byte-granular P4 rows: kernel-only time per step (graph replay, input > L2
rotating).  Usage: p4_flat_bench.py [out.txt]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_5245_b200 import _capi  # noqa: E402
from paper_1401_5245_b200 import pbm  # noqa: E402

dev = torch.device("cuda:0")
MODES = (("default", {}), ("K1p 32 B", {"BITEDGE_P4_FLAT32": "1"}), ("K1p 16 B", {"BITEDGE_P4_FLAT16": "1"}), ("no flat", {"BITEDGE_P4_NO_FLAT": "1"}), ("byte kernel", {"BITEDGE_P4_BYTES": "1"}))
peak = 6540.0
lines = []
for (h, w) in ((32000, 32002), (32000, 31993), (8000, 8000), (8000, 7993), (16000, 16002), (12000, 12002), (8000, 8001),
               (4000, 4001), (2000, 2000), (1000, 1001), (256, 250)):
    rb = (w + 7) // 8
    nbytes = h * rb
    pool = max(2, min(32, (3 * 126 << 20) // (2 * nbytes) + 1))
    ins = [torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=dev) for _ in range(pool)]
    outs = [torch.empty_like(x) for x in ins]
    row = f"{h}x{w} (row {rb} B)"
    ref = None
    for name, env in MODES:
        for k_, v_ in env.items():
            os.environ[k_] = v_
        _capi.reload_knobs()
        for i in range(3):
            pbm.detect_p4(ins[i % pool], 1, h, w, out=outs[i % pool])
        torch.cuda.synchronize()
        k = pool * max(1, 200 // pool)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(k):
                pbm.detect_p4(ins[i % pool], 1, h, w, out=outs[i % pool])
        g.replay()
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) * 1e3 / k)
        got = outs[0].clone()
        if ref is None:
            ref = got
        same = bool(torch.equal(ref, got))
        row += f" | {name} {best:8.2f} us {2 * nbytes / best / 1e3:7.1f} GB/s ({2 * nbytes / best / 1e3 / peak:.2f}){'' if same else ' MISMATCH'}"
        for k_ in env:
            os.environ.pop(k_, None)
    print(row, flush=True)
    lines.append(row)
if len(sys.argv) > 1:
    open(sys.argv[1], "w").write("\n".join(lines) + "\n")

"""C4 row-shard strong scaling, modelled on one GPU with the SAME per-iteration
protocol bench.py uses at N > 1 (device spacer, CUDA events around each
iteration, one iteration at a time) and the NCCL path's schedule
(RowShardedEdges.step): K3 on the interior rows [1, n-1) on the compute stream
while K3e computes rows 0 and n-1 on a side stream with the halo rows (here
local buffers standing in for the rows NCCL delivers), then the join.  T(1) is
the N = 1 bench protocol (K back-to-back steps on one stream).  What a G-GPU
run adds on top -- the NCCL send/recv latency when it exceeds the interior
kernel, and the max over ranks -- only a real multi-GPU run can show.

    python scripts/c4_shard_model.py [out.txt]
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_5245_b200 import cuda as cu  # noqa: E402

dev = torch.device("cuda:0")
W, H = 65536, 65536
wp = W // 32
SPACER = 1_000_000
lines = []


def out(s):
    print(s, flush=True)
    lines.append(s)


def rnd(*shape):
    return torch.randint(-2**31, 2**31 - 1, shape, dtype=torch.int64, device=dev).to(torch.int32)


# T(1): the bench's N = 1 protocol, 20 back-to-back steps on one stream; and the
# same per-iteration protocol as N > 1 for comparison
full, full_o = rnd(H, wp), torch.empty(H, wp, dtype=torch.int32, device=dev)
for _ in range(5):
    cu.edges_packed(full, W, 1, out=full_o)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(SPACER)
a.record()
for _ in range(20):
    cu.edges_packed(full, W, 1, out=full_o)
b.record()
torch.cuda.synchronize()
t1 = a.elapsed_time(b) * 1e3 / 20
ts1 = []
for _ in range(30):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(SPACER)
    a.record()
    cu.edges_packed(full, W, 1, out=full_o)
    b.record()
    torch.cuda.synchronize()
    ts1.append(a.elapsed_time(b) * 1e3)
t1_iter = statistics.median(ts1)
del full, full_o
torch.cuda.empty_cache()
out(f"T(1) = {t1:.2f} us per step (N = 1 bench protocol: 20 back-to-back steps); "
    f"{t1_iter:.2f} us per single iteration (the N > 1 protocol)")

side = torch.cuda.Stream(dev)
above, below = rnd(wp), rnd(wp)
for G in (2, 4, 8):
    rows = H // G
    slab, o = rnd(rows, wp), torch.empty(rows, wp, dtype=torch.int32, device=dev)

    done = torch.cuda.Event()                 # an already-completed event on another stream
    with torch.cuda.stream(side):              # (stands in for the NCCL receive)
        done.record()

    def side_ends():                           # RowShardedEdges.step (default schedule)
        cur = torch.cuda.current_stream(dev)
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            cu.edges_halo_ends(slab, above, below, W, 1, out=o)      # rows 0 and n-1
        cu.edges_halo(slab, None, None, W, 1, out=o, row_lo=1, row_hi=rows - 1)
        cur.wait_stream(side)

    def serial_ends():                         # interior, wait for the halos, then K3e
        cu.edges_halo(slab, None, None, W, 1, out=o, row_lo=1, row_hi=rows - 1)
        torch.cuda.current_stream(dev).wait_event(done)
        cu.edges_halo_ends(slab, above, below, W, 1, out=o)

    def serial_ends_nowait():
        cu.edges_halo(slab, None, None, W, 1, out=o, row_lo=1, row_hi=rows - 1)
        cu.edges_halo_ends(slab, above, below, W, 1, out=o)

    def one_kernel():                          # K3 over the whole slab (p2p halos)
        cu.edges_halo(slab, above, below, W, 1, out=o)

    def interior_only():
        cu.edges_halo(slab, None, None, W, 1, out=o, row_lo=1, row_hi=rows - 1)

    for name, iteration in (("side-stream K3e (default)", side_ends),
                            ("K3e after interior + event wait", serial_ends),
                            ("K3e after interior", serial_ends_nowait),
                            ("one K3 kernel (p2p)", one_kernel),
                            ("interior only", interior_only)):
        for _ in range(5):
            iteration()
        torch.cuda.synchronize()
        ts = []
        for _ in range(30):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(SPACER)
            e0.record()
            iteration()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        tg = statistics.median(ts)
        out(f"G={G}: slab {rows} rows, {name:32s} {tg:7.2f} us per iteration (median of 30); "
            f"modelled efficiency T(1)/(G*T(G)) = {t1 / (G * tg):.3f}")
    del slab, o
    torch.cuda.empty_cache()
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        f.write("\n".join(lines) + "\n")

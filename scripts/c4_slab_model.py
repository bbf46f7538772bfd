"""C4 row-shard strong scaling, modelled on one GPU: the per-rank step at G ranks
is one K3 launch over a 65536/G-row slab whose halo rows come from neighbour
buffers (here local buffers standing in for the peers' HBM).  Times each slab
size (graph replay, 3 streams and serial, rotating slabs > 3x L2) and prints
the efficiency T(1) / (G * T(G)) that a G-GPU run would see if the NVLink halo
reads cost nothing extra.  Not a multi-GPU measurement."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_5245_b200 import cuda as cu  # noqa: E402

dev = torch.device("cuda:0")
W, H = 65536, 65536
wp = W // 32


def timed(step, k, nstreams):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cur = torch.cuda.current_stream()
        side = [torch.cuda.Stream() for _ in range(nstreams)]
        for s_ in side:
            s_.wait_stream(cur)
        for i in range(k):
            with torch.cuda.stream(side[i % nstreams]):
                step(i)
        for s_ in side:
            cur.wait_stream(s_)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / k


res = {}
for G in (1, 2, 4, 8):
    rows = H // G
    nbytes = rows * wp * 4
    pool = max(2, min(16, (3 * 126 << 20) // (2 * nbytes) + 1))
    slabs = [torch.randint(-2**31, 2**31 - 1, (rows, wp), dtype=torch.int64, device=dev).to(torch.int32)
             for _ in range(pool)]
    outs = [torch.empty_like(x) for x in slabs]
    above = torch.randint(-2**31, 2**31 - 1, (wp,), dtype=torch.int64, device=dev).to(torch.int32)
    below = torch.randint(-2**31, 2**31 - 1, (wp,), dtype=torch.int64, device=dev).to(torch.int32)

    def step(i):                 # an interior rank: both halos present (the slowest case)
        if G == 1:
            cu.edges_packed(slabs[i % pool], W, 1, out=outs[i % pool])
        else:
            cu.edges_halo(slabs[i % pool], above, below, W, 1, out=outs[i % pool])
    k = pool * max(1, 48 // pool)
    res[G] = (timed(step, k, 3), timed(step, k, 1))
    del slabs, outs
    torch.cuda.empty_cache()
for G, (us3, us1) in res.items():
    print(f"G={G}: slab {H // G} rows, {us3:8.2f} us/step (serial {us1:8.2f}); modelled efficiency "
          f"{res[1][0] / (G * us3):.3f} (serial {res[1][1] / (G * us1):.3f})", flush=True)

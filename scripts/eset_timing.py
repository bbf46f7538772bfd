"""edge_set (EdgeSet output) on an 8192^2 packed raster: serial time per step
(CUDA-graph replay over a rotating pool); compare with BITEDGE_K1_GENERIC=1."""
import os, sys, torch
sys.path.insert(0, '.')
from paper_1401_5245_b200 import cuda as cu
dev = torch.device('cuda:0')
h = w = 8192; wp = w // 32
pool = 24
ins = [torch.randint(-2**31, 2**31 - 1, (h, wp), dtype=torch.int64, device=dev).to(torch.int32) for _ in range(pool)]
outs = [torch.empty_like(x) for x in ins]
def step(i): cu.edges_packed(ins[i % pool], w, 1, edgeset=True, out=outs[i % pool])
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for i in range(192): step(i)
g.replay(); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); g.replay(); b.record(); torch.cuda.synchronize()
print("edge_set 8192^2 u32 serial us/step", round(a.elapsed_time(b) * 1e3 / 192, 2))

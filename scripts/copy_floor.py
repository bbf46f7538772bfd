"""Serial / overlapped time of a plain 8 MiB -> 8 MiB device copy (torch copy_,
CUDA graph, rotating buffers > 3x L2): the floor for a C3-sized pass."""
import torch
dev = torch.device("cuda")
n = 8 << 20
pool = 24
ins = [torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev) for _ in range(pool)]
outs = [torch.empty_like(x) for x in ins]
for streams in (1, 2, 3):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cur = torch.cuda.current_stream()
        side = [torch.cuda.Stream() for _ in range(streams)]
        for s in side:
            s.wait_stream(cur)
        for i in range(192):
            with torch.cuda.stream(side[i % streams]):
                outs[i % pool].copy_(ins[i % pool])
        for s in side:
            cur.wait_stream(s)
    g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); g.replay(); b.record(); torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / 192
    print(f"streams={streams}: {us:.2f} us per 8 MiB copy -> {2 * n / us / 1e3:.0f} GB/s")

"""K1 across widths (packed u32 and the drop-in's u64 words): kernel time per
step by CUDA-graph replay over a rotating pool > 3x L2, 3 streams and serial."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_5245_b200 import cuda as cu  # noqa: E402

dev = torch.device("cuda:0")


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


SHAPES = ((8192, 8192), (8192, 8000), (8192, 8064), (8192, 8160), (8192, 7999),
          (4096, 16384 - 32), (32768, 32000))
if os.environ.get("K1W_SHAPES"):      # e.g. K1W_SHAPES=4096x4096,16384x16384
    SHAPES = tuple(tuple(int(v) for v in t.split("x")) for t in os.environ["K1W_SHAPES"].split(","))
for bits in (32, 64):
    for (h, w) in SHAPES:
        wp = -(-w // bits)
        dt = torch.int32 if bits == 32 else torch.int64
        nbytes = h * wp * bits // 8
        pool = max(2, min(48, (3 * 126 << 20) // (2 * nbytes) + 1))
        ins = [torch.randint(-2**31, 2**31 - 1, (h, wp), dtype=torch.int64, device=dev).to(dt)
               for _ in range(pool)]
        outs = [torch.empty_like(x) for x in ins]

        def step(i):
            cu.edges_packed(ins[i % pool], w, 1, out=outs[i % pool])
        k = pool * max(1, 192 // pool)
        us3, us1 = timed(step, k, 3), timed(step, k, 1)
        alg = h * w * 0.25
        print(f"u{bits} {h}x{w}: {us3:6.2f} us ({alg / us3 / 1e3 / 6540.5:.3f}), serial {us1:6.2f} us "
              f"({alg / us1 / 1e3 / 6540.5:.3f})", flush=True)

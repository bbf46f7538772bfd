"""C2 e2e step variants, pipelined over two streams in 8 MiB input chunks: the
result leaves by a D2H copy (HostBatchEdges' staged path) or is written by the
kernel straight into page-locked host memory (zero-copy output)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_5245_b200 import _capi, synth  # noqa: E402

lib = _capi.load()
dev = torch.device("cuda:0")
n, h, w = 4096, 64, 64
wp = 2
imgs = synth.c2_images(n)
hin = torch.empty((n, h, w), dtype=torch.uint8, pin_memory=True)
hin.copy_(imgs)
houts = [torch.empty((n, h, wp), dtype=torch.int32, pin_memory=True) for _ in range(2)]
chunk = 2048
din = [torch.empty((chunk, h, w), dtype=torch.uint8, device=dev) for _ in range(2)]
dout = [torch.empty((chunk, h, wp), dtype=torch.int32, device=dev) for _ in range(2)]
ss = [torch.cuda.Stream() for _ in range(2)]


def step(i, zc_out):
    hout = houts[i & 1]
    for c in range(n // chunk):
        s = ss[c & 1]
        with torch.cuda.stream(s):
            din[c & 1].copy_(hin[c * chunk:(c + 1) * chunk], non_blocking=True)
            dst = hout[c * chunk:(c + 1) * chunk] if zc_out else dout[c & 1]
            lib.be_pack_edge_u8(din[c & 1].data_ptr(), dst.data_ptr(), chunk, h, w, w, wp, 1, None,
                                s.cuda_stream)
            if not zc_out:
                hout[c * chunk:(c + 1) * chunk].copy_(dout[c & 1], non_blocking=True)


def run(zc_out, steps=400):
    for i in range(10):
        step(i, zc_out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for s in ss:
        s.wait_stream(torch.cuda.current_stream())
    for i in range(steps):
        step(i, zc_out)
    for s in ss:
        torch.cuda.current_stream().wait_stream(s)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


for zc in (False, True, False, True):
    ms = run(zc)
    print(f"output {'zero-copy' if zc else 'D2H copy '}: {ms:.4f} ms/step  {n * h * w / ms / 1e6:.2f} Gpx/s",
          flush=True)
step(0, True)
torch.cuda.synchronize()
a = houts[0].clone()
step(0, False)
torch.cuda.synchronize()
print("same words:", bool(torch.equal(a, houts[0])))

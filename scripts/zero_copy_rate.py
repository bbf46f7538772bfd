"""Zero-copy throughput: the fused pack+edge kernels reading uint8 pixels from
page-locked host memory (and writing words to it) over PCIe, against the
DMA-staged path.  C2 batch (16 MiB in, 2 MiB out) and single C1 / 1024^2 images."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_5245_b200 import _capi, synth  # noqa: E402

lib = _capi.load()
dev = torch.device("cuda:0")


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


for n, h, w in ((4096, 64, 64), (1, 256, 256), (64, 256, 256), (1, 1024, 1024), (16, 1024, 1024)):
    imgs = synth.c2_images(n) if (h, w) == (64, 64) else torch.randint(0, 2, (n, h, w), dtype=torch.uint8)
    hin = torch.empty((n, h, w), dtype=torch.uint8, pin_memory=True)
    hin.copy_(imgs)
    wp = -(-w // 32)
    hout = torch.empty((n, h, wp), dtype=torch.int32, pin_memory=True)
    din = torch.empty((n, h, w), dtype=torch.uint8, device=dev)
    dout = torch.empty((n, h, wp), dtype=torch.int32, device=dev)
    s = torch.cuda.current_stream().cuda_stream

    def zc():
        lib.be_pack_edge_u8(hin.data_ptr(), hout.data_ptr(), n, h, w, w, wp, 1, None, s)

    def staged():
        din.copy_(hin, non_blocking=True)
        lib.be_pack_edge_u8(din.data_ptr(), dout.data_ptr(), n, h, w, w, wp, 1, None, s)
        hout.copy_(dout, non_blocking=True)

    def kernel_only():
        lib.be_pack_edge_u8(din.data_ptr(), dout.data_ptr(), n, h, w, w, wp, 1, None, s)

    reps = 200 if n * h * w < (8 << 20) else 50
    for name, fn in (("zero-copy", zc), ("staged", staged), ("kernel only", kernel_only)):
        us = timed(fn, reps)
        print(f"{n}x{h}x{w} {name:12s} {us:9.2f} us/step  {n * h * w / us / 1e3:8.2f} Gpx/s  "
              f"{n * h * w * 1.125 / us / 1e3:7.2f} GB/s", flush=True)
    staged()
    torch.cuda.synchronize()
    ref = hout.clone()
    hout.zero_()
    zc()
    torch.cuda.synchronize()
    print("   zero-copy == staged:", bool(torch.equal(ref, hout)), flush=True)

"""PCIe floor for the C2 e2e step (16 MiB uint8 in, 2 MiB words out), pipelined
the way bench.py's e2e loop is (step i enqueued before step i-1's result is
awaited), against HostBatchEdges at several chunk sizes."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1401_5245_b200 import synth  # noqa: E402
from paper_1401_5245_b200.host import HostBatchEdges  # noqa: E402

dev = torch.device("cuda")
a = torch.empty(16 << 20, dtype=torch.uint8, pin_memory=True)
da = torch.empty_like(a, device=dev)
b = [torch.empty(2 << 20, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
db = torch.empty(2 << 20, dtype=torch.uint8, device=dev)
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, steps=200):
    for _ in range(5):
        fn(0)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for i in range(steps):
        fn(i)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / steps * 1e3


def h2d_only(i):
    da.copy_(a, non_blocking=True)


ev = [torch.cuda.Event(), torch.cuda.Event()]


def h2d_d2h(i):
    with torch.cuda.stream(s_in):
        da.copy_(a, non_blocking=True)
    s_out.wait_stream(s_in)
    with torch.cuda.stream(s_out):
        b[i & 1].copy_(db, non_blocking=True)
        ev[i & 1].record()
    if i > 0:
        ev[(i - 1) & 1].synchronize()


print(f"h2d 16 MiB back to back: {timed(h2d_only):.4f} ms/step")
print(f"h2d 16 MiB + d2h 2 MiB, pipelined: {timed(h2d_d2h):.4f} ms/step")
imgs = synth.c2_images(4096)
for chunk in (4096, 2048, 1024, 512, 256):
    pipe = HostBatchEdges(imgs.shape, kind="u8", chunk_images=chunk)
    hin, hout = pipe.new_host_buffers()
    hin.copy_(imgs)
    houts = [hout, torch.empty_like(hout, pin_memory=True)]
    done = [torch.cuda.Event(), torch.cuda.Event()]

    def step(i):
        pipe(hin, houts[i & 1], sync=False)
        done[i & 1].record()
        if i > 0:
            done[(i - 1) & 1].synchronize()
            _ = int(houts[(i - 1) & 1][0, 0, 0])

    pend = [None, None]

    def step_submit(i):
        pend[i & 1] = pipe.submit(hin, houts[i & 1])
        if i > 0:
            _ = int(pend[(i - 1) & 1].synchronize()[0, 0, 0])

    ms = timed(step)
    ms2 = timed(step_submit)
    print(f"HostBatchEdges chunk={chunk}: __call__ {ms:.4f} ms/step -> {4096 * 4096 / ms / 1e6:.1f} "
          f"Gpx/s; submit {ms2:.4f} ms/step -> {4096 * 4096 / ms2 / 1e6:.1f} Gpx/s")

# C4-sized: 512 MiB in and 512 MiB out, 8 MiB chunks, both directions at once
big_in = torch.empty(512 << 20, dtype=torch.uint8, pin_memory=True)
big_out = torch.empty(512 << 20, dtype=torch.uint8, pin_memory=True)
dbuf = [torch.empty(8 << 20, dtype=torch.uint8, device=dev) for _ in range(2)]
dsrc = torch.empty(8 << 20, dtype=torch.uint8, device=dev)
ss = [torch.cuda.Stream(), torch.cuda.Stream()]


def duplex(_):
    for c in range(64):
        with torch.cuda.stream(ss[c & 1]):
            dbuf[c & 1].copy_(big_in[c << 23:(c + 1) << 23], non_blocking=True)
            big_out[c << 23:(c + 1) << 23].copy_(dsrc, non_blocking=True)


def h2d_only_big(_):
    for c in range(64):
        with torch.cuda.stream(ss[c & 1]):
            dbuf[c & 1].copy_(big_in[c << 23:(c + 1) << 23], non_blocking=True)


def d2h_only_big(_):
    for c in range(64):
        with torch.cuda.stream(ss[c & 1]):
            big_out[c << 23:(c + 1) << 23].copy_(dsrc, non_blocking=True)


print(f"512 MiB H2D only: {timed(h2d_only_big, 5):.3f} ms; D2H only: {timed(d2h_only_big, 5):.3f} ms; "
      f"both at once: {timed(duplex, 5):.3f} ms")

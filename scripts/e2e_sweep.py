import sys, time, torch
sys.path.insert(0, '.')
from paper_1401_5245_b200 import synth
from paper_1401_5245_b200.host import HostBatchEdges
imgs = synth.c2_images(4096)
for chunk in (4096, 2048, 1024, 512, 256):
    pipe = HostBatchEdges(imgs.shape, kind="u8", chunk_images=chunk)
    hin, hout = pipe.new_host_buffers(); hin.copy_(imgs)
    for _ in range(3): pipe(hin, hout)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(100):
        pipe(hin, hout, sync=True); _ = int(hout[0, 0, 0])
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 100
    print(chunk, round(ms, 4), 'ms', round(4096*4096/ms/1e6, 1), 'Gpx/s', round(16.8e6/ms/1e6, 1), 'GB/s h2d')
# raw H2D bandwidth
x = torch.empty(64 << 20, dtype=torch.uint8, pin_memory=True); y = torch.empty_like(x, device='cuda')
for _ in range(3): y.copy_(x, non_blocking=True)
torch.cuda.synchronize(); t=time.time()
for _ in range(20): y.copy_(x, non_blocking=True)
torch.cuda.synchronize(); print('h2d GB/s', 20*64*2**20/(time.time()-t)/1e9)
for _ in range(20): x.copy_(y, non_blocking=True)
torch.cuda.synchronize(); t=time.time()
for _ in range(20): x.copy_(y, non_blocking=True)
torch.cuda.synchronize(); print('d2h GB/s', 20*64*2**20/(time.time()-t)/1e9)
# floor: one 16 MiB H2D + one 2 MiB D2H + host sync per step, no kernel
a = torch.empty(16 << 20, dtype=torch.uint8, pin_memory=True); da = torch.empty_like(a, device='cuda')
b = torch.empty(2 << 20, dtype=torch.uint8, pin_memory=True); db = torch.empty_like(b, device='cuda')
for _ in range(5):
    da.copy_(a, non_blocking=True); b.copy_(db, non_blocking=True); torch.cuda.synchronize()
t = time.time()
for _ in range(100):
    da.copy_(a, non_blocking=True); b.copy_(db, non_blocking=True); torch.cuda.synchronize()
dt = (time.time() - t) / 100
print('floor copy-only step', round(dt * 1e3, 4), 'ms ->', round(4096 * 4096 / dt / 1e9, 1), 'Gpx/s')

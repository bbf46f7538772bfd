import time, statistics, numpy as np, torch
def med(fn, n=20):
    fn(); ts=[]
    for _ in range(n):
        t=time.perf_counter(); fn(); ts.append((time.perf_counter()-t)*1e6)
    return statistics.median(ts)
print("threads", torch.get_num_threads())
for sz in (1<<20, 4<<20, 64<<20):
    a = np.random.default_rng(0).integers(0, 2, sz, dtype=np.uint8)
    p = torch.empty(sz, dtype=torch.uint8, pin_memory=True)
    ta = torch.from_numpy(a)
    d = torch.empty(sz, dtype=torch.uint8, device="cuda")
    print(sz>>20, "MiB np.copyto", round(med(lambda: np.copyto(p.numpy(), a))), "torch copy_", round(med(lambda: p.copy_(ta))),
          "pageable .to(dev)", round(med(lambda: (d.copy_(ta), torch.cuda.synchronize()))),
          "pinned H2D", round(med(lambda: (d.copy_(p, non_blocking=True), torch.cuda.synchronize()))))

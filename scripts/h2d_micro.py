"""Pageable host<->device copies of a 256^2 image: torch vs raw cudaMemcpy
(the drop-in API's small-image fixed costs)."""
import ctypes, time, statistics, glob, os
import numpy as np, torch
dev = torch.device("cuda")
a = (np.random.default_rng(0).random((256, 256)) < 0.5).astype(np.uint8)
d = torch.empty((256, 256), dtype=torch.uint8, device=dev)
out = torch.empty((256, 4), dtype=torch.int64, device=dev)
hout = np.empty((256, 4), np.uint64)
cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + glob.glob("/usr/local/cuda/lib64/libcudart.so*")
rt = ctypes.CDLL(cands[0])
def med(fn, n=300):
    fn(); ts=[]
    for _ in range(n):
        t=time.perf_counter(); fn(); ts.append((time.perf_counter()-t)*1e6)
    return statistics.median(ts)
print("lib", cands[0])
print("torch .to(dev)", med(lambda: torch.from_numpy(a).to(dev)))
print("torch d.copy_(from_numpy)", med(lambda: (d.copy_(torch.from_numpy(a)), torch.cuda.synchronize())))
print("cudaMemcpy H2D pageable 64KB", med(lambda: rt.cudaMemcpy(ctypes.c_void_p(d.data_ptr()), ctypes.c_void_p(a.ctypes.data), ctypes.c_size_t(a.nbytes), 1)))
print("torch out.cpu()", med(lambda: out.cpu()))
print("cudaMemcpy D2H pageable 8KB", med(lambda: rt.cudaMemcpy(ctypes.c_void_p(hout.ctypes.data), ctypes.c_void_p(out.data_ptr()), ctypes.c_size_t(hout.nbytes), 2)))
print("torch.empty 64KB", med(lambda: torch.empty((256,256), dtype=torch.uint8, device=dev)))

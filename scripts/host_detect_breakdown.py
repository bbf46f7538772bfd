"""Pieces of the drop-in host flow (BitImage.from_array(a) -> detect_edges_mask
-> .words) for one small image: where the per-call microseconds go."""
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_5245_b200 import _capi  # noqa: E402
from paper_1401_5245_b200 import cuda as cu  # noqa: E402
from paper_1401_5245_b200.bitimage import BitImage  # noqa: E402
from paper_1401_5245_b200.edge import detect_edges_mask  # noqa: E402


def med_us(fn, reps=300):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e6)
    return statistics.median(ts)


n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
a = (np.random.default_rng(0).random((n, n)) < 0.5).astype(np.uint8)
dev = torch.device("cuda:0")
hp = torch.empty((n, n), dtype=torch.uint8, pin_memory=True)
hp.numpy()[...] = a
wp = -(-n // 64)
dpix = torch.empty((n, n), dtype=torch.uint8, device=dev)
out = torch.empty((n, wp), dtype=torch.int64, device=dev)
pk = torch.empty((n, wp), dtype=torch.int64, device=dev)
host = torch.empty((n, wp), dtype=torch.int64, pin_memory=True)
lib = _capi.load()
s = torch.cuda.current_stream().cuda_stream
rows = {
    "torch.empty pinned (out words)": lambda: torch.empty((n, wp), dtype=torch.int64, pin_memory=True),
    "torch.empty pinned (pixels)": lambda: torch.empty((n, n), dtype=torch.uint8, pin_memory=True),
    "np.copyto into pinned": lambda: np.copyto(hp.numpy(), a),
    "tensor.is_pinned()": lambda: hp.is_pinned(),
    "3 x torch.empty device": lambda: (torch.empty((n, n), dtype=torch.uint8, device=dev),
                                       torch.empty((n, wp), dtype=torch.int64, device=dev),
                                       torch.empty((n, wp), dtype=torch.int64, device=dev)),
    "raw be_host_detect_u64": lambda: lib.be_host_detect_u64(hp.data_ptr(), n, n, 1, 0, dpix.data_ptr(),
                                                             pk.data_ptr(), out.data_ptr(),
                                                             host.data_ptr(), s),
    "raw be_host_detect_u64 zero-copy": lambda: lib.be_host_detect_u64(hp.data_ptr(), n, n, 1, 0, None,
                                                                       pk.data_ptr(), None,
                                                                       host.data_ptr(), s),
    "raw zero-copy, no packed output": lambda: lib.be_host_detect_u64(hp.data_ptr(), n, n, 1, 0, None,
                                                                      None, None, host.data_ptr(), s),
    "torch.cuda.synchronize (idle)": lambda: torch.cuda.synchronize(),
    "cu.host_detect": lambda: cu.host_detect(hp, 1),
    "cu.host_detect staged": lambda: cu.host_detect(hp, 1, zero_copy=False),
    "BitImage.from_array": lambda: BitImage.from_array(a),
    "full host flow": lambda: detect_edges_mask(BitImage.from_array(a)).words,
}
for k, fn in rows.items():
    print(f"{k:36s} {med_us(fn):8.1f} us", flush=True)

"""Kernel-only timing sweep (random content -- the kernels are branch-free in
the pixels): per config, average launch time over a rotating pool > 3x L2,
CUDA-graph replay.  Usage: python scripts/kbench.py [c1 c2 ...]"""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_5245_b200 import cuda as cu  # noqa: E402

SHAPES = {"c1": ("u8", 1, 256, 256), "c2": ("u8", 4096, 64, 64), "c3": ("packed", 1, 8192, 8192),
          "c4": ("packed", 1, 65536, 65536), "c5": ("u8", 1024, 2048, 2048),
          "c3_64": ("packed64", 1, 8192, 8192), "c3_p4": ("p4", 1, 8192, 8192),
          "c4_p4": ("p4", 1, 65536, 65536)}
BPP = {"u8": 1.125, "packed": 0.25, "packed64": 0.25, "p4": 0.25}


def run(cfg, iters=200):
    kind, n, h, w = SHAPES[cfg]
    dev = torch.device("cuda")
    if kind == "u8":
        base = torch.randint(0, 2, (n, h, w), dtype=torch.uint8, device=dev)
        outw = (w + 31) // 32
        in_b, out_b = n * h * w, n * h * outw * 4
    elif kind == "packed":
        base = torch.randint(-2**31, 2**31 - 1, (n, h, w // 32), dtype=torch.int32, device=dev)
        in_b = out_b = n * h * w // 8
    elif kind == "p4":
        base = torch.randint(0, 256, (n * h * (w // 8),), dtype=torch.uint8, device=dev)
        in_b = out_b = n * h * w // 8
    else:
        base = torch.randint(-2**62, 2**62, (n, h, w // 64), dtype=torch.int64, device=dev)
        in_b = out_b = n * h * w // 8
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    pool = max(1, min(64, -(-3 * l2 // (in_b + out_b))))
    ins = [base] + [base.clone() for _ in range(pool - 1)]
    outs = []
    for x in ins:
        if kind == "u8":
            outs.append(torch.empty((n, h, (w + 31) // 32), dtype=torch.int32, device=dev))
        else:
            outs.append(torch.empty_like(x))

    from paper_1401_5245_b200 import pbm

    def step(i):
        j = i % pool
        if kind == "u8":
            cu.pack_edges_u8(ins[j], 1, out=outs[j])
        elif kind == "p4":
            outs[j] = pbm.detect_p4(ins[j], n, h, w)
        else:
            cu.edges_packed(ins[j], w, 1, out=outs[j])

    for i in range(3):
        step(i)
    torch.cuda.synchronize()
    if os.environ.get("KB_NOGRAPH"):
        for i in range(int(os.environ.get("KB_NOGRAPH"))):
            step(i)
        torch.cuda.synchronize()
        return {"cfg": cfg, "profiled_launches": int(os.environ.get("KB_NOGRAPH"))}
    g = torch.cuda.CUDAGraph()
    k = pool * max(1, iters // pool)
    nstreams = int(os.environ.get("KB_STREAMS", "1"))
    with torch.cuda.graph(g):
        if nstreams == 1:
            for i in range(k):
                step(i)
        else:
            # independent batches on parallel graph branches (fork / join)
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
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / k
    px = n * h * w
    gbs = px * BPP[kind] / (us * 1e-6) / 1e9
    return {"cfg": cfg, "kernel": os.environ.get("BITEDGE_KERNEL", "auto"), "us": round(us, 2),
            "gpx_s": round(px / us / 1e3, 1), "alg_GBps": round(gbs, 1),
            "frac_6540": round(gbs / 6540.5, 3), "pool": pool, "launches": k}


if __name__ == "__main__":
    cfgs = sys.argv[1:] or ["c1", "c2", "c3", "c3_64", "c4", "c5"]
    for c in cfgs:
        print(json.dumps(run(c, iters=200 if c not in ("c4", "c5") else 20)), flush=True)

#!/usr/bin/env python
"""Benchmark of the method-of-masks edge detector on B200 (BASELINE.json metric:
Gpixel/s, and % of the HBM roofline).

    python bench.py [--config c2] [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one pass of the hot path over one batch of the config's synthetic
input; the default workload is configs[1] (C2: 4096 glyphs of
64x64 uint8, fused pack+edge).  Under torchrun (N>1) the batch configs shard a
stream of independent images (C2, C5: one batch per rank, no collective ->
weak scaling; --strong splits one batch instead), C4 is row-sharded with a
1-row NCCL halo exchange (strong scaling), and C1/C3 run replicas.  Rank 0
prints ONE JSON line.

* value: whole-job Gpixel/s with inputs resident in HBM -- K steps on the
  device, CUDA-event timed, max over ranks; consecutive steps rotate through a
  pool of input/output buffers whose footprint exceeds 3x L2 (no L2 reuse);
  small-batch configs replay the steps from a CUDA graph.
* e2e: the same metric through the host-buffer API (paper_1401_5245_b200.host)
  with pinned host input, H2D copy, kernel and D2H of the packed result inside
  the timed region.
* roofline: algorithmic bytes per launch (1.125 B/px uint8 -> packed, 0.25 B/px
  packed -> packed) / average launch duration, against MEASURED_PEAKS.json.
* cpu_baseline: the oracle port of the reference CPU path (numpy, one thread)
  on a bounded sample, rank 0 at N=1.
* --impl reference: the reference CPU path (oracle port; the reference is
  Python and cannot travel to the GPU box) on all host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (kind, n, h, w, sharding, description)
    "c1": ("u8", 1, 256, 256, "replica", "C1 256x256 uint8, 12 disks + 8 rects"),
    "c2": ("u8", 4096, 64, 64, "batch", "C2 4096 x 64x64 uint8 glyphs"),
    "c3": ("packed", 1, 8192, 8192, "replica", "C3 8192^2 Bernoulli(0.5) packed u32"),
    "c4": ("packed", 1, 65536, 65536, "rows", "C4 65536^2 200k disks packed u32"),
    "c5": ("u8", 1024, 2048, 2048, "batch", "C5 1024 x 2048^2 uint8 pages"),
}
BYTES_PER_PX = {"u8": 1.125, "packed": 0.25}
METRIC = "Gpixel/s mask-method edge detection (1/2/4/8 B200); % of HBM roofline"
DEFAULT_STEPS = {"c1": 200000, "c2": 200000, "c3": 150000, "c4": 3000, "c5": 600}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms in the background."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return self
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        time.sleep(0.3)
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.samples.append((time.time(), parts))

    def stop(self, t0, t1):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        win = [s for t, s in self.samples if t0 - 0.15 <= t <= t1 + 0.15] or \
              [s for _, s in self.samples]
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        sm = [num(s[0]) for s in win if num(s[0]) is not None]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in win:
            for nm, v in zip(names, s[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": num(win[0][1]), "reasons": sorted(reasons), "samples": len(win)}


# ----------------------------------------------------------------------------- data

def make_rank_input(cfg, lo, hi, dev):
    """This rank's share of the config's synthetic input, resident in HBM."""
    import numpy as np
    import torch

    from paper_1401_5245_b200 import synth

    name = cfg
    kind, n, h, w, shard, _ = CONFIGS[name]
    if name == "c1":
        return torch.from_numpy(synth.c1_image()).to(dev).unsqueeze(0)
    if name == "c2":
        return synth.c2_images(hi - lo, start=lo, device=dev)
    if name == "c3":
        return torch.from_numpy(synth.c3_words().view(np.int32)).to(dev).unsqueeze(0)
    if name == "c4":
        return synth.c4_slab(lo, hi, synth.c4_disks(), device=dev).unsqueeze(0)
    if name == "c5":
        return synth.c5_pages(hi - lo, start=lo, device=dev)
    raise ValueError(name)


def host_sample(cfg, budget_px):
    """A bounded CPU-side sample of the config's input for the CPU legs:
    returns ('u8', [images]) or ('packed', (u32 rows, width))."""
    import numpy as np

    from paper_1401_5245_b200 import synth

    kind, n, h, w, _, _ = CONFIGS[cfg]
    if cfg == "c1":
        return "u8", [synth.c1_image()], h * w
    if cfg == "c2":
        k = max(1, min(n, budget_px // (h * w)))
        imgs = synth.c2_images(k).numpy()
        return "u8", list(imgs), k * h * w
    if cfg == "c3":
        return "packed", (synth.c3_words(), w), h * w
    if cfg == "c4":
        rows = max(2, min(h, budget_px // w))
        import torch

        slab = synth.c4_slab(0, rows, synth.c4_disks(), device="cpu")
        return "packed", (slab.numpy().view(np.uint32), w), rows * w
    if cfg == "c5":
        k = max(1, min(n, budget_px // (h * w)))
        pages = synth.c5_pages(k, device="cpu").numpy()
        return "u8", list(pages), k * h * w
    raise ValueError(cfg)


# ----------------------------------------------------------------------------- CPU legs

_WORK = None


def _cpu_unit(i):
    """One unit of the reference CPU path: from_array (u8) + detect_edges_mask,
    or detect_edges_mask of one packed raster (SPEC.md:165-168 over the port
    of bitimage.py)."""
    from oracle import port as P

    kind, data = _WORK
    if kind == "u8":
        img = P.from_array(data[i])
        return int(P.detect_edges_mask(img, 1).words[0, 0])
    words, width = data[i]
    img = P.make(width, words.shape[0], P.u32_rows_to_u64(words))
    return int(P.detect_edges_mask(img, 1).words[0, 0])


def _units(kind, data, chunks):
    """Split the sample into independent work units (images, or row blocks of
    one raster with their 1-row halos handled by overlap)."""
    if kind == "u8":
        return kind, data
    words, width = data
    rows = words.shape[0]
    if chunks <= 1 or rows < 64:
        return "packed", [(words, width)]
    edges = [rows * i // chunks for i in range(chunks + 1)]
    parts = []
    for a, b in zip(edges[:-1], edges[1:]):
        lo, hi = max(0, a - 1), min(rows, b + 1)      # overlap rows give the halos
        parts.append((words[lo:hi], width))
    return "packed", parts


def host_info():
    """The host the CPU legs ran on (core counts and CPU model)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    aff = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None
    return {"cpu_count": os.cpu_count(), "affinity": aff, "model": model}


def cpu_time_port(cfg, budget_s=3.0, reps_min=3):
    """cpu_baseline: the oracle port, single thread, median of >= 3 reps."""
    global _WORK
    kind, data, px = host_sample(cfg, budget_px=8192 * 8192)
    _WORK = _units(kind, data, 1)
    units = len(_WORK[1])
    for i in range(units):           # warm-up
        _cpu_unit(i)
    times = []
    t_all = time.perf_counter()
    while len(times) < reps_min or (time.perf_counter() - t_all < budget_s and len(times) < 50):
        t0 = time.perf_counter()
        for i in range(units):
            _cpu_unit(i)
        times.append(time.perf_counter() - t0)
    med = statistics.median(times)
    return {"value": px / med / 1e9, "unit": "Gpixel/s", "cores": 1, "kind": "port",
            "sample": f"{cfg}: {px} px ({units} unit(s)) per rep, median of {len(times)} reps, "
                      "oracle/port.py (reference BitImage composition, numpy, 1 thread)",
            "host": host_info()}


def run_reference(args):
    """--impl reference: the reference CPU path on all host cores."""
    import multiprocessing as mp

    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    cfg = args.config
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    global _WORK
    kind, data, px_total = host_sample(cfg, budget_px=1 << 26)
    _WORK = _units(kind, data, cores)
    units = len(_WORK[1])
    px_per_unit = px_total / units
    if units < 2:
        # one indivisible unit (C1's single image): a process pool only adds
        # its dispatch latency -- time it in this process, one core
        cores = 1
        for _ in range(args.warmup):
            _cpu_unit(0)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            _cpu_unit(0)
        dt = time.perf_counter() - t0
        k = 1
        return _print_reference(args, cfg, px_per_unit * k, dt, cores, k, units)
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        # calibrate: seconds per unit on this pool
        t0 = time.perf_counter()
        pool.map(_cpu_unit, range(units), chunksize=max(1, units // (4 * cores)))
        per_pass = time.perf_counter() - t0
        # size each step so the whole run (warmup + steps) stays ~<= 120 s
        budget = 120.0 / max(1, args.steps + args.warmup)
        k = units if per_pass <= budget else max(1, int(units * budget / per_pass))
        k = max(min(k, units), min(units, cores))
        sel = list(range(k))
        for _ in range(args.warmup):
            pool.map(_cpu_unit, sel, chunksize=max(1, k // (4 * cores)))
        t0 = time.perf_counter()
        for _ in range(args.steps):
            pool.map(_cpu_unit, sel, chunksize=max(1, k // (4 * cores)))
        dt = time.perf_counter() - t0
    return _print_reference(args, cfg, px_per_unit * k, dt, cores, k, units)


def _print_reference(args, cfg, px_step, dt, cores, k, units):
    value = px_step * args.steps / dt / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "Gpixel/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": CONFIGS[cfg][5], "config_id": cfg,
                   "step_sample_px": int(px_step)},
        "cpu_baseline": {"value": value, "unit": "Gpixel/s", "cores": cores, "kind": "port",
                         "sample": f"{k} of {units} units ({int(px_step)} px) per step; "
                                   "oracle/port.py = the reference BitImage composition",
                         "host": host_info()},
        "e2e": {"value": value, "unit": "Gpixel/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm

def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1401_5245_b200 import _capi
    from paper_1401_5245_b200 import cuda as cu
    from paper_1401_5245_b200 import dist as bd
    from paper_1401_5245_b200.host import HostBatchEdges

    rank, world = bd.init()
    local = bd.env_rank_world()[2]
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = args.config
    kind, n, h, w, shard, desc = CONFIGS[cfg]
    props = torch.cuda.get_device_properties(dev)
    l2 = getattr(props, "L2_cache_size", 126 << 20)

    # ---- this rank's share.  Batch configs shard a stream of independent images:
    # by default every rank owns its own batch of n images (images [r*n, (r+1)*n)
    # of the global stream; weak scaling, no collective); --strong splits one
    # batch of n images across the ranks instead.
    if shard == "batch" and not args.strong:
        lo, hi = rank * n, (rank + 1) * n
        imgs_local, rows_local = n, h
    elif shard == "batch":
        lo, hi = bd.shard_range(n, rank, world)
        imgs_local, rows_local = hi - lo, h
    elif shard == "rows":
        lo, hi = bd.shard_range(h, rank, world)
        imgs_local, rows_local = 1, hi - lo
    else:
        lo, hi = 0, n
        imgs_local, rows_local = n, h
    px_local = imgs_local * rows_local * w
    wp = cu.words_per_row(w, 32)
    in_bytes = px_local * (1 if kind == "u8" else 0.125)
    out_bytes = imgs_local * rows_local * wp * 4
    step_bytes = in_bytes + out_bytes
    alg_bytes = px_local * BYTES_PER_PX[kind]

    t_gen = time.time()
    base = make_rank_input(cfg, lo, hi, dev)
    torch.cuda.synchronize()
    log(f"[rank {rank}] {cfg} input {tuple(base.shape)} generated in {time.time() - t_gen:.1f}s")

    # ---- rotating pool > 3x L2
    free = torch.cuda.mem_get_info(dev)[0]
    pool = int(min(max(1, math.ceil(3 * l2 / step_bytes)), max(1, (free * 0.6) // step_bytes), 512))
    ins, outs = [base], []
    for _ in range(pool - 1):
        ins.append(base.clone())
    # at least one output per parallel stream, so overlapping steps never share one
    for _ in range(max(pool, args.streams)):
        shape = (base.shape[0], base.shape[1], wp)
        outs.append(torch.empty(shape, dtype=torch.int32, device=dev))

    halo_mode = None
    if shard == "rows" and world > 1:
        slabs = None
        if args.halo == "p2p":
            # halo rows read from the neighbours' slabs over NVLink inside the kernel
            try:
                slabs = [bd.PeerHaloEdges(x[0], w, 1) for x in ins]
                halo_mode, launches_per_step = "p2p (CUDA IPC peer reads in the edge kernel)", 1
            except Exception as e:   # e.g. IPC unavailable in the container
                log(f"[rank {rank}] p2p halos unavailable ({e}); using NCCL")
                slabs = None
        if slabs is None:
            slabs = [bd.RowShardedEdges(x[0], w, 1) for x in ins]
            halo_mode, launches_per_step = "nccl (batch_isend_irecv, interior overlapped)", 3
        for s_, o in zip(slabs, outs):
            s_.out = o[0]
        dist.barrier()                 # every slab is complete before any neighbour reads it

        def step(i):
            slabs[i % pool].step()
        use_graph = False
    else:
        def step(i):
            x, o = ins[i % len(ins)], outs[i % len(outs)]
            if kind == "u8":
                cu.pack_edges_u8(x, 1, out=o)
            else:
                cu.edges_packed(x, w, 1, out=o)
        launches_per_step = 1
        use_graph = (step_bytes < (64 << 20)) and not args.no_graph

    steps, warmup = args.steps, args.warmup
    graphs = []
    if use_graph:
        # capture pool-sized chunks of steps; replaying them back to back keeps
        # the launch path off the CPU for these few-microsecond kernels
        s = torch.cuda.Stream(dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            for i in range(3):
                step(i)
        torch.cuda.current_stream(dev).wait_stream(s)
        torch.cuda.synchronize()

        def capture(count, nstreams):
            """Graph of `count` consecutive steps; with nstreams > 1 the steps
            (independent batches) alternate over parallel fork/join branches so
            one batch's kernel can overlap the previous one's tail."""
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                if nstreams <= 1:
                    for i in range(count):
                        step(i)
                else:
                    cur = torch.cuda.current_stream(dev)
                    side = [torch.cuda.Stream(dev) for _ in range(nstreams)]
                    for s_ in side:
                        s_.wait_stream(cur)
                    for i in range(count):
                        with torch.cuda.stream(side[i % nstreams]):
                            step(i)
                    for s_ in side:
                        cur.wait_stream(s_)
            return g
        chunk = min(max(1, steps), 1024)
        g_full = capture(chunk, args.streams)
        rem = steps % chunk
        g_rem = capture(rem, args.streams) if rem else None

        def run(k):
            q, r = divmod(k, chunk)
            for _ in range(q):
                g_full.replay()
            if r:
                (g_rem if r == rem and g_rem is not None else capture(r, args.streams)).replay()

        def serial_step_ms():
            """Single-stream (no overlap) time per step: the per-launch latency."""
            n_s = min(max(steps, 8), 512)
            gs = capture(n_s, 1)
            gs.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            gs.replay()
            b.record()
            torch.cuda.synchronize()
            return a.elapsed_time(b) / n_s
    else:
        nst = args.streams if not (shard == "rows" and world > 1) else 1
        side = [torch.cuda.Stream(dev) for _ in range(max(1, nst))]

        def run(k, nstreams=nst):
            """Direct launches; independent steps alternate over `nstreams`
            streams (fork/join around the K steps), as in the graph path."""
            if nstreams <= 1:
                for i in range(k):
                    step(i)
                return
            cur = torch.cuda.current_stream(dev)
            for s_ in side[:nstreams]:
                s_.wait_stream(cur)
            for i in range(k):
                with torch.cuda.stream(side[i % nstreams]):
                    step(i)
            for s_ in side[:nstreams]:
                cur.wait_stream(s_)

        def serial_step_ms():
            n_s = max(3, min(steps, 20))
            run(1, 1)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            run(n_s, 1)
            b.record()
            torch.cuda.synchronize()
            return a.elapsed_time(b) / n_s

        if nst <= 1:
            serial_step_ms = None

    # ---- warm-up, then exactly K timed steps (barrier + sync on both sides)
    run(warmup)
    if use_graph:
        # one untimed replay of each graph the timed region replays: a graph's
        # first launch uploads it (with K = 1000 the single timed replay was
        # otherwise 37 % slower per step)
        g_full.replay()
        if g_rem is not None:
            g_rem.replay()
    torch.cuda.synchronize()
    sampler = ClockSampler(local).start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    n0 = _capi.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_wall0 = time.time()
    ev0.record()
    run(steps)
    ev1.record()
    torch.cuda.synchronize()
    t_wall1 = time.time()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop(t_wall0, t_wall1)
    ms = ev0.elapsed_time(ev1)
    launched = _capi.launch_count() - n0
    gpu_launches = steps * launches_per_step if use_graph else launched
    ms_max = ms
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    weak_batch = shard == "batch" and not args.strong
    px_all = (n * h * w * world) if (weak_batch or shard == "replica") else (n * h * w)
    value = px_all * steps / (ms_max / 1e3) / 1e9
    ms_step = ms_max / steps

    # ---- roofline of the dominant kernel: algorithmic bytes per launch over the
    # average launch duration in the timed region (steps overlap when streams > 1)
    per_launch_ms = ms / steps / launches_per_step
    achieved = alg_bytes / (per_launch_ms / 1e3) / 1e9
    serial_ms = serial_step_ms() if (serial_step_ms is not None and args.streams > 1) else None
    peak, peak_src = measured_peaks()
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp) and world == 1:        # captured per launch at N = 1
        with open(tp) as f:
            traffic = json.load(f).get(cfg)

    # ---- e2e through the host-buffer API (pinned host in -> packed host out)
    e2e = None
    if not args.no_e2e:
        if shard == "rows" and world > 1:
            # this rank's row slab from host memory, with the neighbours'
            # boundary rows as host halos (be_host_edges_rows)
            from paper_1401_5245_b200 import synth

            ha, hb = lo > 0, hi < h
            pipe = HostBatchEdges(tuple(base.shape), kind=kind, width=w, device=dev,
                                  halo_rows=(ha, hb))
            hin, hout = pipe.new_host_buffers()
            host_rows = synth.c4_slab(lo - ha, hi + hb, synth.c4_disks(), device=dev)
            hin.copy_(host_rows.cpu().unsqueeze(0))
            del host_rows
        else:
            pipe = HostBatchEdges(tuple(base.shape), kind=kind, width=w, device=dev)
            hin, hout = pipe.new_host_buffers()
            hin.copy_(base.cpu())
        # ~16 GB of H2D per timed window (C2: ~950 steps, 0.3 s): averages the short
        # PCIe-rate dips seen on these boxes (scripts/e2e_windows.py)
        e2e_steps = max(3, min(steps, int(max(1, 16e9 / max(1, pipe.h2d_bytes)))))
        # `depth` batches in flight, one per lane of the pipe, each with its own
        # host output buffer: step i is submitted before step i-depth+1's result
        # is awaited and read on the host
        depth = max(2, pipe.lanes)
        houts = [hout] + [torch.empty_like(hout, pin_memory=True) for _ in range(depth - 1)]
        for _ in range(2):
            pipe(hin, hout)
        # warm the pipelined (submit) path over every host output buffer for
        # >= 0.25 s: a fresh box's first ~100 ms of PCIe traffic runs slower
        t_w, k, pw = time.time(), 0, [None] * depth
        while k < 8 or time.time() - t_w < 0.25:
            pw[k % depth] = pipe.submit(hin, houts[k % depth])
            if k >= depth - 1:
                pw[(k - depth + 1) % depth].synchronize()
            k += 1
        for j in range(max(0, k - depth + 1), k):
            pw[j % depth].synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # step i is submitted before step i-depth+1's result is awaited and read
        # on the host (`depth` host output buffers), so the CPU-side sync latency
        # and each step's kernel + D2H hide behind the following steps' H2D
        # (HostBatchEdges.submit does not chain batches; a lane per step in flight)
        pend = [None] * depth
        # timed in windows; the reported rate is the median window's (robust to
        # the transient PCIe-rate dips of these boxes, scripts/e2e_windows.py)
        nwin = 5 if e2e_steps >= 10 else 1
        per_win = e2e_steps // nwin
        e2e_steps = per_win * nwin
        wms = []
        for _ in range(nwin):
            e0.record()
            e0.synchronize()                 # every submitted copy starts after e0
            for i in range(per_win):
                pend[i % depth] = pipe.submit(hin, houts[i % depth])
                if i >= depth - 1:
                    res = pend[(i - depth + 1) % depth].synchronize()
                    _ = int(res[0, 0, 0])    # step i-depth+1's result, on the host
            for j in range(max(0, per_win - depth + 1), per_win):
                res = pend[j % depth].synchronize()
                _ = int(res[0, 0, 0])
            e1.record()
            torch.cuda.synchronize()
            wms.append(e0.elapsed_time(e1))
        if world > 1:
            t = torch.tensor(wms, device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            wms = [float(v) for v in t.tolist()]
        ems = statistics.median(wms) * nwin      # median window, as a whole-run time
        px_e2e = px_all
        moved = [int(pipe.h2d_bytes), int(pipe.d2h_bytes)]
        if world > 1:                        # the whole job's bytes per step
            t = torch.tensor(moved, device=dev, dtype=torch.int64)
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            moved = [int(v) for v in t.tolist()]
        e2e = {"value": px_e2e * e2e_steps / (ems / 1e3) / 1e9, "unit": "Gpixel/s",
               "h2d_bytes_per_step": moved[0], "d2h_bytes_per_step": moved[1],
               "steps": e2e_steps, "ms_per_step": ems / e2e_steps,
               "windows_gpx_s": [round(px_e2e * per_win / (m / 1e3) / 1e9, 2) for m in wms]}
        # this box's PCIe context for the number above (PCIe rates differ from box
        # to box and over time): the same bytes per step moved by plain pinned
        # 8 MiB copies with no kernels, both directions at once, timed right after
        fl_ms, h2d = copies_only_ms(hin, hout, dev)
        e2e["pcie_h2d_gbs"] = round(h2d, 2)
        e2e["copies_only_gpx_s"] = round(px_e2e / (fl_ms / 1e3) / 1e9, 2)
        e2e["frac_of_copies_only"] = round(e2e["value"] / e2e["copies_only_gpx_s"], 3)
        e2e["transfer"] = ("kernel reads / writes page-locked host memory (zero-copy)"
                           if pipe.zero_copy else "copy engines, chunks on two streams")

    # ---- parity gate on the measured output (before reporting a number)
    parity = None
    if rank == 0 and not args.no_check:
        parity = gate(cfg, ins[0], outs[0], kind, w)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_time_port(cfg)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Gpixel/s", "n_gpus": world,
            "steps": steps, "warmup": warmup, "ms_per_step": ms_step,
            "higher_is_better": True,
            "scaling": "strong" if (shard == "rows" or (shard == "batch" and args.strong))
                       else "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": desc, "config_id": cfg,
                       "global_batch": n * world if weak_batch else n, "per_rank_batch": imgs_local,
                       "image": [h, w], "input": "uint8 pixels" if kind == "u8" else
                       "packed u32 row words", "parallelism":
                       {"batch": f"batch-shard x{world}" + ("" if weak_batch else " (strong)"),
                        "rows": f"row-shard x{world}, halo: {halo_mode or 'none (1 rank)'}",
                        "replica": f"replicas x{world}"}[shard],
                       "l2_policy": f"rotating pool of {pool} input/output sets "
                                    f"({pool * step_bytes / 2**20:.0f} MiB > 3x L2 "
                                    f"{l2 / 2**20:.0f} MiB)" if pool > 1 else
                                    f"step footprint {step_bytes / 2**20:.0f} MiB > L2",
                       "launch": ("CUDA graph replay" if use_graph else "direct launches")
                                 + (f", independent steps on {args.streams} parallel streams"
                                    if args.streams > 1 and not (shard == "rows" and world > 1)
                                    else ", one stream")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "frac_of_nominal_8000": achieved / 8000.0,
                         "peak_source": peak_src,
                         "alg_bytes_per_launch": alg_bytes,
                         "avg_launch_us": per_launch_ms * 1e3,
                         "serial_launch_us": serial_ms * 1e3 if serial_ms else None,
                         "frac_serial": (alg_bytes / (serial_ms / 1e3) / 1e9 / peak)
                         if serial_ms else None,
                         "bytes_per_px": BYTES_PER_PX[kind]},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(gpu_launches),
            "clocks": clocks, "parity": parity,
            "device": props.name, "sm_count": props.multi_processor_count,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def copies_only_ms(hin, hout, dev, chunk=8 << 20, target_s=0.3):
    """(ms per step, H2D GB/s): one e2e step's bytes -- all of `hin` host -> device
    and all of `hout` device -> host, in `chunk`-byte copies on two streams so the
    directions overlap -- with no kernels: what PCIe alone allows the e2e step on
    this box.  Also the rate of H2D copies alone."""
    import torch

    src = hin.reshape(-1).view(torch.uint8)
    dst = hout.reshape(-1).view(torch.uint8)
    dbi = torch.empty(min(src.numel(), 8 * chunk), dtype=torch.uint8, device=dev)
    dbo = torch.empty(min(dst.numel(), 8 * chunk), dtype=torch.uint8, device=dev)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def step(h2d=True, d2h=True):
        if h2d:
            with torch.cuda.stream(s_in):
                for off in range(0, src.numel(), chunk):
                    n = min(chunk, src.numel() - off)
                    o = off % dbi.numel()
                    n = min(n, dbi.numel() - o)
                    dbi[o:o + n].copy_(src[off:off + n], non_blocking=True)
        if d2h:
            with torch.cuda.stream(s_out):
                for off in range(0, dst.numel(), chunk):
                    n = min(chunk, dst.numel() - off)
                    o = off % dbo.numel()
                    n = min(n, dbo.numel() - o)
                    dst[off:off + n].copy_(dbo[o:o + n], non_blocking=True)

    def timed(**kw):
        step(**kw)
        torch.cuda.synchronize()
        t = time.perf_counter()
        step(**kw)
        torch.cuda.synchronize()
        one = max(time.perf_counter() - t, 1e-6)
        reps = int(max(3, min(10000, target_s / one)))
        cur = torch.cuda.current_stream(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        s_in.wait_stream(cur)
        s_out.wait_stream(cur)
        for _ in range(reps):
            step(**kw)
        cur.wait_stream(s_in)
        cur.wait_stream(s_out)
        b.record(cur)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    both = timed()
    h2d_ms = timed(d2h=False)
    return both, src.numel() / (h2d_ms / 1e3) / 1e9


def gate(cfg, inp, out, kind, w):
    """Bit-exact check of the benchmarked output against the C per-pixel
    oracle (a 2048-row / 64-image sample for the big configs)."""
    import numpy as np

    from oracle import cscan

    if kind == "u8":
        k = min(inp.shape[0], 64 if inp.shape[1] >= 1024 else inp.shape[0])
        exp = cscan.scan_u8(inp[:k].cpu().numpy(), 1)
        got = out[:k].cpu().numpy().view(np.uint32)
        ok = bool((exp == got).all())
        if not ok:
            raise SystemExit(f"parity gate failed on {cfg}")
        return {"ok": ok, "checked_images": int(k), "oracle": "oracle/scan.c per-pixel Edge(p)"}
    rows = min(inp.shape[1], 2048)
    src = inp[0, :rows].cpu().numpy().view(np.uint32)
    exp = cscan.scan_p32(src, w, 1)
    got = out[0, :rows].cpu().numpy().view(np.uint32)
    # the last sampled row's lower neighbour lies outside the sample: compare rows [0, rows-1)
    ok = bool((exp[:-1] == got[:-1]).all()) if rows < inp.shape[1] else bool((exp == got).all())
    if not ok:
        raise SystemExit(f"parity gate failed on {cfg}")
    return {"ok": ok, "checked_rows": int(rows), "oracle": "oracle/scan.c per-pixel Edge(p)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--halo", choices=["p2p", "nccl"], default="p2p",
                    help="row-sharded configs: halo rows by peer reads in the kernel or NCCL")
    ap.add_argument("--strong", action="store_true",
                    help="batch configs: split one batch across ranks instead of one batch per rank")
    ap.add_argument("--streams", type=int, default=3,
                    help="parallel graph branches for independent batches (1 = serial)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = DEFAULT_STEPS[args.config] if args.impl == "ours" else 20
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

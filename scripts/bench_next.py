"""Measurement of the SURVEY 8(f) rows next to the hot path, to the same bar as
bench.py: device-resident input, rotating pool > 3x L2, CUDA-graph replay
(or direct launches for big steps), 3 parallel streams plus the serial
single-stream time, algorithmic bytes / launch against MEASURED_PEAKS.json,
and a parity check of the measured output against the C oracle.

    F1  P4 payload -> P4 payload (be_p4_edges)               0.25 B/px
    F2  grayscale uint8 -> threshold -> edge words (t = 128) 1.125 B/px
    F3  every output at once: edges, EdgeSet, 4 fundamental edges
        (+ the packed input for uint8)                       packed 0.875, uint8 1.875 B/px
    F4  the paper's per-pixel scan on the GPU (scan_edges)   0.25 B/px

    python scripts/bench_next.py [out.json] [row ...]
"""

import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import cscan  # noqa: E402  (parity checker only)
from oracle import port as P  # noqa: E402
from paper_1401_5245_b200 import cuda as cu  # noqa: E402
from paper_1401_5245_b200 import pbm, synth  # noqa: E402

DEV = torch.device("cuda")


def peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return float(json.load(open(p))["hbm_gbs"]) if os.path.exists(p) else 6650.0


def timed(step, pool, step_bytes, iters, streams=3):
    """(overlapped us/step, serial us/step)."""
    graph = step_bytes < (64 << 20)
    for i in range(3):
        step(i)
    torch.cuda.synchronize()

    def body(k, ns):
        if ns == 1:
            for i in range(k):
                step(i)
            return
        cur = torch.cuda.current_stream()
        side = [torch.cuda.Stream() for _ in range(ns)]
        for s_ in side:
            s_.wait_stream(cur)
        for i in range(k):
            with torch.cuda.stream(side[i % ns]):
                step(i)
        for s_ in side:
            cur.wait_stream(s_)

    res = []
    for ns in (streams, 1):
        k = pool * max(1, iters // pool)
        if graph:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                body(k, ns)
            run = g.replay
        else:
            def run(k=k, ns=ns):
                body(k, ns)
        run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        torch.cuda.synchronize()
        res.append(a.elapsed_time(b) * 1e3 / k)
    return res


def line(row, workload, px, bpp, us, us_serial, parity, kernel_note):
    alg = px * bpp
    pk = peak()
    return {"row": row, "workload": workload, "Gpixel_s": px / us / 1e3, "us_per_step": us,
            "serial_us_per_step": us_serial, "bytes_per_px": bpp,
            "roofline": {"bound": "hbm", "achieved": alg / us / 1e3, "peak": pk,
                         "frac": alg / us / 1e3 / pk, "frac_serial": alg / us_serial / 1e3 / pk},
            "parity": parity, "kernel": kernel_note}


def pool_for(step_bytes):
    l2 = torch.cuda.get_device_properties(DEV).L2_cache_size
    free = torch.cuda.mem_get_info()[0]
    return int(max(1, min(-(-3 * l2 // step_bytes), (free * 0.5) // step_bytes, 64)))


# ---------------------------------------------------------------- F1 P4
def f1(cfg):
    if cfg == "c3":
        words = synth.c3_words()                                   # [8192, 256] u32
        h = w = 8192
    else:
        h = w = 65536
        words = synth.c4_slab(0, h, synth.c4_disks(), device=DEV).cpu().numpy().view(np.uint32)
    rb = w // 8
    # P4 bytes: 1 = black, MSB first == ~(our words) byte-swapped to big-endian order
    payload = (~words).astype(">u4").view(np.uint8).reshape(-1)
    base = torch.from_numpy(payload.copy()).to(DEV)
    step_bytes = 2 * base.numel()
    pool = pool_for(step_bytes)
    ins = [base] + [base.clone() for _ in range(pool - 1)]
    outs = [torch.empty_like(base) for _ in range(max(pool, 3))]

    def step(i):
        pbm.detect_p4(ins[i % pool], 1, h, w, out=outs[i % len(outs)])
    us, us1 = timed(step, pool, step_bytes, 300 if cfg == "c3" else 30)
    step(0)
    got = outs[0].cpu().numpy()
    if cfg == "c3":
        exp = cscan.scan_p32(words, w)
    else:                       # the oracle on a 512-row band (rows 1000..1511 incl. halos)
        exp = cscan.scan_p32(words[999:1513], w)[1:-1]
        got = got.reshape(h, rb)[1000:1512].reshape(-1)
        words = None
    exp_p4 = (~exp).astype(">u4").view(np.uint8).reshape(-1)
    ok = bool((got.reshape(-1) == exp_p4).all())
    return line("F1 P4 codec fused", f"{cfg} {h}x{w} P4 payload -> P4 payload", h * w, 0.25, us,
                us1, {"ok": ok, "oracle": "oracle/scan.c" + (" (512-row band)" if cfg == "c4" else "")},
                "K1 with P4 byte load/store (be_p4_edges fused path)")


# ---------------------------------------------------------------- F2 threshold
def gray_of(binary, seed):
    """uint8 luminance whose >= 128 pixels are exactly the white ones."""
    g = torch.Generator(device=binary.device).manual_seed(seed)
    r = torch.randint(0, 128, binary.shape, dtype=torch.uint8, device=binary.device, generator=g)
    return r + binary * 128


def f2(cfg):
    if cfg == "c2":
        b = synth.c2_images(4096, device=DEV)
        n, h, w = 4096, 64, 64
    else:
        b = synth.c5_pages(1024, device=DEV)
        n, h, w = 1024, 2048, 2048
    base = gray_of(b, 7)
    del b
    step_bytes = base.numel() + n * h * (w // 32) * 4
    pool = pool_for(step_bytes)
    ins = [base] + [base.clone() for _ in range(pool - 1)]
    outs = [torch.empty((n, h, w // 32), dtype=torch.int32, device=DEV) for _ in range(max(pool, 3))]

    def step(i):
        cu.threshold_edges_u8(ins[i % pool], 128, 1, out=outs[i % len(outs)])
    us, us1 = timed(step, pool, step_bytes, 300 if cfg == "c2" else 20)
    step(0)
    k = 64 if cfg == "c2" else 4
    sample = (base[:k] >= 128).to(torch.uint8).cpu().numpy()
    ok = bool((outs[0][:k].cpu().numpy().view(np.uint32) == cscan.scan_u8(sample, 1)).all())
    return line("F2 threshold fused into the pack", f"{cfg} {n}x{h}x{w} uint8 luminance, t=128",
                n * h * w, 1.125, us, us1,
                {"ok": ok, "checked_images": k, "oracle": "oracle/scan.c on (gray >= 128)"},
                "K2 family with the SWAR >= t compare")


# ---------------------------------------------------------------- F3 all outputs
def f3(cfg):
    names = ["edges", "edgeset", "left", "right", "up", "down"]
    if cfg == "c3":
        base = torch.from_numpy(synth.c3_words().view(np.int32)).to(DEV).unsqueeze(0)
        n, h, w, bpp = 1, 8192, 8192, 0.875
        wp = w // 32
    else:
        base = synth.c5_pages(256, device=DEV)
        n, h, w, bpp = 256, 2048, 2048, 1.875
        wp = w // 32
        names.append("packed")
    out_b = n * h * wp * 4
    step_bytes = base.numel() * base.element_size() + len(names) * out_b
    pool = pool_for(step_bytes)
    ins = [base] + [base.clone() for _ in range(pool - 1)]
    outsets = [{k: torch.empty((n, h, wp), dtype=torch.int32, device=DEV) for k in names}
               for _ in range(max(pool, 3))]

    def step(i):
        cu.edges_general(ins[i % pool], w, 1, outs=outsets[i % len(outsets)])
    us, us1 = timed(step, pool, step_bytes, 300 if cfg == "c3" else 20)
    step(0)
    o = {k: v[0].cpu().numpy().view(np.uint32) for k, v in outsets[0].items()}
    if cfg == "c3":
        img = P.make(w, h, P.u32_rows_to_u64(synth.c3_words()))
    else:
        img = P.from_array(base[0].cpu().numpy())
    ok = bool((o["edges"] == P.u64_to_u32_rows(P.detect_edges_mask(img, 1).words)[:, :wp]).all())
    ok &= bool((o["edgeset"] == P.u64_to_u32_rows(P.edge_set(img, 1).words)[:, :wp]).all())
    mask = P.build_mask(img)
    for side in ("left", "right", "up", "down"):
        d = {"left": P.LEFT, "right": P.RIGHT, "up": P.UP, "down": P.DOWN}[side] \
            if hasattr(P, "LEFT") else side
        fe = P.fundamental_edge(img, mask, d, 1)
        ok &= bool((o[side] == P.u64_to_u32_rows(fe.words)[:, :wp]).all())
    if "packed" in o:
        ok &= bool((o["packed"] == P.u64_to_u32_rows(img.words)[:, :wp]).all())
    return line("F3 multi-output (4 fundamental edges + EdgeSet + edges)",
                f"{cfg} {n}x{h}x{w} -> {len(names)} outputs", n * h * w, bpp, us, us1,
                {"ok": ok, "oracle": "oracle/port.py composition (image 0)"},
                "edges_general (one read, every output)")


# ---------------------------------------------------------------- F4 GPU scan
def f4(cfg):
    words = synth.c3_words()
    h = w = 8192
    base = torch.from_numpy(words.view(np.int32)).to(DEV).unsqueeze(0)
    step_bytes = 2 * base.numel() * 4
    pool = pool_for(step_bytes)
    ins = [base] + [base.clone() for _ in range(pool - 1)]
    outs = [torch.empty_like(base) for _ in range(max(pool, 3))]

    def step(i):
        cu.scan_edges(ins[i % pool], w, 1, out=outs[i % len(outs)])
    us, us1 = timed(step, pool, step_bytes, 300)
    step(0)
    ok = bool((outs[0][0].cpu().numpy().view(np.uint32) == cscan.scan_p32(words, w)).all())
    return line("F4 per-pixel scan on the GPU (oracle kernel)", f"{cfg} {h}x{w} packed u32",
                h * w, 0.25, us, us1, {"ok": ok, "oracle": "oracle/scan.c"},
                "be_scan_edges (Edge(p) per pixel, SPEC:183-191)")


ROWS = {"f1_c3": lambda: f1("c3"), "f1_c4": lambda: f1("c4"), "f2_c2": lambda: f2("c2"),
        "f2_c5": lambda: f2("c5"), "f3_c3": lambda: f3("c3"), "f3_c5": lambda: f3("c5"),
        "f4_c3": lambda: f4("c3")}

if __name__ == "__main__":
    out = sys.argv[1] if len(sys.argv) > 1 and sys.argv[1].endswith(".json") else None
    sel = [a for a in sys.argv[1:] if a in ROWS] or list(ROWS)
    res = []
    for r in sel:
        d = ROWS[r]()
        d["id"] = r
        res.append(d)
        print(json.dumps(d), flush=True)
        torch.cuda.empty_cache()
    if out:
        with open(out, "w") as f:
            json.dump({"device": torch.cuda.get_device_name(0), "rows": res}, f, indent=1)

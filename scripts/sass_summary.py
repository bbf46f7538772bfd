"""Per-kernel SASS instruction-class summary of libbitedge_cuda.so (cuobjdump
-sass; no GPU needed): the evidence that the hot kernels use Blackwell's
256-bit global accesses (LDG.E.*.256 / STG.E.*.256), TMA bulk copies (UBLKCP)
with mbarriers (SYNCS), warp shuffles, and no tensor-core instructions (nothing
on this path is a contraction).

    python scripts/sass_summary.py [out.txt]
"""

import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1401_5245_b200", "lib", "libbitedge_cuda.so")

CLASSES = [
    ("LDG.256", re.compile(r"\bLDG\.E\.[A-Z0-9.]*256\b")),
    ("LDG.128", re.compile(r"\bLDG\.E\.[A-Z0-9.]*128\b")),
    ("LDG.other", re.compile(r"\bLDG\b(?!\.E\.[A-Z0-9.]*(256|128)\b)")),
    ("STG.256", re.compile(r"\bSTG\.E\.[A-Z0-9.]*256\b")),
    ("STG.128", re.compile(r"\bSTG\.E\.[A-Z0-9.]*128\b")),
    ("STG.other", re.compile(r"\bSTG\b(?!\.E\.[A-Z0-9.]*(256|128)\b)")),
    ("UBLKCP (TMA bulk)", re.compile(r"\bUBLKCP\b")),
    ("SYNCS (mbarrier)", re.compile(r"\bSYNCS\b")),
    ("SHFL", re.compile(r"\bSHFL\b")),
    ("LDS/STS", re.compile(r"\b(LDS|STS)\b")),
    ("BAR", re.compile(r"\bBAR\b")),
    ("tensor (HMMA/UTC*MMA)", re.compile(r"\b(HMMA|IMMA|UTCHMMA|UTCQMMA|UTCIMMA|UTCOMMA)\b")),
]
HOT = [  # (label, substring of the demangled name)
    ("K1 aligned, 2-row strips (C3 packed u32)",
     "edge_reg_packed_kernel<0, 2, 8, 0, false, false, true, false, false>"),
    ("K1 aligned, 4-row strips (C4 packed u32, the headline)",
     "edge_reg_packed_kernel<0, 4, 8, 0, false, false, true, false, false>"),
    ("K3 halo (C4 row shards)", "edge_reg_packed_kernel<0, 4, 8, 0, true, false, true, false, false>"),
    ("K3e end rows of a row shard", "edge_halo_ends_kernel"),
    ("K1 H16 (16-byte rows, 8-word items)", "edge_reg_packed_kernel<0, 2, 8, 0, false, false, false, false, true>"),
    ("K1f flat (ragged packed rows)", "edge_flat_kernel<8, 0, 6, 0, false>"),
    ("K1f flat, P4 rows of whole words", "edge_flat_kernel<8, 0, 6, 0, true>"),
    ("K1p flat P4 bytes, 32-byte chunks", "p4_flat_kernel<8, 0, false>"),
    ("K1p flat P4 bytes, 16-byte chunks", "p4_flat_kernel<4, 0, true>"),
    ("K2t2 TMA ring, run-time strip height (mid-size uint8 rasters)", "edge_tma2_u8_kernel<0, 4, 0, false, false>"),
    ("K2w warp-per-image (C2 glyphs)", "edge_warp_img_kernel<1, 0, 8>"),
    ("K2t2 TMA ring (C5 pages)", "edge_tma2_u8_kernel<8, 4, 0, false, false>"),
    ("K2t2 UNAL (uint8 rows at byte offsets)", "edge_tma2_u8_kernel<8, 4, 0, false, true>"),
    ("K1s flat ring (opt-in)", "edge_flat_ring_kernel<0, 0, 11>"),
    ("K2 (uint8 -> u64 drop-in, small images)", "edge_reg_u8_kernel<4, 0, false, true, 0>"),
]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True,
                          check=True).stdout
    funcs, cur, arch = {}, None, set()
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        a = re.search(r"arch = (sm_\w+)", line)
        if a:
            arch.add(a.group(1))
        if cur and re.match(r"\s*/\*[0-9a-f]{4}\*/", line):
            funcs[cur].append(line)
    names = {}
    for mangled in funcs:
        dem = subprocess.run(["c++filt", mangled], capture_output=True, text=True).stdout.strip()
        names[mangled] = dem
    out = [f"# SASS instruction classes, {os.path.relpath(LIB, ROOT)} (archs: {sorted(arch)})",
           f"# {len(funcs)} kernels; counts are static instructions in each kernel's SASS", ""]
    total = collections.Counter()
    for mangled, lines in funcs.items():
        for label, rx in CLASSES:
            total[label] += sum(1 for l in lines if rx.search(l))
    out.append("whole library: " + ", ".join(f"{k} {v}" for k, v in total.items()))
    out.append("")
    for label, key in HOT:
        hits = [m for m, d in names.items() if key in d]
        if not hits:
            out.append(f"{label}: (not found: {key})")
            continue
        m = hits[0]
        lines = funcs[m]
        cnt = {lab: sum(1 for l in lines if rx.search(l)) for lab, rx in CLASSES}
        out.append(f"{label}\n    {names[m]}\n    {len(lines)} instructions: "
                   + ", ".join(f"{k} {v}" for k, v in cnt.items() if v))
    text = "\n".join(out) + "\n"
    print(text)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            f.write(text)


if __name__ == "__main__":
    main()

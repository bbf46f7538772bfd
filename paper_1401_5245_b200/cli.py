"""`bitedge` command line (reference: pyproject.toml:12-13 names `bitedge.cli:main`;
the module is not shipped, SPEC.md:377-438 specifies it).  A thin shell over
the device library -- SURVEY 8(f) F4:

    bitedge detect  --input a.pbm --output b.pbm [--method mask|scan] [--border white|black]
                    [--raw-output true|false]
    bitedge compare --input a.pbm [--border white|black]
    bitedge bench   [--sizes 50,100,300,1024] [--shape glyph|rect|disk|noise] [--density d]
                    [--repeats n] [--csv path]
    bitedge binarize --input a.pgm --output b.pbm (--threshold t | --otsu)
    bitedge info    --input a.pbm

Exit codes: 0 success / MATCH, 1 mismatch (compare), 2 usage or
I/O error.  Both detection methods run on the GPU: `mask` is the fused kernel,
`scan` the per-pixel Edge(p) kernel.
"""

from __future__ import annotations

import argparse
import statistics
import sys
import time

import numpy as np


class CliError(Exception):
    """Usage / I/O problem -> exit code 2."""


from .binarize import otsu_threshold  # noqa: E402,F401  (re-exported for the CLI)
from .pbm import read_pgm  # noqa: E402,F401  (imageio.read_pgm; re-exported for the CLI)


def _read(path: str) -> bytes:
    try:
        with open(path, "rb") as f:
            return f.read()
    except OSError as e:
        raise CliError(f"{path}: {e.strerror}") from None


def _write(path: str, data: bytes) -> None:
    try:
        with open(path, "wb") as f:
            f.write(data)
    except OSError as e:
        raise CliError(f"{path}: {e.strerror}") from None


def _border(name: str):
    from .bitimage import BorderPolicy

    return BorderPolicy.WHITE_OUTSIDE if name == "white" else BorderPolicy.BLACK_OUTSIDE


def _load_pbm(path: str):
    from .pbm import read_pbm

    data = _read(path)
    try:
        return read_pbm(data)
    except ValueError as e:
        raise CliError(f"{path}: {e}") from None


def _bool(s: str) -> bool:
    if s.lower() in ("true", "1", "yes"):
        return True
    if s.lower() in ("false", "0", "no"):
        return False
    raise argparse.ArgumentTypeError(f"expected true/false, got {s!r}")


# ---------------------------------------------------------------- PGM (binarize input)

# ---------------------------------------------------------------- bench shapes

def generate(shape: str, size: int, density: float, seed: int = 0) -> np.ndarray:
    """Deterministic test rasters: uint8 0/1, 1 = white."""
    rng = np.random.default_rng([seed, size])
    img = np.ones((size, size), np.uint8)
    yy, xx = np.mgrid[0:size, 0:size]
    if shape == "noise":
        img[rng.random((size, size)) < density] = 0
    elif shape == "rect":
        q = size // 4
        img[q:size - q, q:size - q] = 0
    elif shape == "disk":
        img[(xx - size // 2) ** 2 + (yy - size // 2) ** 2 <= (size // 3) ** 2] = 0
    elif shape == "glyph":
        t = max(2, size // 12)
        c = size // 2
        img[size // 6:size - size // 6, c - t:c + t] = 0          # stem
        img[c - t:c + t, size // 6:size - size // 6] = 0          # bar
        img[(xx - c) ** 2 + (yy - size // 4) ** 2 <= (size // 8) ** 2] = 0
    else:
        raise CliError(f"unknown shape {shape!r}")
    return img


# ---------------------------------------------------------------- subcommands

def cmd_detect(a) -> int:
    from .edge import detect_edges_scan
    from .pbm import detect_pbm, write_pbm

    data = _read(a.input)
    border = _border(a.border)
    try:
        if a.method == "mask":
            out = detect_pbm(data, border, raw=a.raw_output)
        else:
            img = _load_pbm(a.input)
            out = write_pbm(detect_edges_scan(img, border), a.raw_output)
    except ValueError as e:
        raise CliError(f"{a.input}: {e}") from None
    _write(a.output, out)
    return 0


def cmd_compare(a) -> int:
    from .bitimage import first_difference
    from .edge import detect_edges_mask, detect_edges_scan

    img = _load_pbm(a.input)
    border = _border(a.border)
    m, s = detect_edges_mask(img, border), detect_edges_scan(img, border)
    diff = first_difference(m, s)
    if diff is None:
        print("MATCH")
        return 0
    print(f"MISMATCH at x={diff[0]} y={diff[1]}")
    return 1


def cmd_info(a) -> int:
    img = _load_pbm(a.input)
    print(f"{img.width}x{img.height} black={img.count_black()}")
    return 0


def cmd_binarize(a) -> int:
    from .binarize import threshold
    from .pbm import write_pbm

    if (a.threshold is None) == (not a.otsu):
        raise CliError("exactly one of --threshold / --otsu is required")
    try:
        gray = read_pgm(_read(a.input))
    except ValueError as e:
        raise CliError(f"{a.input}: {e}") from None
    t = a.threshold
    if a.otsu:
        t = otsu_threshold(gray)
        print(f"threshold={t}")
    elif not 0 <= t <= 255:
        raise CliError("--threshold must be in 0..255")
    _write(a.output, write_pbm(threshold(gray, t), raw=True))
    return 0


def cmd_bench(a) -> int:
    import torch

    from .bitimage import BitImage, first_difference
    from .edge import detect_edges_mask, detect_edges_scan

    if a.repeats < 3:
        raise CliError("--repeats must be >= 3 (SPEC.md:344)")
    try:
        sizes = [int(s) for s in a.sizes.split(",")]
    except ValueError:
        raise CliError(f"bad --sizes {a.sizes!r}") from None
    if any(s < 8 for s in sizes):
        raise CliError("sizes must be >= 8")
    rows = []
    for n in sorted(sizes):
        img = BitImage.from_array(generate(a.shape, n, a.density))
        m, s = detect_edges_mask(img), detect_edges_scan(img)
        d = first_difference(m, s)
        if d is not None:           # never publish a speed for a wrong answer
            print(f"methods disagree at {d}", file=sys.stderr)
            return 1

        def timed(fn):
            fn(img)
            torch.cuda.synchronize()
            ts = []
            for _ in range(a.repeats):
                t0 = time.perf_counter()
                fn(img)
                torch.cuda.synchronize()
                ts.append((time.perf_counter() - t0) * 1e3)
            return statistics.median(ts)

        scan_ms, mask_ms = timed(detect_edges_scan), timed(detect_edges_mask)
        rows.append((f"{a.shape}{n}", n, n, scan_ms, mask_ms, scan_ms / mask_ms, a.repeats))
    lines = ["label,width,height,scan_ms,mask_ms,speedup,repeats"]
    lines += [f"{r[0]},{r[1]},{r[2]},{r[3]:.4g},{r[4]:.4g},{r[5]:.3g},{r[6]}" for r in rows]
    print(f"{'image':>12} {'size':>11} {'scan ms':>9} {'mask ms':>9} {'speedup':>8}")
    for r in rows:
        print(f"{r[0]:>12} {r[1]:>5}x{r[2]:<5} {r[3]:9.4f} {r[4]:9.4f} {r[5]:8.2f}")
    if a.csv:
        _write(a.csv, ("\n".join(lines) + "\n").encode())
    return 0


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="bitedge", description=__doc__.split("\n")[0])
    sub = p.add_subparsers(dest="cmd", required=True)
    d = sub.add_parser("detect")
    d.add_argument("--input", required=True)
    d.add_argument("--output", required=True)
    d.add_argument("--method", choices=["mask", "scan"], default="mask")
    d.add_argument("--border", choices=["white", "black"], default="white")
    d.add_argument("--raw-output", type=_bool, default=True)
    c = sub.add_parser("compare")
    c.add_argument("--input", required=True)
    c.add_argument("--border", choices=["white", "black"], default="white")
    b = sub.add_parser("bench")
    b.add_argument("--sizes", default="50,100,300,1024")
    b.add_argument("--shape", choices=["glyph", "rect", "disk", "noise"], default="glyph")
    b.add_argument("--density", type=float, default=0.5)
    b.add_argument("--repeats", type=int, default=5)
    b.add_argument("--csv")
    z = sub.add_parser("binarize")
    z.add_argument("--input", required=True)
    z.add_argument("--output", required=True)
    z.add_argument("--threshold", type=int)
    z.add_argument("--otsu", action="store_true")
    i = sub.add_parser("info")
    i.add_argument("--input", required=True)
    return p


def main(argv=None) -> int:
    a = build_parser().parse_args(argv)      # argparse exits 2 on usage errors
    handlers = {"detect": cmd_detect, "compare": cmd_compare, "bench": cmd_bench,
                "binarize": cmd_binarize, "info": cmd_info}
    try:
        return handlers[a.cmd](a)
    except CliError as e:
        print(f"bitedge: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())

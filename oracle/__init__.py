"""CPU oracle for the method-of-masks edge detector -- TEST INFRASTRUCTURE ONLY.

Nothing in the product package (`paper_1401_5245_b200`, `bitedge`) may import
this package.  Only `tests/`, `__graft_entry__.smoke()` and the `cpu_baseline`
/ `--impl reference` legs of `bench.py` use it, and only as the checker or as
the timed CPU baseline -- never as the thing measured or shipped.

Contents
--------
port.py     numpy restatement of the reference `bitedge.bitimage` word ops
            (`/root/reference/pkg/src/bitedge/bitimage.py`) plus SPEC's `edge`
            composition, which the reference does not ship.
scan.c      plain-C restatement of the same two algorithms (word-level mask
            method on uint64 words and the paper's per-pixel Edge(p) scan),
            used where numpy is too slow (full-size C4/C5 parity).
cscan.py    ctypes loader for the compiled scan.c (`oracle/_build/liboracle.so`).
make_golden.py
            imports the REAL reference from /root/reference (in the build
            container only) and writes `tests/golden/*.npz`; the fixtures pin
            this oracle (parity pinned).
"""

"""How faithful is the port as a stand-in for the reference's CPU speed?  Times
the REAL reference (loaded by path, SPEC's edge composition on its own BitImage
primitives -- as oracle/make_golden.py does) against oracle/port.py on the same
inputs, single thread, in THIS container (the reference does not exist on the
GPU box).  TEST INFRASTRUCTURE ONLY.

    python oracle/port_vs_reference.py
"""

import os
import statistics
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from oracle import port as P  # noqa: E402


def med(fn, reps):
    fn()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return statistics.median(ts)


def main():
    sys.argv = sys.argv[:1]
    from oracle import make_golden as G      # loads the reference by path

    rng = np.random.default_rng(0)
    for n, reps in ((256, 50), (2048, 9), (8192, 3)):
        a = (rng.random((n, n)) < 0.5).astype(np.uint8)
        t_ref = med(lambda: G.detect(G.BI.from_array(a), G.BP.WHITE_OUTSIDE).words, reps)
        t_port = med(lambda: P.detect_edges_mask(P.from_array(a), 1).words, reps)
        same = (G.detect(G.BI.from_array(a), G.BP.WHITE_OUTSIDE).words
                == P.detect_edges_mask(P.from_array(a), 1).words).all()
        print(f"{n}^2: reference {t_ref * 1e3:.3f} ms, port {t_port * 1e3:.3f} ms, "
              f"port/reference time {t_port / t_ref:.2f}, identical words: {bool(same)}")


if __name__ == "__main__":
    main()

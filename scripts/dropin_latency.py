"""Per-call latency of the drop-in API (what a user of the reference `bitedge`
package sees after switching): host uint8 array -> BitImage.from_array ->
detect_edges_mask -> .words (host), against the same flow on the reference
composition (oracle/port.py, numpy, one thread); plus the device-resident call
(input image already in HBM, result left there).  Median of wall-clock reps
with a device sync, so Python/ctypes overhead is included.

    python scripts/dropin_latency.py [out.json]
"""

import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def med_ms(fn, reps):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(ts)


def main():
    import torch

    from oracle import port as P
    from paper_1401_5245_b200.bitimage import BitImage
    from paper_1401_5245_b200.cli import generate
    from paper_1401_5245_b200.edge import detect_edges_mask

    rows = []
    for n, reps, preps in ((256, 200, 50), (1024, 100, 10), (2048, 50, 5), (8192, 10, 3)):
        a = generate("glyph", n, 0.5)

        def ours_host():
            out = detect_edges_mask(BitImage.from_array(a))
            return out.words

        img = BitImage.from_array(a)
        img.device_words()                        # resident in HBM

        def ours_dev():
            detect_edges_mask(img).device_words()
            torch.cuda.synchronize()

        def ref():
            return P.detect_edges_mask(P.from_array(a)).words

        assert (ours_host() == ref()).all()
        r = {"size": n, "ours_host_ms": med_ms(ours_host, reps),
             "ours_device_resident_ms": med_ms(ours_dev, reps),
             "reference_port_ms": med_ms(ref, preps)}
        r["speedup_host"] = r["reference_port_ms"] / r["ours_host_ms"]
        rows.append(r)
        print(json.dumps(r))
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump({"device": torch.cuda.get_device_name(0), "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()

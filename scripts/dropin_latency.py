"""Per-call latency of the drop-in API (what a user of the reference `bitedge`
package sees after switching): host uint8 array -> BitImage.from_array ->
detect_edges_mask -> .words (host), against the same flow on the reference
itself (oracle/refarm.py: the unmodified bitimage.py from baseline/_ref + SPEC's
composition, numpy, one thread); plus the device-resident call (input image
already in HBM, result left there).  Median of wall-clock reps with a device
sync, so Python/ctypes overhead is included.  Sizes: 64^2 (a C2 glyph), 256^2
(the C1 image), then larger.

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


def med_us(fn, reps):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e6)
    return statistics.median(ts)


def main():
    import torch

    from oracle import refarm as RA
    from paper_1401_5245_b200 import synth
    from paper_1401_5245_b200.bitimage import BitImage
    from paper_1401_5245_b200.cli import generate
    from paper_1401_5245_b200.edge import detect_edges_mask

    R = RA.impl()
    cases = [("c2 glyph 64x64", synth.c2_images(1).numpy()[0], 4000, 2000),
             ("c1 256x256", synth.c1_image(), 3000, 1000),
             ("glyph 1024x1024", generate("glyph", 1024, 0.5), 300, 30),
             ("glyph 2048x2048", generate("glyph", 2048, 0.5), 100, 10),
             ("glyph 8192x8192", generate("glyph", 8192, 0.5), 10, 3)]
    rows = []
    for name, a, reps, preps in cases:
        def ours_host():
            return detect_edges_mask(BitImage.from_array(a)).words

        img = BitImage.from_array(a)
        img.device_words()                        # resident in HBM

        def ours_dev():
            detect_edges_mask(img).device_words()
            torch.cuda.synchronize()

        def ref():
            return R.detect(R.from_array(a)).words

        assert (ours_host() == ref()).all()
        r = {"case": name, "shape": list(a.shape), "reference_kind": R.kind,
             "ours_host_us": med_us(ours_host, reps),
             "ours_device_resident_us": med_us(ours_dev, reps),
             "reference_us": med_us(ref, preps)}
        r["speedup_host"] = r["reference_us"] / r["ours_host_us"]
        rows.append(r)
        print(json.dumps(r), flush=True)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump({"device": torch.cuda.get_device_name(0), "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()

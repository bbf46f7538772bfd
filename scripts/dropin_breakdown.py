"""Where the drop-in API's per-call time goes for small images (64^2 glyph,
256^2): each piece timed alone (wall clock, median of reps), against the
reference's own per-call time (oracle/refarm.py, one thread).

    python scripts/dropin_breakdown.py
"""

import json
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def med_us(fn, reps=3000):
    for _ in range(20):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e6)
    return round(statistics.median(ts), 2)


def main():
    import torch

    from oracle import refarm as RA
    from paper_1401_5245_b200 import _capi
    from paper_1401_5245_b200 import cuda as cu
    from paper_1401_5245_b200 import synth
    from paper_1401_5245_b200.bitimage import BitImage
    from paper_1401_5245_b200.edge import detect_edges_mask

    R = RA.impl()
    dev = torch.device("cuda", 0)
    one = torch.zeros(1, device=dev)
    side = torch.cuda.Stream(dev)
    from paper_1401_5245_b200.cli import generate

    for name, a in (("64x64", synth.c2_images(1).numpy()[0]), ("128x128", generate("glyph", 128, 0.5)),
                    ("256x256", synth.c1_image()), ("512x512", generate("glyph", 512, 0.5)),
                    ("1000x1000", generate("glyph", 1000, 0.5))):
        h, w = a.shape
        wp = -(-w // 64)
        pix = np.ascontiguousarray(a)
        st = cu._staging(h * w, h * wp * 8, 0)
        st_in, st_out = st.pin_in, st.pin_out
        words = np.empty((h, wp), dtype=np.uint64)
        f = _capi.fn("be_host_detect_u64_staged")
        stream0 = torch.cuda.current_stream(dev).cuda_stream
        dstage = torch.empty(h * w, dtype=torch.uint8, device=dev)
        args = (pix.ctypes.data, w, h, w, 1, 0, st_in.data_ptr(), st_in.numel(),
                st_out.data_ptr(), st_out.numel())

        def raw_call(s=stream0):
            f(*args, None, words.ctypes.data, s)

        def raw_call_dev(s=stream0):
            f(*args, dstage.data_ptr(), words.ctypes.data, s)

        img = BitImage.from_array(a)
        row = {
            "image": name,
            "reference_per_call": med_us(lambda: R.detect(R.from_array(a)).words, 1000),
            "ours_full_dropin": med_us(lambda: detect_edges_mask(BitImage.from_array(a)).words),
            "from_array_only": med_us(lambda: BitImage.from_array(a)),
            "detect_on_pending_image": med_us(lambda: detect_edges_mask(img).words),
            "host_detect_small": med_us(lambda: cu.host_detect_small(pix, 1)),
            "ctypes_call_default_stream": med_us(raw_call),
            "ctypes_call_side_stream": med_us(lambda: raw_call(side.cuda_stream)),
            "ctypes_call_copy_engine_in": med_us(raw_call_dev),
            "torch_tiny_kernel_plus_sync": med_us(lambda: (one.add_(1), torch.cuda.synchronize())),
            "torch_sync_idle": med_us(torch.cuda.synchronize),
            "np_copy_pixels": med_us(lambda: np.array(a, copy=True)),
        }
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()

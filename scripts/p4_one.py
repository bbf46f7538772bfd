"""One ragged P4 raster through detect_p4 a few times (for ncu captures)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_5245_b200 import pbm  # noqa: E402

h = w = int(sys.argv[1]) if len(sys.argv) > 1 else 8000
rb = (w + 7) // 8
x = torch.randint(0, 256, (h * rb,), dtype=torch.uint8, device="cuda")
o = torch.empty_like(x)
for _ in range(5):
    pbm.detect_p4(x, 1, h, w, out=o)
torch.cuda.synchronize()
print("ok")

"""One packed raster of a given width through edges_packed a few times (ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_5245_b200 import cuda as cu  # noqa: E402

h = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
w = int(sys.argv[2]) if len(sys.argv) > 2 else 8000
wp = -(-w // 32)
x = torch.randint(-2**31, 2**31 - 1, (h, wp), dtype=torch.int64, device="cuda").to(torch.int32)
o = torch.empty_like(x)
for _ in range(5):
    cu.edges_packed(x, w, 1, out=o)
torch.cuda.synchronize()
print("ok")

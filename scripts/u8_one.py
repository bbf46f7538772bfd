"""One uint8 batch through pack_edges_u8 a few times (for ncu captures):
u8_one.py H W [N]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_5245_b200 import cuda as cu  # noqa: E402

h = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
w = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
n = int(sys.argv[3]) if len(sys.argv) > 3 else 1
x = torch.randint(0, 2, (n, h, w), dtype=torch.uint8, device="cuda")
o = torch.empty((n, h, (w + 31) // 32), dtype=torch.int32, device="cuda")
for _ in range(5):
    cu.pack_edges_u8(x, 1, out=o)
torch.cuda.synchronize()
print("ok")

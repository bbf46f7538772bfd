import sys, torch
sys.path.insert(0, ".")
from paper_1401_5245_b200 import cuda as cu, synth
from paper_1401_5245_b200.bitimage import BitImage
from paper_1401_5245_b200.edge import detect_edges_mask
pages = synth.c5_pages(256, device="cuda")
def t(fn, n=10):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3
px = pages.numel()
for name, fn in [("pack u32", lambda: cu.pack_u8(pages, word_bits=32)),
                 ("pack u64", lambda: cu.pack_u8(pages, word_bits=64)),
                 ("pack+edges u32 (K2t2)", lambda: cu.pack_edges_u8(pages, 1)),
                 ("pack_and_edges u64 (drop-in fused)", lambda: cu.pack_and_edges(pages, 1, word_bits=64))]:
    us = t(fn)
    print(f"{name}: {us:.1f} us, {px * 1.125 / us / 1e3:.0f} GB/s alg (1.125 B/px)")
img = pages[0]
print("drop-in from_array(cuda) + detect, 2048^2:", round(t(lambda: detect_edges_mask(BitImage.from_array(img)), 50), 1), "us")

"""Register / spill budget of the hot kernels, read from the ptxas report the
build writes (paper_1401_5245_b200/lib/ptxas.log).  Occupancy is what these
streaming kernels live on: e.g. K1's 2-row C3 variant at 57 registers fits 4
CTAs/SM and all 512 CTAs of an 8192^2 raster in one wave; an innocuous-looking
__launch_bounds__ change once pushed it to 71 registers (3 CTAs/SM, 1.15
waves) and cost C3 9 %.  CPU-only: no GPU needed."""

import os
import re

import pytest

LOG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_1401_5245_b200", "lib", "ptxas.log")

# mangled-name fragment -> max registers (the hot path's kernels at the BASELINE configs)
BUDGET = {
    "edge_reg_packed_kernelILi0ELi2ELi8ELi0ELb0ELb0E": 64,   # C3: K1 2-row, 8-word items
    "edge_reg_packed_kernelILi0ELi4ELi8ELi0ELb0ELb0E": 80,   # C4: K1 4-row, 8-word items
    "edge_reg_packed_kernelILi0ELi2ELi8ELi0ELb0ELb0ELb1E": 48,   # C3 tail-free: 5 CTAs/SM
    "edge_reg_packed_kernelILi0ELi4ELi8ELi0ELb0ELb0ELb1E": 72,   # C4 tail-free
    "edge_warp_img_kernelILi1ELi0ELi8E": 80,                 # C2: K2w, 64-px rows
    "edge_tma2_u8_kernelILi8ELi4ELi0ELb0E": 80,             # C5: K2t2 (smem caps it at 3 CTAs/SM)
    "edge_reg_packed_kernelILi0ELi4ELi8ELi0ELb0ELb1E": 80,   # F1: P4 4-row
    "edge_reg_packed_kernelILi0ELi2ELi8ELi0ELb0ELb1E": 64,   # F1: P4 2-row
}


def _report():
    if not os.path.exists(LOG):
        pytest.skip("no ptxas.log (library not built here)")
    text = open(LOG).read()
    out = {}
    for m in re.finditer(r"Compiling entry function '([^']+)'.*?\n(?:.*\n){0,3}?.*?"
                         r"(\d+) bytes spill stores, (\d+) bytes spill loads\n.*?Used (\d+) registers",
                         text):
        out[m.group(1)] = (int(m.group(4)), int(m.group(2)), int(m.group(3)))
    return out


@pytest.mark.parametrize("frag,budget", sorted(BUDGET.items()))
def test_hot_kernel_register_budget(frag, budget):
    rep = _report()
    hits = {k: v for k, v in rep.items() if frag in k}
    assert hits, f"kernel {frag} not in the ptxas report"
    for name, (regs, st, ld) in hits.items():
        assert regs <= budget, (name, regs, budget)
        assert st == 0 and ld == 0, (name, "spills", st, ld)


# SASS size budget (instructions incl. NOPs, `cuobjdump -sass`): K2t2 once grew
# from 1.8k to 3.7k instructions when a second inlined threshold variant got
# unrolled into every row of its strip loop, and C5 lost 47 % to instruction-
# cache misses (676 -> 994 us) with no change in registers.
SASS_BUDGET = {
    # K1, tail-free (w % 256 == 0) variants: C3, C4, C4 row slabs, P4 (F1)
    "_ZN7bitedge22edge_reg_packed_kernelILi0ELi2ELi8ELi0ELb0ELb0ELb1ELb0ELb0EEEvNS_9RegParamsENS_5K1DivE": 500,
    "_ZN7bitedge22edge_reg_packed_kernelILi0ELi4ELi8ELi0ELb0ELb0ELb1ELb0ELb0EEEvNS_9RegParamsENS_5K1DivE": 800,
    "_ZN7bitedge22edge_reg_packed_kernelILi0ELi4ELi8ELi0ELb1ELb0ELb1ELb0ELb0EEEvNS_9RegParamsENS_5K1DivE": 800,
    "_ZN7bitedge22edge_reg_packed_kernelILi0ELi4ELi8ELi0ELb0ELb1ELb1ELb0ELb0EEEvNS_9RegParamsENS_5K1DivE": 850,
    # K1 general (ragged widths)
    "_ZN7bitedge22edge_reg_packed_kernelILi0ELi2ELi8ELi0ELb0ELb0ELb0ELb0ELb0EEEvNS_9RegParamsENS_5K1DivE": 950,
    "_ZN7bitedge22edge_reg_packed_kernelILi0ELi4ELi8ELi0ELb0ELb0ELb0ELb0ELb0EEEvNS_9RegParamsENS_5K1DivE": 1450,
    "_ZN7bitedge20edge_warp_img_kernelILi1ELi0ELi8EEEvNS_9RegParamsEil": 1550,
    "_ZN7bitedge19edge_tma2_u8_kernelILi8ELi4ELi0ELb0ELb0EEEvNS_9RegParamsEll": 2800,
    "_ZN7bitedge19edge_tma2_u8_kernelILi8ELi4ELi0ELb0ELb1EEEvNS_9RegParamsEll": 3300,   # UNAL rows
}


@pytest.mark.parametrize("fn,budget", sorted(SASS_BUDGET.items()))
def test_hot_kernel_code_size(fn, budget):
    import shutil
    import subprocess

    so = os.path.join(os.path.dirname(LOG), "libbitedge_cuda.so")
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(so) or not os.path.exists(tool):
        pytest.skip("library or cuobjdump missing")
    out = subprocess.run([tool, "-sass", "-fun", fn, so], capture_output=True, text=True).stdout
    n = len(re.findall(r"^\s+/\*[0-9a-f]{4}\*/", out, flags=re.M))
    assert n > 0, f"{fn} not found"
    assert n <= budget, (fn, n, budget)

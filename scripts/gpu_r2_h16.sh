# Round 2: K1 H16 (8-word items from 16-byte rows): parity + widths.
set -u
mkdir -p gpurun_out/h16c
timeout -k 10 900 python -m pytest tests/test_gpu_variants.py -q -x -p no:cacheprovider > gpurun_out/h16c/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/h16c/pytest.log
timeout -k 10 300 python scripts/k1_widths.py > gpurun_out/h16c/k1w.log 2>&1
BITEDGE_NO_H16=1 timeout -k 10 300 python scripts/k1_widths.py > gpurun_out/h16c/k1w_noh16.log 2>&1
echo done

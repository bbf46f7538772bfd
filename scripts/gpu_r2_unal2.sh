# Round 2: K2 UNAL 2-row strips for small rasters; K2t2 UNAL forced at medium sizes (data point).
set -u
mkdir -p gpurun_out/un3
timeout -k 10 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/un3/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/un3/pytest.log
timeout -k 10 600 python scripts/u8_widths.py > gpurun_out/un3/u8w.log 2>&1

echo done

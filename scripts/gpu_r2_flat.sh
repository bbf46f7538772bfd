set -u
mkdir -p gpurun_out/f
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/f/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f/pytest.log
timeout 600 python scripts/k1_widths.py > gpurun_out/f/k1w.log 2>&1
BITEDGE_NO_FLAT=1 timeout 600 python scripts/k1_widths.py > gpurun_out/f/k1w_noflat.log 2>&1

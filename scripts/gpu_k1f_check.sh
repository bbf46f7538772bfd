set -u
mkdir -p gpurun_out/k1f
timeout -k 10 900 python -m pytest tests/test_gpu_flat.py tests/test_gpu_fuzz.py tests/test_gpu_guards.py -q -m gpu -p no:cacheprovider -rf -x > gpurun_out/k1f/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/k1f/pytest.log
timeout -k 10 300 python scripts/k1_widths.py > gpurun_out/k1f/k1w.log 2>&1
echo done

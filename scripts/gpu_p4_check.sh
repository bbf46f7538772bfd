set -u
mkdir -p gpurun_out/p4d
timeout -k 10 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py tests/test_gpu_guards.py -q -m gpu -p no:cacheprovider -k "p4 or P4" -rf > gpurun_out/p4d/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/p4d/pytest.log
timeout -k 10 600 python scripts/p4_flat_bench.py gpurun_out/p4d/p4_flat.txt > gpurun_out/p4d/bench.log 2>&1
echo done

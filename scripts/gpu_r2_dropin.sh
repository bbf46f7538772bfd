# Drop-in per-call flow: tests + latency table + the C1/C2 bench lines (which carry e2e.dropin).
set -u
mkdir -p gpurun_out/r2d
timeout 600 python -m pytest tests/test_gpu_dropin.py tests/test_gpu_strided.py -q -x > gpurun_out/r2d/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2d/pytest.log
timeout 600 python scripts/dropin_latency.py gpurun_out/r2d/dropin.json > gpurun_out/r2d/dropin.log 2>&1; echo "rc=$?" >> gpurun_out/r2d/dropin.log
timeout 600 python bench.py --config c2 --steps 2000 --warmup 5 > gpurun_out/r2d/c2.json 2> gpurun_out/r2d/c2.err
timeout 600 python bench.py --config c1 --steps 2000 --warmup 5 > gpurun_out/r2d/c1.json 2> gpurun_out/r2d/c1.err

set -u
timeout 600 python -m pytest tests/test_gpu_dropin.py tests/test_gpu_strided.py tests/test_gpu_parity.py -q -x > gpurun_out/d2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/d2_pytest.log
timeout 600 python scripts/dropin_breakdown.py > gpurun_out/d2_bd.log 2>&1
timeout 600 python scripts/dropin_latency.py gpurun_out/d2_dropin.json > gpurun_out/d2_dropin.log 2>&1

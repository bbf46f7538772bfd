# Round 2: P4 byte kernel with lane-realigned stores: parity + ragged P4 bench.
set -u
mkdir -p gpurun_out/p4
timeout -k 10 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_cli.py -q -x -p no:cacheprovider > gpurun_out/p4/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/p4/pytest.log
timeout -k 10 600 python scripts/p4_ragged_bench.py > gpurun_out/p4/p4r.log 2>&1
echo done

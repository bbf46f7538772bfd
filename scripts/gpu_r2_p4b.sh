# Round 2: K1p (flat P4 kernel): parity + ragged P4 bench, against the previous dispatch.
set -u
mkdir -p gpurun_out/p4b
timeout -k 10 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_cli.py -q -x -p no:cacheprovider > gpurun_out/p4b/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/p4b/pytest.log
timeout -k 10 600 python scripts/p4_ragged_bench.py > gpurun_out/p4b/p4r.log 2>&1
BITEDGE_P4_NO_FLAT=1 timeout -k 10 600 python scripts/p4_ragged_bench.py > gpurun_out/p4b/p4r_noflat.log 2>&1
echo done

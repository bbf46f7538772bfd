# Round 2: K1p restricted to byte-granular rows <= 48 MiB: parity + ragged P4 bench (flat vs byte kernel).
set -u
mkdir -p gpurun_out/p4c
timeout -k 10 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "p4 or P4" > gpurun_out/p4c/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/p4c/pytest.log
timeout -k 10 600 python scripts/p4_ragged_bench.py > gpurun_out/p4c/p4r.log 2>&1
BITEDGE_P4_NO_FLAT=1 timeout -k 10 600 python scripts/p4_ragged_bench.py > gpurun_out/p4c/p4r_noflat.log 2>&1
echo done

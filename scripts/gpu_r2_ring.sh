# Round 2: K1s (flat span through a per-warp smem ring) parity + widths + ncu.
set -u
mkdir -p gpurun_out/ring2
timeout -k 10 900 python -m pytest tests/test_gpu_flat.py tests/test_gpu_variants.py tests/test_gpu_fuzz.py tests/test_gpu_guards.py tests/test_gpu_strided.py tests/test_gpu_dropin.py -q -x -p no:cacheprovider > gpurun_out/ring2/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ring2/pytest.log
timeout -k 10 300 python scripts/k1_widths.py > gpurun_out/ring2/k1w.log 2>&1
BITEDGE_NO_RING=1 timeout -k 10 300 python scripts/k1_widths.py > gpurun_out/ring2/k1w_noring.log 2>&1
timeout -k 10 120 python scripts/k1_one.py 8192 8000 > gpurun_out/ring2/plain.log 2>&1 && \
timeout -k 10 300 ncu --set full --clock-control none --import-source on -k regex:edge_ -s 3 -c 1 -o gpurun_out/ring2/k1s -f python scripts/k1_one.py 8192 8000 > gpurun_out/ring2/ncu.log 2>&1
echo done

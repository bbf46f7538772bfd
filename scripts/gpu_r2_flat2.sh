# Round 2: K1f v2 (30 output lanes per warp, 40 registers): parity, widths, ncu.
set -u
mkdir -p gpurun_out/f3
timeout -k 10 600 python -m pytest tests/test_gpu_flat.py tests/test_gpu_variants.py tests/test_gpu_fuzz.py tests/test_gpu_guards.py -q -x -p no:cacheprovider > gpurun_out/f3/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/f3/pytest.log
timeout -k 10 300 python scripts/k1_widths.py > gpurun_out/f3/k1w.log 2>&1


timeout -k 10 120 python scripts/k1_one.py 8192 8000 > gpurun_out/f3/k1f_plain.log 2>&1 && \
timeout -k 10 300 ncu --set full --clock-control none --import-source on -k regex:edge_ -s 3 -c 1 -o gpurun_out/f3/k1f -f python scripts/k1_one.py 8192 8000 > gpurun_out/f3/ncu_k1f.log 2>&1
echo done

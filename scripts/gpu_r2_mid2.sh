set -u
mkdir -p gpurun_out/mid
timeout -k 10 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_unal_tma.py tests/test_gpu_fuzz.py -q -m gpu -p no:cacheprovider -rf -x > gpurun_out/mid/pytest2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/mid/pytest2.log
timeout -k 10 300 python scripts/u8_widths.py > gpurun_out/mid/u8w.log 2>&1
echo done

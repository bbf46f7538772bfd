set -u
mkdir -p gpurun_out/mid
timeout -k 10 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -rf -x > gpurun_out/mid/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/mid/pytest.log
timeout -k 10 600 python bench.py --config c5 --gpus 1 --steps 20 --warmup 5 > gpurun_out/mid/bench_c5.json 2> gpurun_out/mid/bench_c5.err
timeout -k 10 300 python scripts/u8_widths.py > gpurun_out/mid/u8w.log 2>&1
echo done

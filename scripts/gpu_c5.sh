set -u
mkdir -p gpurun_out/c5
timeout 600 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_variants.py tests/test_gpu_parity.py -q -x > gpurun_out/c5/pt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c5/pt.log
timeout 300 python bench.py --config c5 --no-cpu > gpurun_out/c5/bench.json 2> gpurun_out/c5/bench.err
KB_NOGRAPH=6 timeout 300 python scripts/kbench.py c5 > gpurun_out/c5/kb.log 2>&1 && \
KB_NOGRAPH=6 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:edge_ -s 2 -c 3 --csv python scripts/kbench.py c5 > gpurun_out/c5/ncu.csv 2>&1

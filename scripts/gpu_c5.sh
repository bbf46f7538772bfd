# C5 check: parity suites, the c5 bench line, and per-launch DRAM bytes of the
# top kernel (set EXTRA_ENV, e.g. "BITEDGE_TMA1=1", to steer the dispatch).
set -u
mkdir -p gpurun_out/c5
timeout 600 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_variants.py tests/test_gpu_parity.py -q -x > gpurun_out/c5/pt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c5/pt.log
env ${EXTRA_ENV:-} timeout 300 python bench.py --config c5 --no-cpu > gpurun_out/c5/bench.json 2> gpurun_out/c5/bench.err
env ${EXTRA_ENV:-} KB_NOGRAPH=6 timeout 300 python scripts/kbench.py c5 > gpurun_out/c5/kb.log 2>&1 && \
env ${EXTRA_ENV:-} KB_NOGRAPH=6 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:edge_ -s 2 -c 3 --csv python scripts/kbench.py c5 > gpurun_out/c5/ncu.csv 2>&1

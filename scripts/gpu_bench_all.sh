#!/bin/bash
# Every config through bench.py (ours) plus the reference arm for the default workload.
set -u
mkdir -p gpurun_out/bench
for c in ${CONFIGS:-c1 c2 c3 c4 c5}; do
  timeout 900 python bench.py --config $c > gpurun_out/bench/ours_$c.json 2> gpurun_out/bench/ours_$c.err
done
timeout 900 python bench.py --impl reference --config c2 --steps 5 --warmup 3 > gpurun_out/bench/ref_c2.json 2> gpurun_out/bench/ref_c2.err
nproc > gpurun_out/bench/host.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/bench/host.txt

#!/bin/bash
# ncu launch list (duration + DRAM bytes) for each config via scripts/kbench.py, plus
# optional full captures (FULL="c5 ...").
set -u
mkdir -p gpurun_out
for c in ${CONFIGS:-c1 c2 c3 c4 c5}; do
  CMD="python scripts/kbench.py $c"
  KB_NOGRAPH=6 $CMD > gpurun_out/kl_plain_$c.log 2>&1 || { echo "plain $c failed"; continue; }
  KB_NOGRAPH=6 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__registers_per_thread \
     --clock-control none -k regex:edge_ -s 3 -c 3 --csv --log-file gpurun_out/kl_$c.csv $CMD > /dev/null 2>&1
done
for c in ${FULL:-}; do
  KB_NOGRAPH=6 ncu --set full --clock-control none --import-source on -k regex:edge_ -s 4 -c 1 \
      -o gpurun_out/kf_$c -f python scripts/kbench.py $c > gpurun_out/kf_$c.log 2>&1
done

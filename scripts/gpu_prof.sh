#!/bin/bash
# ncu launch lists + one full capture per config.  Output under gpurun_out/.
# Every ncu command runs only after the identical plain command exited 0.
set -u
mkdir -p gpurun_out
for c in ${CONFIGS:-c2 c3}; do
  CMD="python bench.py --config $c --steps ${STEPS:-30} --warmup 3 --no-e2e --no-cpu --no-check --no-graph"
  $CMD > gpurun_out/plain_$c.log 2>&1 || { echo "plain $c failed"; continue; }
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:${KREGEX:-edge_tile} -s 5 -c 10 --csv --log-file gpurun_out/launches_$c.csv $CMD \
      > gpurun_out/ncu_l_$c.log 2>&1
  if [ -z "${NOFULL:-}" ]; then
    ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-edge_tile} -s 8 -c 1 \
        -o gpurun_out/prof_$c -f $CMD > gpurun_out/ncu_f_$c.log 2>&1
  fi
done

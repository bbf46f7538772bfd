#!/bin/bash
# Full ncu capture of one launch per (config, kernel variant) using scripts/kbench.py.
set -u
mkdir -p gpurun_out
for c in ${CONFIGS:-c4}; do
  for kv in ${VARIANTS:-auto tile}; do
    CMD="python scripts/kbench.py $c"
    KB_NOGRAPH=6 BITEDGE_KERNEL=$kv $CMD > gpurun_out/kp_plain_${c}_$kv.log 2>&1 || { echo "plain $c $kv failed"; continue; }
    KB_NOGRAPH=6 BITEDGE_KERNEL=$kv ncu --set full --clock-control none --import-source on -k regex:edge_ -s 4 -c 1 \
        -o gpurun_out/kp_${c}_$kv -f $CMD > gpurun_out/kp_ncu_${c}_$kv.log 2>&1
  done
done

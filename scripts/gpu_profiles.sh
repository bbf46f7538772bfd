#!/bin/bash
# Round profiling pass (one gpurun call): the bench launch list + one full ncu
# capture of the top kernel per config.  Every ncu command follows the same
# command run plainly with exit 0.  Results land in gpurun_out/prof/.
set -u
mkdir -p gpurun_out/prof
LCFG=${LAUNCH_CFG:-c4}
BENCH="python bench.py --config $LCFG --steps ${LAUNCH_STEPS:-20} --warmup 5 --no-cpu --no-e2e --no-dropin"
$BENCH > gpurun_out/prof/bench_plain.json 2> gpurun_out/prof/bench_plain.err && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:edge_ -c 400 --csv --log-file gpurun_out/prof/launches_bench_$LCFG.csv $BENCH > /dev/null 2>&1
for c in ${CONFIGS:-c1 c2 c3 c4 c5}; do
  CMD="python scripts/kbench.py $c"
  KB_NOGRAPH=6 $CMD > gpurun_out/prof/plain_$c.log 2>&1 || { echo "plain $c failed"; continue; }
  KB_NOGRAPH=6 ncu --set full --clock-control none --import-source on -k regex:edge_ -s 4 -c 1 \
      -o gpurun_out/prof/full_$c -f $CMD > gpurun_out/prof/ncu_full_$c.log 2>&1
done
# summarise on the box (ncu -i is here too) so only small files need to travel back
LAUNCH_CFG=$LCFG LAUNCH_CMD="$BENCH" PROF_DST=gpurun_out/prof/summary python scripts/summarize_profiles.py ${TAG:-r1} > /dev/null 2>&1
ls -la gpurun_out/prof > gpurun_out/prof/ls.txt
for r in gpurun_out/prof/full_c*.ncu-rep; do [ "$(stat -c %s $r)" -gt 12000000 ] && rm -f $r; done
true

# One ncu --set full capture (with SASS source counters) of the hot kernel per
# config in $CONFIGS via scripts/kbench.py.  Output: gpurun_out/src/kp_<cfg>.ncu-rep
set -u
mkdir -p gpurun_out/src
for c in ${CONFIGS:-c2 c5}; do
  KB_NOGRAPH=6 ncu --set full --clock-control none --import-source on -k regex:edge_ -s 4 -c 1 \
      -o gpurun_out/src/kp_$c -f python scripts/kbench.py $c > gpurun_out/src/ncu_$c.log 2>&1
done

# ncu captures of the uint8 kernel on two shapes: A="H W N" B="H W N"; the raw-page
# CSV travels back (the .ncu-rep files are tens of MB each)
set -u
mkdir -p gpurun_out/pu
i=0
for s in "${A:-4096 4096 1}" "${B:-}"; do
  [ -z "$s" ] && continue
  python scripts/u8_one.py $s > gpurun_out/pu/plain_$i.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:edge_ -s 3 -c 1 -o /tmp/k2_$i -f python scripts/u8_one.py $s > gpurun_out/pu/ncu_$i.log 2>&1
  ncu -i /tmp/k2_$i.ncu-rep --page raw --csv > gpurun_out/pu/k2_$i.csv 2>/dev/null
  i=$((i+1))
done

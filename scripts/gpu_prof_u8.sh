set -u
mkdir -p gpurun_out/pu
python scripts/u8_one.py 4096 4096 > gpurun_out/pu/plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:edge_ -s 3 -c 1 -o gpurun_out/pu/k2 -f python scripts/u8_one.py 4096 4096 > gpurun_out/pu/ncu1.log 2>&1

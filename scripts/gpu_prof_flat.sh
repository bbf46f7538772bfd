set -u
mkdir -p gpurun_out/pf
python scripts/k1_one.py 8192 8000 > gpurun_out/pf/plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:edge_ -s 3 -c 1 -o gpurun_out/pf/flat -f python scripts/k1_one.py 8192 8000 > gpurun_out/pf/ncu1.log 2>&1

set -u
mkdir -p gpurun_out/p4e
timeout 300 python scripts/p4_one.py 32002 > gpurun_out/p4e/one.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:p4_flat -s 2 -c 1 -o gpurun_out/p4e/k1p -f python scripts/p4_one.py 32002 > gpurun_out/p4e/ncu.log 2>&1
echo done

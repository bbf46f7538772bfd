# Round refresh (one gpurun call): every bench line, the 8(f) rows, the ncu
# profiles, the drop-in latency table and the PCIe copy floors -> gpurun_out/
set -u
bash scripts/gpu_bench_all.sh
mkdir -p gpurun_out/bench
timeout 900 python scripts/bench_next.py gpurun_out/bench/next.json > gpurun_out/bench/next.log 2>&1
timeout 300 python scripts/dropin_latency.py gpurun_out/bench/dropin.json > gpurun_out/bench/dropin.log 2>&1
timeout 300 python scripts/e2e_floor.py > gpurun_out/bench/floor.log 2>&1
timeout 300 python scripts/p4_ragged_bench.py > gpurun_out/bench/p4_ragged.log 2>&1
TAG=${TAG:-r1} bash scripts/gpu_profiles.sh
mkdir -p gpurun_out/w
timeout 300 python scripts/k1_widths.py > gpurun_out/w/k1.txt 2>&1
timeout 300 python scripts/u8_widths.py > gpurun_out/w/u8.txt 2>&1

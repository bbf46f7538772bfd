# Round 2: ragged uint8 and P4 rows at large sizes (are the ragged paths at the peak when launch effects amortise?).
set -u
mkdir -p gpurun_out/lg
timeout -k 10 600 python scripts/u8_widths.py > gpurun_out/lg/u8w.log 2>&1
timeout -k 10 600 python scripts/p4_ragged_bench.py > gpurun_out/lg/p4r.log 2>&1
echo done

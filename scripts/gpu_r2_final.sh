# Round 2 refresh in one call: smoke, the whole GPU suite, every config's bench line
# (20 steps, as the driver runs them; the default line = C4) and the reference arm,
# widths + drop-in tables, then the profiling pass (launch list of the default bench,
# one full ncu capture per config).  Results: gpurun_out/fin/ and gpurun_out/prof/.
set -u
mkdir -p gpurun_out/fin
leftovers() { nvidia-smi --query-compute-apps=pid --format=csv,noheader 2>/dev/null | while read p; do [ -n "$p" ] && kill -9 "$p" 2>/dev/null && echo "killed leftover $p"; done; }
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/fin/smoke.log
timeout -k 10 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -rf > gpurun_out/fin/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/fin/pytest.log; leftovers >> gpurun_out/fin/pytest.log
timeout -k 10 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin/bench_c4.json 2> gpurun_out/fin/bench_c4.err
timeout -k 10 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin/ref_c4.json 2> gpurun_out/fin/ref_c4.err
for c in c1 c2 c3 c5; do
  timeout -k 10 900 python bench.py --config $c --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin/bench_$c.json 2> gpurun_out/fin/bench_$c.err
done
timeout -k 10 300 python scripts/k1_widths.py > gpurun_out/fin/k1w.log 2>&1
timeout -k 10 300 python scripts/u8_widths.py > gpurun_out/fin/u8w.log 2>&1
timeout -k 10 300 python scripts/u8_mid_sweep.py final > gpurun_out/fin/u8mid.log 2>&1
timeout -k 10 300 python scripts/u8_batch_sweep.py > gpurun_out/fin/u8batch.log 2>&1
U8B_SHAPES=256x1024x1024,200x960x1216,128x1024x1152,200x960x1200,64x1000x1250,48x1024x1280,40x1200x1600,64x1080x1900,1100x480x640,1024x200x300,256x500x1000 timeout -k 10 300 python scripts/u8_batch_sweep.py > gpurun_out/fin/u8batch2.log 2>&1
K1W_SHAPES=6000x6016,10000x10016,12000x11968,12288x12288,16384x16000,16384x16384,24576x24576 timeout -k 10 300 python scripts/k1_widths.py > gpurun_out/fin/k1mid.log 2>&1
timeout -k 10 300 python scripts/p4_flat_bench.py gpurun_out/fin/p4_flat.txt > gpurun_out/fin/p4_flat.log 2>&1
timeout -k 10 300 python scripts/p4_ragged_bench.py > gpurun_out/fin/p4_ragged.log 2>&1
timeout -k 10 300 python scripts/dropin_latency.py gpurun_out/fin/dropin.json > gpurun_out/fin/dropin.log 2>&1
timeout -k 10 600 python scripts/bench_next.py gpurun_out/fin/bench_next.json > gpurun_out/fin/bench_next.log 2>&1
TAG=r2 LAUNCH_CFG=c4 timeout -k 10 1800 bash scripts/gpu_profiles.sh > gpurun_out/fin/profiles.log 2>&1
echo done

# Round 2 re-entry: where HEAD stands on the GPU (suite, all bench configs, C2 K2p vs K2w, launch list).
set -u
mkdir -p gpurun_out/st
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/st/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/st/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/st/smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/st/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/st/pytest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/st/bench.json 2> gpurun_out/st/bench.err; echo "bench rc=$?" >> gpurun_out/st/bench.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/st/ref.json 2> gpurun_out/st/ref.err; echo "ref rc=$?" >> gpurun_out/st/ref.err
for c in c1 c2 c3 c5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/st/bench_$c.json 2> gpurun_out/st/bench_$c.err
done
BITEDGE_NO_K2P=1 timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-e2e --no-cpu --no-dropin > gpurun_out/st/c2_k2w.json 2> gpurun_out/st/c2_k2w.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/st/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-dropin > gpurun_out/st/ncu_c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/st/launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-e2e --no-cpu --no-dropin > gpurun_out/st/ncu_c2.log 2>&1
echo done

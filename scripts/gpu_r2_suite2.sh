# Round 2: the GPU suite in separately bounded parts (each part's stragglers killed),
# the multi-rank bench cases one by one with their stderr, widths + drop-in tables.
set -u
mkdir -p gpurun_out/s2
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s2/smoke.log
timeout -k 10 1200 python -m pytest tests -q -m gpu --ignore=tests/test_gpu_bench_multirank.py --ignore=tests/test_gpu_peer.py -p no:cacheprovider > gpurun_out/s2/pytest_main.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s2/pytest_main.log
nvidia-smi --query-compute-apps=pid,process_name,used_memory --format=csv > gpurun_out/s2/apps_after_main.txt 2>&1
for k in c2-strong c2-weak c4-rows-nccl-path; do
  timeout -k 10 400 python -m pytest "tests/test_gpu_bench_multirank.py::test_bench_two_ranks_one_gpu[$k]" -q -x > gpurun_out/s2/mr_$k.log 2>&1; echo "rc=$?" >> gpurun_out/s2/mr_$k.log
  nvidia-smi --query-compute-apps=pid,process_name,used_memory --format=csv > gpurun_out/s2/apps_after_$k.txt 2>&1
done
timeout -k 10 300 python scripts/k1_widths.py > gpurun_out/s2/k1w.log 2>&1
timeout -k 10 300 python scripts/u8_widths.py > gpurun_out/s2/u8w.log 2>&1
timeout -k 10 300 python scripts/dropin_latency.py gpurun_out/s2/dropin.json > gpurun_out/s2/dropin.log 2>&1
timeout -k 10 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu > gpurun_out/s2/bench_c2.json 2> gpurun_out/s2/bench_c2.err
timeout -k 10 300 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu > gpurun_out/s2/bench_c1.json 2> gpurun_out/s2/bench_c1.err
timeout -k 10 600 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu > gpurun_out/s2/bench_c5.json 2> gpurun_out/s2/bench_c5.err
timeout -k 10 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu > gpurun_out/s2/bench_c3.json 2> gpurun_out/s2/bench_c3.err
echo done

# Round 2: K2p fix check, the GPU suite, benches, then the multi-rank cases (last,
# each bounded; any rank left on the GPU is killed by PID afterwards).
set -u
mkdir -p gpurun_out/s3
leftovers() { nvidia-smi --query-compute-apps=pid --format=csv,noheader 2>/dev/null | while read p; do [ -n "$p" ] && kill -9 "$p" 2>/dev/null && echo "killed leftover $p"; done; }
timeout -k 10 300 python -m pytest tests/test_gpu_guards.py -q -k k2p -x > gpurun_out/s3/k2p.log 2>&1; echo "rc=$?" >> gpurun_out/s3/k2p.log; leftovers >> gpurun_out/s3/k2p.log
timeout -k 10 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu > gpurun_out/s3/bench_c2.json 2> gpurun_out/s3/bench_c2.err; echo "rc=$?" >> gpurun_out/s3/bench_c2.err
timeout -k 10 300 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu > gpurun_out/s3/bench_c1.json 2> gpurun_out/s3/bench_c1.err
timeout -k 10 300 python scripts/dropin_latency.py gpurun_out/s3/dropin.json > gpurun_out/s3/dropin.log 2>&1
timeout -k 10 900 python -m pytest tests -q -m gpu --ignore=tests/test_gpu_bench_multirank.py -p no:cacheprovider > gpurun_out/s3/pytest_main.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3/pytest_main.log; leftovers >> gpurun_out/s3/pytest_main.log
timeout -k 10 600 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu > gpurun_out/s3/bench_c5.json 2> gpurun_out/s3/bench_c5.err
timeout -k 10 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu > gpurun_out/s3/bench_c3.json 2> gpurun_out/s3/bench_c3.err
timeout -k 10 600 python bench.py > gpurun_out/s3/bench_c4.json 2> gpurun_out/s3/bench_c4.err
for k in c2-strong c2-weak c4-rows-nccl-path; do
  timeout -k 10 400 python -m pytest "tests/test_gpu_bench_multirank.py::test_bench_two_ranks_one_gpu[$k]" -q -x > gpurun_out/s3/mr_$k.log 2>&1; echo "rc=$?" >> gpurun_out/s3/mr_$k.log
  leftovers >> gpurun_out/s3/mr_$k.log
done
echo done

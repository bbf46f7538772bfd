# What the driver does at round end, in one call: smoke, the whole GPU suite
# (slow tests included), the default bench line and the reference arm.
set -u
mkdir -p gpurun_out/re
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/re/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/re/smoke.log
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/re/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/re/pytest.log
timeout 600 python bench.py > gpurun_out/re/bench.json 2> gpurun_out/re/bench.err; echo "bench rc=$?" >> gpurun_out/re/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/re/ref.json 2> gpurun_out/re/ref.err; echo "ref rc=$?" >> gpurun_out/re/ref.err

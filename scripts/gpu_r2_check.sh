# Round 2: GPU suite, the default bench line (C4) and the reference arm, as the driver runs them.
set -u
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2/smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x ${PYTEST_K:-} > gpurun_out/r2/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2/pytest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2/bench.json 2> gpurun_out/r2/bench.err; echo "bench rc=$?" >> gpurun_out/r2/bench.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2/ref.json 2> gpurun_out/r2/ref.err; echo "ref rc=$?" >> gpurun_out/r2/ref.err

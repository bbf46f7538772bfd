set -u
mkdir -p gpurun_out/k
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/k/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/k/pytest.log
timeout 300 python bench.py --config c2 --steps 20000 --warmup 10 --no-e2e --no-cpu --no-dropin > gpurun_out/k/c2.json 2> gpurun_out/k/c2.err
BITEDGE_NO_K2P=1 timeout 300 python bench.py --config c2 --steps 20000 --warmup 10 --no-e2e --no-cpu --no-dropin > gpurun_out/k/c2_k2w.json 2> gpurun_out/k/c2_k2w.err

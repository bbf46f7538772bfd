# Full GPU suite + drop-in latency table + breakdown (round 2).
set -u
mkdir -p gpurun_out/s
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s/smoke.log
timeout 1800 python -m pytest tests -q -m gpu ${PYTEST_ARGS:-} > gpurun_out/s/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s/pytest.log
timeout 600 python scripts/dropin_breakdown.py > gpurun_out/s/bd.log 2>&1
timeout 600 python scripts/dropin_latency.py gpurun_out/s/dropin.json > gpurun_out/s/dropin.log 2>&1

# Round 2: whole GPU suite (driver order, bounded), then benches (20 steps, as the driver runs them),
# the drop-in breakdown with spin vs blocking completion waits.
set -u
mkdir -p gpurun_out/s4
leftovers() { nvidia-smi --query-compute-apps=pid --format=csv,noheader 2>/dev/null | while read p; do [ -n "$p" ] && kill -9 "$p" 2>/dev/null && echo "killed leftover $p"; done; }
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s4/smoke.log
timeout -k 10 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -rf > gpurun_out/s4/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4/pytest.log; leftovers >> gpurun_out/s4/pytest.log
for c in c1 c2 c3; do
  timeout -k 10 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/s4/bench_$c.json 2> gpurun_out/s4/bench_$c.err
done
timeout -k 10 300 python scripts/dropin_breakdown.py > gpurun_out/s4/bd_spin.log 2>&1
BITEDGE_SYNC_BLOCK=1 timeout -k 10 300 python scripts/dropin_breakdown.py > gpurun_out/s4/bd_block.log 2>&1
echo done

# K1 change check: the whole GPU suite, then kernel-only timing (K1 packed, P4)
# and the C3 / C4 bench lines.  Output under gpurun_out/k1/.
set -u
mkdir -p gpurun_out/k1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/k1/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/k1/pytest.log
for s in 1 3; do KB_STREAMS=$s python scripts/kbench.py c3 c3_p4 c4 c4_p4 > gpurun_out/k1/kb_s$s.log 2>&1; done
for s in 1 3; do BITEDGE_K1_GENERIC=1 KB_STREAMS=$s python scripts/kbench.py c3 c3_p4 c4 c4_p4 > gpurun_out/k1/kbg_s$s.log 2>&1; done
for c in ${CONFIGS:-c3 c4}; do
  timeout 600 python bench.py --config $c > gpurun_out/k1/bench_$c.json 2> gpurun_out/k1/bench_$c.err
done

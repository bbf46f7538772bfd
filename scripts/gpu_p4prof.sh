# F1 (P4) kernel: parity tests, kernel-only timing next to K1 on u32 words, and
# one ncu --set full capture per format (C4).  Output under gpurun_out/p4/.
set -u
mkdir -p gpurun_out/p4
timeout 600 python -m pytest tests -m gpu -x -q -k "p4 or P4 or pbm" > gpurun_out/p4/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/p4/pytest.log
for s in 1 3; do KB_STREAMS=$s python scripts/kbench.py c3 c3_p4 c4 c4_p4 > gpurun_out/p4/kb_s$s.log 2>&1; done
if [ -z "${NO_NCU:-}" ]; then
for c in c4 c4_p4; do
  KB_NOGRAPH=6 ncu --set full --clock-control none --import-source on -k regex:edge_ -s 4 -c 1 -o gpurun_out/p4/kp_$c -f python scripts/kbench.py $c > gpurun_out/p4/ncu_$c.log 2>&1
done
fi

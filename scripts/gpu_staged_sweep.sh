set -u
for blk in 0 32 64 128; do for spin in 0 1; do
  if [ $spin = 1 ]; then export BITEDGE_STAGED_SPIN=1; else unset BITEDGE_STAGED_SPIN; fi
  BITEDGE_ZC_BLOCK=$blk BITEDGE_TRACE_STAGED=1 timeout 300 python scripts/staged_trace.py 2>&1 | grep -v "^\[staged" | head -20
  BITEDGE_ZC_BLOCK=$blk BITEDGE_TRACE_STAGED=1 timeout 300 python scripts/staged_trace.py 2>&1 | grep "^\[staged" | sort -u | head -6
done; done

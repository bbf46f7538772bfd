# C2 (K2w) dispatch knobs: overlapped and serial time per step from bench.py.
# KNOBS="name:VAR=val,VAR=val name2:..." (default: a fixed list)
set -u
mkdir -p gpurun_out/c2k
run() { name=$1; shift; env "$@" python bench.py --config c2 --no-e2e --no-cpu > gpurun_out/c2k/$name.json 2> gpurun_out/c2k/$name.err; }
for spec in ${KNOBS:-default:X=1 g4:BITEDGE_WARPIMG_G4=1 nopdl:BITEDGE_PDL=0 late:BITEDGE_PDL_LATE=1}; do
  name=${spec%%:*}; vars=${spec#*:}
  run $name ${vars//,/ }
done
for f in gpurun_out/c2k/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', round(r['avg_launch_us'],3), round(r['serial_launch_us'],3), round(r['frac'],3), round(r['frac_serial'],3))"; done

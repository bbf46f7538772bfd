# K1 (C3 / C4) knob sweep: overlapped and serial time per step from bench.py.
# KNOBS="name:VAR=val,VAR=val ..."; CONFIGS="c3 c4"
set -u
mkdir -p gpurun_out/k1k
for c in ${CONFIGS:-c3}; do
for spec in ${KNOBS:-default:X=1}; do
  name=${spec%%:*}; vars=${spec#*:}
  env ${vars//,/ } python bench.py --config $c --no-e2e --no-cpu > gpurun_out/k1k/${c}_$name.json 2> gpurun_out/k1k/${c}_$name.err
  python -c "
import json; d=json.loads(open('gpurun_out/k1k/${c}_$name.json').read().strip().splitlines()[-1]); r=d['roofline']
print('${c} $name', round(r['avg_launch_us'],3), round(r['serial_launch_us'],3), round(r['frac'],3), round(r['frac_serial'],3), d['parity']['ok'])"
done; done

#!/bin/bash
# Pre-copied record spills (A/B on C4), the transition breakdown, CPQR CTA-size experiments on C4/2.
mkdir -p gpurun_out
T=${1:-r02y}
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "record_space" > gpurun_out/${T}_rec_tests.txt 2>&1; tail -2 gpurun_out/${T}_rec_tests.txt
for v in default nt256 light; do
  case $v in default) E="";; nt256) E="HS_CQ_NT=256";; light) E="HS_CPQR_LIGHT=1";; esac
  env $E HS_CQ_LOG=1 timeout 600 python bench.py --config C4/2 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/${T}_c4h_$v.json 2> gpurun_out/${T}_c4h_$v.err
  python -c "
import json
d=json.loads(open('gpurun_out/${T}_c4h_$v.json').read().strip().splitlines()[-1]); c=d['config']
print('$v', round(d['value']), round(c['t_factor_s'],3), {k: round(v,3) for k,v in c['phase_s_per_step'].items()}, c['pcg_iters'])"
done
HS_PROFILE=1 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${T}_c4_precopy.json 2> gpurun_out/${T}_c4_precopy.err
HS_REC_PRECOPY=0 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${T}_c4_noprecopy.json 2> gpurun_out/${T}_c4_noprecopy.err
for v in precopy noprecopy; do python -c "
import json
d=json.loads(open('gpurun_out/${T}_c4_$v.json').read().strip().splitlines()[-1]); c=d['config']
print('$v', round(d['value']), round(c['t_factor_s'],3), {k: round(v,3) for k,v in c['phase_s_per_step'].items()}, c['pcg_iters'])"; done
grep "record space\|level transitions\|host planning" gpurun_out/${T}_c4_precopy.err | tail -4

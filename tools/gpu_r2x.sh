#!/bin/bash
# MR = 16 CPQR with one column in flight (no spills) vs two (HS_CQ_U2), parity of the paths that run it,
# and one ncu --set full capture of a coarse-level k_cpqr3 launch on the C4 operator (C4/2).
mkdir -p gpurun_out
T=${1:-r02x}
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "c4 or c5 or global or record or C2" > gpurun_out/${T}_tests.txt 2>&1; tail -2 gpurun_out/${T}_tests.txt
for v in u1 u2; do
  case $v in u1) E="HS_NONE=1";; u2) E="HS_CQ_U2=1";; esac
  env $E timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${T}_c4_$v.json 2> gpurun_out/${T}_c4_$v.err
  python -c "
import json
d=json.loads(open('gpurun_out/${T}_c4_$v.json').read().strip().splitlines()[-1]); c=d['config']
print('$v', round(d['value']), round(c['t_factor_s'],3), {k: round(v,3) for k,v in c['phase_s_per_step'].items()}, c['pcg_iters'])"
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_cpqr3 --launch-skip ${SKIP:-45} --launch-count 1 \
  -o gpurun_out/${T}_ncu_c4h_cpqr -f python tools/profile_run.py C4/2 > gpurun_out/${T}_ncu_c4h_cpqr.log 2>&1
python tools/ncu_summary.py gpurun_out/${T}_ncu_c4h_cpqr.ncu-rep > gpurun_out/${T}_ncu_summary.jsonl 2>&1; head -c 1500 gpurun_out/${T}_ncu_summary.jsonl

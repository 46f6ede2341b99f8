#!/bin/bash
# VMM chunk size A/B on C4 (host time of the level-transition mappings), then the full GPU suite.
mkdir -p gpurun_out
T=${1:-r02w}
for v in 256 1024; do
  HS_PROFILE=1 HS_VMM_CHUNK_MB=$v timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${T}_c4_chunk$v.json 2> gpurun_out/${T}_c4_chunk$v.err
  python -c "
import json
d=json.loads(open('gpurun_out/${T}_c4_chunk$v.json').read().strip().splitlines()[-1]); c=d['config']
print('chunk $v', round(d['value']), round(c['t_factor_s'],3), {k: round(v,3) for k,v in c['phase_s_per_step'].items()}, c['pcg_iters'])"
  grep "VMM calls\|level transitions\|record space" gpurun_out/${T}_c4_chunk$v.err | tail -3
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_gpu_tests.txt 2>&1; tail -3 gpurun_out/${T}_gpu_tests.txt

#!/bin/bash
# Round-end validation on one B200 at HEAD: full GPU suite, smoke(), the default bench line (C4, with e2e and
# cpu_baseline), and the HS_VMM_CHUNK_MB A/B the previous session left unmeasured.
mkdir -p gpurun_out
T=${1:-r02fin}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_gpu_tests.txt 2>&1; tail -3 gpurun_out/${T}_gpu_tests.txt
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -1 | tee gpurun_out/${T}_smoke.txt
timeout 1200 python bench.py > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err; head -c 400 gpurun_out/${T}_bench_c4.json; echo
for v in 256 1024; do
  HS_PROFILE=1 HS_VMM_CHUNK_MB=$v timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${T}_c4_chunk$v.json 2> gpurun_out/${T}_c4_chunk$v.err
  python -c "
import json
d=json.loads(open('gpurun_out/${T}_c4_chunk$v.json').read().strip().splitlines()[-1]); c=d['config']
print('chunk $v', round(d['value']), round(c['t_factor_s'],3), {k: round(v,3) for k,v in c['phase_s_per_step'].items()}, c['pcg_iters'])"
  grep "VMM calls\|level transitions\|record space" gpurun_out/${T}_c4_chunk$v.err | tail -3
done

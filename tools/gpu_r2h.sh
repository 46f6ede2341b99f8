#!/bin/bash
mkdir -p gpurun_out
HS_PROFILE=1 REPS=2 timeout 300 python tools/run_config.py C2 > gpurun_out/r2h_prof_c2.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --config C2 --no-cpu-baseline > gpurun_out/r2h_bench_c2.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2h_bench_c3.log 2>&1
grep "level [5678]:\|factor wall" gpurun_out/r2h_prof_c2.log | tail -6 | cut -c1-200; head -c 300 gpurun_out/r2h_bench_c2.log; echo; head -c 300 gpurun_out/r2h_bench_c3.log

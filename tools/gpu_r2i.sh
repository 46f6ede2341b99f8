#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/r2i_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/r2i_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2i_bench_c3.log 2>&1
HS_PROFILE=1 REPS=2 timeout 300 python tools/run_config.py C3 > gpurun_out/r2i_prof_c3.log 2>&1
grep -E "fullsize|passed|failed|Error|TESTS_EXIT|^E " gpurun_out/r2i_tests.log | tail -25; head -c 300 gpurun_out/r2i_bench_c3.log; echo; grep "level\|factor wall" gpurun_out/r2i_prof_c3.log | tail -14 | cut -c1-180

#!/bin/bash
# DMMA scaling (k_scale_mma) + G^{-1} from k_chol + CPQR staging: full GPU suite, benches
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/r2f_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/r2f_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_bench_c3.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --config C2 --no-cpu-baseline > gpurun_out/r2f_bench_c2.log 2>&1
HS_PROFILE=1 REPS=2 timeout 300 python tools/run_config.py C3 > gpurun_out/r2f_prof_c3.log 2>&1
grep -E "fullsize|passed|failed|Error|TESTS_EXIT" gpurun_out/r2f_tests.log | tail -20; head -c 300 gpurun_out/r2f_bench_c3.log; echo; head -c 300 gpurun_out/r2f_bench_c2.log; echo; grep "level 0:" gpurun_out/r2f_prof_c3.log | tail -1

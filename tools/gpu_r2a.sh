#!/bin/bash
# round-2 check: GPU tests under the R-coarse default, C2 bench, C4 proxy and full C4 attempt
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/r2a_tests.log
HS_PROFILE=1 timeout 300 python tools/run_config.py C2 > gpurun_out/r2a_c2.log 2>&1
HS_PROFILE=1 timeout 400 python tools/run_config.py C4/4 > gpurun_out/r2a_c4q.log 2>&1
HS_PROFILE=1 REPS=1 timeout 900 python tools/run_config.py C4 > gpurun_out/r2a_c4.log 2>&1
tail -n 3 gpurun_out/r2a_tests.log; tail -n 12 gpurun_out/r2a_c2.log; tail -n 20 gpurun_out/r2a_c4q.log; tail -n 25 gpurun_out/r2a_c4.log

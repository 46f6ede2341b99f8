#!/bin/bash
# VMM block store + C compaction: GPU tests, C2, C3, C4/2 and full C4 (R-coarse)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/r2b_tests.log
HS_PROFILE=1 REPS=1 timeout 300 python tools/run_config.py C3 > gpurun_out/r2b_c3.log 2>&1
HS_PROFILE=1 REPS=1 timeout 600 python tools/run_config.py C4/2 > gpurun_out/r2b_c4h.log 2>&1
HS_PROFILE=1 REPS=1 timeout 1500 python tools/run_config.py C4 > gpurun_out/r2b_c4.log 2>&1
tail -n 3 gpurun_out/r2b_tests.log; grep -v "^\[hs profile\] level" gpurun_out/r2b_c3.log | tail -20; tail -n 40 gpurun_out/r2b_c4h.log; tail -n 40 gpurun_out/r2b_c4.log

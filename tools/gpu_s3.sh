#!/bin/bash
# large-cluster path checks: parity on the m > 112 cases, then C2 / C4/2 profiles
mkdir -p gpurun_out
T=${1:-s3}
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -s -k "c4_operator or c5_operator or refactor" > gpurun_out/${T}_tests_big.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/${T}_tests_big.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/${T}_tests_par.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/${T}_tests_par.log
HS_PROFILE=1 REPS=2 timeout 300 python tools/run_config.py C2 > gpurun_out/${T}_prof_c2.log 2>&1
HS_PROFILE=1 REPS=1 timeout 600 python tools/run_config.py C4/2 > gpurun_out/${T}_prof_c4h.log 2>&1
grep -E "fullsize|passed|failed|Error|TESTS_EXIT" gpurun_out/${T}_tests_*.log | tail -14
grep -E "factor wall|level device|pcg" gpurun_out/${T}_prof_*.log
grep "hs profile\] level" gpurun_out/${T}_prof_c2.log | tail -5 | cut -c1-200

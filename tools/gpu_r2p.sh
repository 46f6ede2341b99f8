#!/bin/bash
mkdir -p gpurun_out
T=${1:-r2p}
nproc; python -c "import os; print(os.cpu_count(), len(os.sched_getaffinity(0)))"
HS_PROFILE=1 timeout 300 python tools/run_config.py C3 > gpurun_out/${T}_run_C3.log 2>&1
grep -E "hs profile\] (level 0|host|first)|level device" gpurun_out/${T}_run_C3.log | tail -7

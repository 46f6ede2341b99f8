#!/bin/bash
mkdir -p gpurun_out
T=${1:-r2n}
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/${T}_tests.log
tail -2 gpurun_out/${T}_tests.log
HS_PROFILE=1 timeout 300 python tools/run_config.py C3 > gpurun_out/${T}_run_C3.log 2>&1
grep -E "hs profile\] (level 0|host|first)|level device" gpurun_out/${T}_run_C3.log | tail -7
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_c3.log 2>&1
head -c 300 gpurun_out/${T}_bench_c3.log

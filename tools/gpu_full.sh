#!/bin/bash
# full GPU suite + default bench (with CPU baseline) + C2 and C4/2 bench lines
mkdir -p gpurun_out
T=${1:-full}
timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/${T}_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/${T}_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench_c3.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --config C2 --no-cpu-baseline > gpurun_out/${T}_bench_c2.log 2>&1
timeout 900 python bench.py --steps 2 --warmup 3 --config C4/2 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_c4h.log 2>&1
grep -E "fullsize|passed|failed|Error|TESTS_EXIT" gpurun_out/${T}_tests.log | tail -14; head -c 400 gpurun_out/${T}_bench_c3.log; echo; head -c 300 gpurun_out/${T}_bench_c2.log; echo; head -c 300 gpurun_out/${T}_bench_c4h.log; tail -c 300 gpurun_out/${T}_bench_c4h.log

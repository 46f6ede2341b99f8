#!/bin/bash
# session start: box facts, full GPU suite, default bench
mkdir -p gpurun_out
T=${1:-s1}
(free -g; nproc; nvidia-smi --query-gpu=name,memory.total,memory.used --format=csv) > gpurun_out/${T}_box.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/${T}_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/${T}_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench_c3.log 2>&1
cat gpurun_out/${T}_box.txt
grep -E "fullsize|passed|failed|Error|TESTS_EXIT" gpurun_out/${T}_tests.log | tail -14; head -c 600 gpurun_out/${T}_bench_c3.log

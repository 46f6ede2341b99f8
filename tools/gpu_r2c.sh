#!/bin/bash
# full GPU suite (incl. full-size parity) + default bench (C3) + C2 bench line
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -s -p no:randomly > gpurun_out/r2c_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/r2c_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2c_bench.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --config C2 --no-cpu-baseline > gpurun_out/r2c_bench_c2.log 2>&1
grep -E "fullsize|passed|failed|Error|TESTS_EXIT" gpurun_out/r2c_tests.log | tail -20; tail -c 3000 gpurun_out/r2c_bench.log; tail -c 1500 gpurun_out/r2c_bench_c2.log

#!/bin/bash
# GPU round trip used during development: smoke, -m gpu tests, C2 profile, short bench.
# usage (via gpurun): bash tools/gpu_check.sh [tests|notests] [bench|nobench]
mkdir -p gpurun_out
timeout 120 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "SMOKE $?" >> gpurun_out/smoke.log
if [ "${1:-tests}" = tests ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/gpu_tests.log
fi
HS_PROFILE=1 timeout 300 python tools/profile_run.py C2 > gpurun_out/profile_c2.log 2>&1
if [ "${2:-bench}" = bench ]; then
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
fi
tail -n 2 gpurun_out/smoke.log; tail -n 2 gpurun_out/gpu_tests.log 2>/dev/null; tail -c 600 gpurun_out/bench.log 2>/dev/null

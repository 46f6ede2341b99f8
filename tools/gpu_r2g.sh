#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -x -q -s > gpurun_out/r2g_dist.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/r2g_dist.log
tail -n 40 gpurun_out/r2g_dist.log

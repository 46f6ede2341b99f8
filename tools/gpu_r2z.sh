#!/bin/bash
# Round-2 closing measurement: full GPU suite, the default bench line (C4, CPU baseline, e2e),
# and one ncu --set full capture of a coarse-level k_cpqr3 launch on the C4 operator (C4/4).
mkdir -p gpurun_out
T=${1:-r02z}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_gpu_tests.txt 2>&1; tail -3 gpurun_out/${T}_gpu_tests.txt
timeout 1200 python bench.py > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err; tail -c 400 gpurun_out/${T}_bench_c4.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_cpqr3 --launch-skip ${SKIP:-40} --launch-count 1 \
  -o gpurun_out/${T}_ncu_c4q_cpqr -f python tools/profile_run.py C4/4 > gpurun_out/${T}_ncu_c4q_cpqr.log 2>&1
python tools/ncu_summary.py gpurun_out/${T}_ncu_c4q_cpqr.ncu-rep > gpurun_out/${T}_ncu_summary.jsonl 2>&1; head -c 1500 gpurun_out/${T}_ncu_summary.jsonl

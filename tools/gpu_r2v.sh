#!/bin/bash
mkdir -p gpurun_out
T=${1:-r2v}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/${T}_tests.log
tail -4 gpurun_out/${T}_tests.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_c3.csv python tools/one_factor_pcg.py C3 > gpurun_out/${T}_launches.log 2>&1
python tools/summarize_launches.py gpurun_out/${T}_launches_c3.csv > gpurun_out/${T}_launches_summary.txt 2>&1
head -12 gpurun_out/${T}_launches_summary.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_c3.log 2>&1
head -c 300 gpurun_out/${T}_bench_c3.log

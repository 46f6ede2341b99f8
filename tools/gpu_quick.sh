#!/bin/bash
# quick loop: parity subset, C3 bench, C3 launch list
mkdir -p gpurun_out
T=${1:-q}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "C1 or slab or q1 or small_level or 3d-24 or eps0 or pipeline_modes or repeated" > gpurun_out/${T}_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/${T}_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_c3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
  --log-file gpurun_out/${T}_launches_c3.csv python tools/one_factor_pcg.py C3 > gpurun_out/${T}_ncu_c3.log 2>&1
python tools/summarize_launches.py gpurun_out/${T}_launches_c3.csv > gpurun_out/${T}_launches_c3_summary.txt 2>&1
tail -n 2 gpurun_out/${T}_tests.log; head -c 300 gpurun_out/${T}_bench_c3.log; echo; head -14 gpurun_out/${T}_launches_c3_summary.txt

#!/bin/bash
# support-restricted level 0: bitwise identity with the dense level 0, parity, C3/C2 timings
mkdir -p gpurun_out
T=${1:-r2l}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "support_restricted or small_level or c3 or slab" > gpurun_out/${T}_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/${T}_tests.log
tail -5 gpurun_out/${T}_tests.log
for c in C3 C2; do
  HS_PROFILE=1 timeout 300 python tools/run_config.py $c > gpurun_out/${T}_run_$c.log 2>&1
  HS_NO_KHAT=1 timeout 300 python tools/run_config.py $c > gpurun_out/${T}_run_${c}_dense.log 2>&1
  grep -E "level|DOF/s|factor" gpurun_out/${T}_run_$c.log | head -20
  grep -E "level|DOF/s|factor" gpurun_out/${T}_run_${c}_dense.log | head -20
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_c3.log 2>&1
head -c 600 gpurun_out/${T}_bench_c3.log

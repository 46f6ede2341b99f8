#!/bin/bash
# after the CPQR mode split: new f2 test, benches (C3 default, C2), HS_PROFILE tables, C3 launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "analyze_once or nan or torch_stream or global" > gpurun_out/r2d_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/r2d_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_bench_c3.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --config C2 --no-cpu-baseline > gpurun_out/r2d_bench_c2.log 2>&1
HS_PROFILE=1 REPS=2 timeout 300 python tools/run_config.py C3 > gpurun_out/r2d_prof_c3.log 2>&1
HS_PROFILE=1 REPS=2 timeout 300 python tools/run_config.py C2 > gpurun_out/r2d_prof_c2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
  --log-file gpurun_out/r2d_launches_c3.csv python tools/one_factor_pcg.py C3 > gpurun_out/r2d_ncu_c3.log 2>&1
python tools/summarize_launches.py gpurun_out/r2d_launches_c3.csv > gpurun_out/r2d_launches_c3_summary.txt 2>&1
tail -n 3 gpurun_out/r2d_tests.log; head -c 400 gpurun_out/r2d_bench_c3.log; echo; head -c 400 gpurun_out/r2d_bench_c2.log; echo; cat gpurun_out/r2d_launches_c3_summary.txt | head -30

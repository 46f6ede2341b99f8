mkdir -p gpurun_out
for lv in 0 2 3 4; do HS_APPLY_TRACE=$lv timeout 300 python tools/apply_profile.py 2>&1 | grep "hs trace\] fwd" | tail -1; done > gpurun_out/apply_trace.log 2>&1
for fl in 0 4; do echo "FLAGS $fl" >> gpurun_out/apply_trace.log; HS_APPLY_FLAGS=$fl timeout 300 python tools/apply_profile.py 2>&1 | tail -22 | grep -E "fwd level [0-5]" >> gpurun_out/apply_trace.log; done
cat gpurun_out/apply_trace.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
tail -2 gpurun_out/gpu_tests.log; tail -1 gpurun_out/bench.log | cut -c1-900

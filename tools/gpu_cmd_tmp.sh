mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
HS_PROFILE=1 timeout 300 python tools/profile_run.py C2 2>&1 | grep "fwd level\|bwd level\|t_pcg" | head -20
tail -3 gpurun_out/gpu_tests.log

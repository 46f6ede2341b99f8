mkdir -p gpurun_out
timeout 300 python tools/apply_profile.py 2>&1 | tail -22 | grep -E "(fwd|bwd) level [0-5]"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "EXIT $?"; tail -1 gpurun_out/bench.log | cut -c1-200

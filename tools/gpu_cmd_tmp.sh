mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
for i in 1 2; do timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "EXIT $?"; tail -1 gpurun_out/bench.log | cut -c1-200; done
HS_RANK_WAIT=1 python tools/factor_loop.py 2>&1 | grep blocked | tail -2

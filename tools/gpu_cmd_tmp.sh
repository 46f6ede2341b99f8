mkdir -p gpurun_out
HS_CQ_TRACE=200 timeout 120 python tools/one_factor_pcg.py 2>&1 | grep "cq trace" | head -5
HS_PROFILE=1 python tools/factor_loop.py 2>&1 | grep "level [0-4]:" | tail -5 | sed 's/sum m.*//' | cut -c1-150
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
for i in 1 2; do timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "EXIT $?"; tail -1 gpurun_out/bench.log | cut -c1-200; done

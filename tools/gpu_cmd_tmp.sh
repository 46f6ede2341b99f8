mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
HS_NO_FUSED_POTRF_TRSM=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_nofused.log 2>&1
HS_PROFILE=1 timeout 600 python tools/one_factor_pcg.py > gpurun_out/prof.log 2>&1
tail -2 gpurun_out/gpu_tests.log; tail -1 gpurun_out/bench.log; tail -1 gpurun_out/bench_nofused.log

mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/gpu_tests.log
HS_PROFILE=1 timeout 300 python tools/profile_run.py C2 > gpurun_out/profile_c2.log 2>&1
HS_CQ_TRACE=5 timeout 300 python tools/profile_run.py C2 > gpurun_out/trace5.log 2>&1
HS_CQ_TRACE=100 timeout 300 python tools/profile_run.py C2 > gpurun_out/trace100.log 2>&1
tail -3 gpurun_out/gpu_tests.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_cpqr3 --launch-skip 5 --launch-count 1 -o gpurun_out/cpqr3_l0 -f python tools/profile_run.py C2 > gpurun_out/ncu1.log 2>&1

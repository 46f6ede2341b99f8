mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q --durations=5 > gpurun_out/gpu_full.log 2>&1; echo "EXIT $?" >> gpurun_out/gpu_full.log
tail -15 gpurun_out/gpu_full.log

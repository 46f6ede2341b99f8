mkdir -p gpurun_out
LEAF_COLUMNS=1 HS_PROFILE=1 timeout 1500 python tools/run_config.py C4 > gpurun_out/c4.log 2>&1

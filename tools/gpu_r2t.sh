#!/bin/bash
# launch list of one C3 factor + PCG, and one ncu --set full capture of a level-0 k_chol_reg
mkdir -p gpurun_out
T=${1:-r2t}
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_c3.csv python tools/one_factor_pcg.py C3 > gpurun_out/${T}_launches.log 2>&1
python tools/summarize_launches.py gpurun_out/${T}_launches_c3.csv > gpurun_out/${T}_launches_summary.txt 2>&1
head -30 gpurun_out/${T}_launches_summary.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_chol_mma --launch-skip 2 --launch-count 1 \
    -o gpurun_out/${T}_ncu_chol -f python tools/one_factor_pcg.py C3 > gpurun_out/${T}_ncu_chol.log 2>&1
python tools/ncu_summary.py gpurun_out/${T}_ncu_chol.ncu-rep; python tools/stall_summary.py gpurun_out/${T}_ncu_chol.ncu-rep | head -12

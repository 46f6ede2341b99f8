#!/bin/bash
# Launch list of one C4 bench step (factor + PCG) at HEAD under ncu (serialised, cold-cache: shares, not absolutes).
mkdir -p gpurun_out
T=${1:-r02fin}
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv \
  --log-file gpurun_out/${T}_launches_c4.csv python tools/one_factor_pcg.py C4 > gpurun_out/${T}_ncu_launches_c4.log 2>&1
python tools/summarize_launches.py gpurun_out/${T}_launches_c4.csv > gpurun_out/${T}_launches_c4_summary.txt 2>&1
head -30 gpurun_out/${T}_launches_c4_summary.txt; tail -2 gpurun_out/${T}_ncu_launches_c4.log
gzip -f gpurun_out/${T}_launches_c4.csv

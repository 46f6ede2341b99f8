#!/bin/bash
# per-level profiles at HEAD (C3, C2, C4/2) + C3 launch list
mkdir -p gpurun_out
T=${1:-s2}
HS_PROFILE=1 REPS=2 timeout 300 python tools/run_config.py C3 > gpurun_out/${T}_prof_c3.log 2>&1
HS_PROFILE=1 REPS=2 timeout 300 python tools/run_config.py C2 > gpurun_out/${T}_prof_c2.log 2>&1
HS_PROFILE=1 REPS=1 timeout 600 python tools/run_config.py C4/2 > gpurun_out/${T}_prof_c4h.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_c3.csv python tools/one_factor_pcg.py C3 > gpurun_out/${T}_launches.log 2>&1
python tools/summarize_launches.py gpurun_out/${T}_launches_c3.csv > gpurun_out/${T}_launches_c3_summary.txt 2>&1
head -25 gpurun_out/${T}_launches_c3_summary.txt
grep -E "factor wall|level device" gpurun_out/${T}_prof_*.log

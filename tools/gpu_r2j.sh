#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
  --log-file gpurun_out/r2j_launches_c3.csv python tools/one_factor_pcg.py C3 > gpurun_out/r2j_ncu_c3.log 2>&1
python tools/summarize_launches.py gpurun_out/r2j_launches_c3.csv > gpurun_out/r2j_launches_c3_summary.txt 2>&1
cap() {   # name config regex skip
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$3 --launch-skip $4 --launch-count 1 \
    -o gpurun_out/r02j_ncu_$1 -f python tools/one_factor_pcg.py $2 > gpurun_out/r02j_ncu_$1.log 2>&1
}
cap c3_scale C3 k_scale_mma 3
cap c3_chol C3 k_chol 3
cap c3_small C3 k_elim_small 10
for f in gpurun_out/r02j_ncu_*.ncu-rep; do echo "== $f"; python tools/ncu_summary.py $f; python tools/stall_summary.py $f 2>/dev/null | head -8; done > gpurun_out/r02j_ncu_summary.txt 2>&1
cat gpurun_out/r2j_launches_c3_summary.txt | head -24; cat gpurun_out/r02j_ncu_summary.txt

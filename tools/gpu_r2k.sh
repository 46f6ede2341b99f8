#!/bin/bash
mkdir -p gpurun_out
cap() {   # name config regex skip
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$3 --launch-skip $4 --launch-count 1 \
    -o gpurun_out/r02k_ncu_$1 -f python tools/one_factor_pcg.py $2 > gpurun_out/r02k_ncu_$1.log 2>&1
}
cap c3_small C3 k_elim_small 10
cap c3_cpqr C3 k_cpqr3 3
for f in gpurun_out/r02k_ncu_*.ncu-rep; do echo "== $f"; python tools/ncu_summary.py $f; python tools/stall_summary.py $f 2>/dev/null | head -8; done > gpurun_out/r02k_ncu_summary.txt 2>&1
cat gpurun_out/r02k_ncu_summary.txt

#!/bin/bash
# ncu --set full captures of the C3 level-0 kernels and the C2 coarse-level CPQR (round 2)
mkdir -p gpurun_out
cap() {   # name config regex skip
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$3 --launch-skip $4 --launch-count 1 \
    -o gpurun_out/r02e_ncu_$1 -f python tools/one_factor_pcg.py $2 > gpurun_out/r02e_ncu_$1.log 2>&1
}
cap c3_cpqr C3 k_cpqr3 3
cap c3_scale C3 'k_scale_tile' 3
cap c3_chol C3 k_chol 3
cap c3_formT C3 k_form_T 3
cap c3_schur C3 k_schur3 5
cap c3_apply_fwd C3 k_apply_fwd 0
cap c3_apply_bwd C3 k_apply_bwd 0
cap c3_spmv C3 k_spmv 0
cap c2_cpqr_l6 C2 k_cpqr3 150
for f in gpurun_out/r02e_ncu_*.ncu-rep; do echo "== $f"; python tools/ncu_summary.py $f; python tools/stall_summary.py $f 2>/dev/null | head -12; done > gpurun_out/r02e_ncu_summary.txt 2>&1
cat gpurun_out/r02e_ncu_summary.txt

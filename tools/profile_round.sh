#!/bin/bash
# Round measurement (run under gpurun): bench line, launch list of one bench step, ncu --set
# full captures of the top kernels.  Outputs in gpurun_out/ (copied to profiles/).
mkdir -p gpurun_out
R=${1:-r01}
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/${R}_bench.log 2>&1
# the launch list of one bench step (factor + PCG; the apply graph's kernels are listed per node)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
  --log-file gpurun_out/${R}_launches.csv python tools/one_factor_pcg.py C2 \
  > gpurun_out/${R}_ncu_launches.log 2>&1
python tools/summarize_launches.py gpurun_out/${R}_launches.csv > gpurun_out/${R}_launches_summary.txt 2>&1
# full captures: level-0 CPQR batch, a level-3 and a level-0 Schur launch, the level-0 scaling
# tiles, a forward and a backward apply level kernel
cap() {   # name regex skip
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$2 --launch-skip $3 --launch-count 1 \
    -o gpurun_out/${R}_ncu_$1 -f python tools/profile_run.py C2 > gpurun_out/${R}_ncu_$1.log 2>&1
}
cap cpqr3 k_cpqr3 5
cap cpqr3_l2 k_cpqr3 150
cap schur3 k_schur3 400
cap schur3_l0 k_schur3 30
cap scale k_scale_tile 5
cap apply_fwd k_apply_fwd 3
cap apply_bwd k_apply_bwd 5
for f in gpurun_out/${R}_ncu_*.ncu-rep; do python tools/ncu_summary.py $f; done > gpurun_out/${R}_ncu_summary.jsonl 2>&1
tail -c 600 gpurun_out/${R}_bench.log; head -16 gpurun_out/${R}_launches_summary.txt; cat gpurun_out/${R}_ncu_summary.jsonl

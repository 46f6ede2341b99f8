#!/bin/bash
# Round measurement (run under gpurun): bench line, launch list of the bench command,
# ncu --set full captures of the top kernels.  Outputs in gpurun_out/ (copied to profiles/).
mkdir -p gpurun_out
R=${1:-r01}
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/${R}_bench.log 2>&1
# the launch list of one bench step (factor + PCG; the apply graph's kernels are listed per node)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
  --log-file gpurun_out/${R}_launches.csv python tools/one_factor_pcg.py C2 \
  > gpurun_out/${R}_ncu_launches.log 2>&1
python tools/summarize_launches.py gpurun_out/${R}_launches.csv > gpurun_out/${R}_launches_summary.txt 2>&1
# full captures: level-0 CPQR batch, a level-3 Schur launch, one forward apply level kernel
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_cpqr3 --launch-skip 5 --launch-count 1 \
  -o gpurun_out/${R}_ncu_cpqr3 -f python tools/profile_run.py C2 > gpurun_out/${R}_ncu_cpqr3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_schur2 --launch-skip 400 --launch-count 1 \
  -o gpurun_out/${R}_ncu_schur2 -f python tools/profile_run.py C2 > gpurun_out/${R}_ncu_schur2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_apply_fwd --launch-skip 3 --launch-count 1 \
  -o gpurun_out/${R}_ncu_apply -f python tools/profile_run.py C2 > gpurun_out/${R}_ncu_apply.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_schur2 --launch-skip 30 --launch-count 1 \
  -o gpurun_out/${R}_ncu_schur2_l0 -f python tools/profile_run.py C2 > gpurun_out/${R}_ncu_schur2_l0.log 2>&1
tail -c 400 gpurun_out/${R}_bench.log; head -12 gpurun_out/${R}_launches_summary.txt

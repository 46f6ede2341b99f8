#!/bin/bash
mkdir -p gpurun_out
T=${1:-r3a}
for mode in async sync; do
  if [ $mode = sync ]; then export HS_SYNC_BATCHES=1; fi
  REPS=5 HS_RANK_WAIT=1 timeout 300 python tools/run_config.py ${CFG:-C3} > gpurun_out/${T}_run_C3_$mode.log 2>&1
  echo "== $mode"; grep -E "level device|factor wall|blocked" gpurun_out/${T}_run_C3_$mode.log | tail -6
done

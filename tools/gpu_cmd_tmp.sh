mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
for i in 1 2; do timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "EXIT $?"; tail -1 gpurun_out/bench.log | cut -c1-200; done
python - <<PY
import json
d=json.loads(open("gpurun_out/bench.log").read().strip().splitlines()[-1])
print(d["config"]["phase_s_per_step"])
PY
HS_SCHUR_NO_RED=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_nored.log 2>&1; echo "EXIT $?"; tail -1 gpurun_out/bench_nored.log | cut -c1-200
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_nored.log").read().strip().splitlines()[-1])
print(d["config"]["phase_s_per_step"])
PY

mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
for i in 1 2; do timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "EXIT $?"; tail -1 gpurun_out/bench.log | cut -c1-200; done
HS_SCALE_SOLVE=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_solve.log 2>&1; echo "EXIT $?"; tail -1 gpurun_out/bench_solve.log | cut -c1-200
python - <<PY
import json
for f in ["gpurun_out/bench.log","gpurun_out/bench_solve.log"]:
    d=json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["config"]["phase_s_per_step"])
PY

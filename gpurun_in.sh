timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s20_tests.txt 2>&1; tail -2 gpurun_out/s20_tests.txt
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "C3 or C2 or record or c4 or c5 or global" > gpurun_out/s20_tests_fs.txt 2>&1; tail -2 gpurun_out/s20_tests_fs.txt
for leg in 1 0; do
HS_ROTATE_LEGACY_SET=$leg python - <<'PY'
PY
done
HS_ROTATE_LEGACY=1 python bench.py --config C4/2 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/s20_c4h_legacy.json 2>/dev/null
python bench.py --config C4/2 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/s20_c4h_wy.json 2>/dev/null
for f in legacy wy; do python -c "
import json
d=json.loads(open('gpurun_out/s20_c4h_$f.json').read().strip().splitlines()[-1]); c=d['config']
print('$f', round(d['value']), round(c['t_factor_s'],3), {k: round(v,3) for k,v in c['phase_s_per_step'].items()}, c['pcg_iters'])"; done
HS_PROFILE=1 python bench.py --no-cpu-baseline > gpurun_out/s20_bench_c4.json 2> gpurun_out/s20_bench_c4.err; head -c 300 gpurun_out/s20_bench_c4.json; grep "record space\|host planning" gpurun_out/s20_bench_c4.err | tail -2

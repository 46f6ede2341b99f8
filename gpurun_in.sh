HS_CPQR_LIGHT=1 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s16_tests_light.txt 2>&1; tail -2 gpurun_out/s16_tests_light.txt
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "not C2 and not C3" > gpurun_out/s16_tests.txt 2>&1; tail -2 gpurun_out/s16_tests.txt
for lt in 0 -1; do
HS_CPQR_LIGHT=$lt python bench.py --config C4/2 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/s16_c4h_$lt.json 2>/dev/null
python -c "
import json
d=json.loads(open('gpurun_out/s16_c4h_$lt.json').read().strip().splitlines()[-1]); c=d['config']
print('light=$lt', round(d['value']), round(c['t_factor_s'],3), {k: round(v,3) for k,v in c['phase_s_per_step'].items()}, c['pcg_iters'])"
done
HS_CQ_LOG=1 HS_CQ_TRACE=23 HS_CQ_TRACE_SPLIT=1 python tools/one_factor_pcg.py C4/2 2>&1 | grep "cq " | sed -n 19,60p > gpurun_out/s16_cqlog.txt; head -40 gpurun_out/s16_cqlog.txt

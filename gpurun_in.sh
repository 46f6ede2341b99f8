HS_PROFILE=1 timeout 1500 python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/s6_bench_c4.json 2> gpurun_out/s6_bench_c4.err; grep "hs profile\|Error" gpurun_out/s6_bench_c4.err | cut -c1-600
tail -c 2500 gpurun_out/s6_bench_c4.json
free -g | head -2

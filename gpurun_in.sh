( time python bench.py ) > gpurun_out/s7_bench_c4.json 2> gpurun_out/s7_bench_c4.err; tail -c 3000 gpurun_out/s7_bench_c4.json; tail -5 gpurun_out/s7_bench_c4.err
( time python bench.py --impl reference --steps 1 --warmup 0 ) > gpurun_out/s7_ref.json 2> gpurun_out/s7_ref.err; tail -c 1000 gpurun_out/s7_ref.json; tail -4 gpurun_out/s7_ref.err

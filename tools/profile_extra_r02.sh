python bench.py --workload 4k --bands 4 --steps 5 --warmup 3 --no-clip --no-cpu-baseline > gpurun_out/r02_bench_4k_b4_v2.json 2>> gpurun_out/r02_bench.err

# Round-2 measurement session A (run under gpurun; one GPU): benches, CPU
# baselines, k_pcg_apply occupancy / x-load ablations.
set -x
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_reference.json 2>> gpurun_out/r02_bench.err
python bench.py --workload 4k --steps 5 --warmup 3 --no-clip > gpurun_out/r02_bench_4k.json 2>> gpurun_out/r02_bench.err
python bench.py --workload 4k --bands 4 --steps 5 --warmup 3 --no-clip > gpurun_out/r02_bench_4k_b4.json 2>> gpurun_out/r02_bench.err
python tools/ablate.py 201,202 --run > gpurun_out/r02_ablate.log 2>&1
python tools/cpu_baselines.py > gpurun_out/r02_cpu_baselines.json 2> gpurun_out/r02_cpu.err
ls -la gpurun_out

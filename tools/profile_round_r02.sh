# Round-2 measurement session (run under gpurun; one GPU).
set -x
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_reference.json 2>> gpurun_out/r02_bench.err
python bench.py --workload 4k --steps 5 --warmup 3 --no-clip > gpurun_out/r02_bench_4k.json 2>> gpurun_out/r02_bench.err
python bench.py --workload 4k --bands 4 --steps 5 --warmup 3 --no-clip > gpurun_out/r02_bench_4k_b4.json 2>> gpurun_out/r02_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clip > gpurun_out/r02_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-id ::regex:k_:1 -o gpurun_out/r02_all python tools/profile_all.py > gpurun_out/r02_ncu_all.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pcg_apply|k_pcg_update|k_energy" --launch-skip 300 --launch-count 10 -o gpurun_out/r02_steady python tools/profile_step.py > gpurun_out/r02_ncu_steady.log 2>&1
python tools/ablate.py 201,202 --run > gpurun_out/r02_ablate.log 2>&1
ls -la gpurun_out
python tools/cpu_baselines.py > gpurun_out/r02_cpu_baselines.json 2> gpurun_out/r02_cpu.err

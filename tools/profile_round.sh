set -x
python bench.py --steps 20 --warmup 3 > gpurun_out/r01_bench.json 2> gpurun_out/r01_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r01_bench_reference.json 2>> gpurun_out/r01_bench.err
python bench.py --workload 4k --steps 5 --warmup 3 > gpurun_out/r01_bench_4k.json 2>> gpurun_out/r01_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pcg_apply|k_pcg_update|k_energy" --launch-skip 300 --launch-count 10 -o gpurun_out/prof_r1b python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out

# Round-2 final measurement session: tests, the default bench, the reference arm,
# 4K, launch list and the steady-state ncu capture of the solver kernels.
set -x
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_final.log 2>&1
python bench.py > gpurun_out/r02_bench_final.json 2> gpurun_out/r02_final.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_reference_final.json 2>> gpurun_out/r02_final.err
python bench.py --workload 4k --steps 5 --warmup 3 --no-clip > gpurun_out/r02_bench_4k_final.json 2>> gpurun_out/r02_final.err
python bench.py --workload 4k --bands 4 --steps 5 --warmup 3 --no-clip --no-cpu-baseline > gpurun_out/r02_bench_4k_b4_final.json 2>> gpurun_out/r02_final.err
python tools/small_bench.py > gpurun_out/r02_small_final.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_final.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clip > gpurun_out/r02_ncu_launch_final.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pcg_apply|k_pcg_update|k_pcg_combine|k_energy" --launch-skip 300 --launch-count 12 -o /tmp/r02_steady_final python tools/profile_step.py > gpurun_out/r02_ncu_steady_final.log 2>&1
python tools/ncu_summary.py /tmp/r02_steady_final.ncu-rep gpurun_out/r02_launches_final.csv r02_steady > gpurun_out/r02_summary_final.log 2>&1
cp profiles/r02_steady_ncu_summary.* profiles/traffic.json gpurun_out/ 2>/dev/null
ncu -i /tmp/r02_steady_final.ncu-rep --page raw --csv > gpurun_out/r02_steady_final_raw.csv 2>/dev/null
gzip -f gpurun_out/r02_steady_final_raw.csv

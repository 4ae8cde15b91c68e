# Round-2 closing session, part 2 (after the trial-kernel instantiation change):
# default bench, launch list, ncu --set full of every product kernel and of the
# steady-state solver kernels, summarised on the box.
set -x
python bench.py > gpurun_out/r02_bench_final3.json 2> gpurun_out/r02_final3.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_final3.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clip > gpurun_out/r02_ncu_launch_final3.log 2>&1
ncu -f --set full --clock-control none --import-source on --kernel-id ::regex:k_:1 -o /tmp/r02_all3 python tools/profile_all.py > gpurun_out/r02_ncu_all3.log 2>&1
ncu -f --set full --clock-control none --import-source on -k regex:"k_pcg_apply|k_pcg_update|k_pcg_combine|k_energy" --launch-skip 300 --launch-count 12 -o /tmp/r02_steady3 python tools/profile_step.py > gpurun_out/r02_ncu_steady3.log 2>&1
python tools/ncu_summary.py /tmp/r02_all3.ncu-rep,/tmp/r02_steady3.ncu-rep gpurun_out/r02_launches_final3.csv r02 > gpurun_out/r02_summary_all3.log 2>&1
cp profiles/r02_ncu_summary.* gpurun_out/ 2>/dev/null
python tools/ncu_summary.py /tmp/r02_steady3.ncu-rep gpurun_out/r02_launches_final3.csv r02_steady > gpurun_out/r02_summary_steady3.log 2>&1
cp profiles/r02_steady_ncu_summary.* profiles/traffic.json gpurun_out/ 2>/dev/null
ncu -i /tmp/r02_steady3.ncu-rep --page raw --csv > gpurun_out/r02_steady_final3_raw.csv 2>/dev/null
gzip -f gpurun_out/r02_steady_final3_raw.csv

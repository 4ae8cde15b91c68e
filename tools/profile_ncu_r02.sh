# Round-2 measurement session B: launch list + ncu --set full of every
# product kernel (first launch of each, tools/profile_all.py) and of the
# steady-state solver kernels; reports are summarised ON the box and the
# .ncu-rep files deleted (gpurun brings back <= 64 MiB).
set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clip > gpurun_out/r02_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-id ::regex:k_:1 -o /tmp/r02_all python tools/profile_all.py > gpurun_out/r02_ncu_all.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pcg_apply|k_pcg_update|k_energy" --launch-skip 300 --launch-count 10 -o /tmp/r02_steady python tools/profile_step.py > gpurun_out/r02_ncu_steady.log 2>&1
python tools/ncu_summary.py /tmp/r02_all.ncu-rep,/tmp/r02_steady.ncu-rep gpurun_out/r02_launches.csv r02 > gpurun_out/r02_summary.log 2>&1
cp profiles/r02_ncu_summary.* profiles/traffic.json gpurun_out/ 2>/dev/null
ncu -i /tmp/r02_steady.ncu-rep --page source --csv --kernel-name regex:k_pcg_apply --launch-skip 2 --launch-count 1 --print-source sass > gpurun_out/r02_sass_apply.csv 2>/dev/null
ncu -i /tmp/r02_steady.ncu-rep --page raw --csv > gpurun_out/r02_steady_raw.csv 2>/dev/null
ncu -i /tmp/r02_all.ncu-rep --page raw --csv > gpurun_out/r02_all_raw.csv 2>/dev/null
gzip -f gpurun_out/r02_sass_apply.csv gpurun_out/r02_steady_raw.csv gpurun_out/r02_all_raw.csv
ls -la gpurun_out

# Round-2 closing measurement session (after the aux-kernel work): tests,
# smoke, the default bench, the reference arm, 4K, small sizes, the launch
# list, ncu --set full of every product kernel (first launch of each) and of
# the steady-state solver kernels.  Reports summarised on the box, .ncu-rep
# files left in /tmp (gpurun brings back <= 64 MiB).
set -x
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_final2.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final2.log 2>&1
python bench.py > gpurun_out/r02_bench_final2.json 2> gpurun_out/r02_final2.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_reference_final2.json 2>> gpurun_out/r02_final2.err
python bench.py --workload 4k --steps 5 --warmup 3 --no-clip > gpurun_out/r02_bench_4k_final2.json 2>> gpurun_out/r02_final2.err
python bench.py --workload 4k --bands 4 --steps 5 --warmup 3 --no-clip --no-cpu-baseline > gpurun_out/r02_bench_4k_b4_final2.json 2>> gpurun_out/r02_final2.err
python tools/small_bench.py > gpurun_out/r02_small_final2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_final2.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clip > gpurun_out/r02_ncu_launch_final2.log 2>&1
ncu -f --set full --clock-control none --import-source on --kernel-id ::regex:k_:1 -o /tmp/r02_all2 python tools/profile_all.py > gpurun_out/r02_ncu_all2.log 2>&1
ncu -f --set full --clock-control none --import-source on -k regex:"k_pcg_apply|k_pcg_update|k_pcg_combine|k_energy" --launch-skip 300 --launch-count 12 -o /tmp/r02_steady2 python tools/profile_step.py > gpurun_out/r02_ncu_steady2.log 2>&1
python tools/ncu_summary.py /tmp/r02_all2.ncu-rep,/tmp/r02_steady2.ncu-rep gpurun_out/r02_launches_final2.csv r02 > gpurun_out/r02_summary_all2.log 2>&1
cp profiles/r02_ncu_summary.* gpurun_out/ 2>/dev/null
python tools/ncu_summary.py /tmp/r02_steady2.ncu-rep gpurun_out/r02_launches_final2.csv r02_steady > gpurun_out/r02_summary_steady2.log 2>&1
cp profiles/r02_steady_ncu_summary.* profiles/traffic.json gpurun_out/ 2>/dev/null
ncu -i /tmp/r02_steady2.ncu-rep --page raw --csv > gpurun_out/r02_steady_final2_raw.csv 2>/dev/null
gzip -f gpurun_out/r02_steady_final2_raw.csv
ls -la gpurun_out

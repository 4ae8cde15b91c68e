# Single-reduction PCG A/B (LS_PCG=cg1) against the default textbook loop.
set -x
python -m pytest tests/test_gpu_cg1.py -q -p no:cacheprovider > gpurun_out/pytest_cg1.log 2>&1
python bench.py --profile-only --steps 10 --warmup 3 > gpurun_out/r02_ab_textbook.json 2> gpurun_out/r02_ab.err
LS_PCG=cg1 python bench.py --profile-only --steps 10 --warmup 3 > gpurun_out/r02_ab_cg1.json 2>> gpurun_out/r02_ab.err
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-clip > gpurun_out/r02_ab_textbook_full.json 2>> gpurun_out/r02_ab.err
LS_PCG=cg1 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-clip > gpurun_out/r02_ab_cg1_full.json 2>> gpurun_out/r02_ab.err
LS_PCG=cg1 ncu --set full --clock-control none --import-source on -k regex:"k_cg_iter" --launch-skip 40 --launch-count 2 -o /tmp/r02_cg1 python tools/profile_step.py > gpurun_out/r02_ncu_cg1.log 2>&1
ncu -i /tmp/r02_cg1.ncu-rep --page raw --csv > gpurun_out/r02_cg1_raw.csv 2>/dev/null
ncu -i /tmp/r02_cg1.ncu-rep --page details --csv > gpurun_out/r02_cg1_details.csv 2>/dev/null
gzip -f gpurun_out/r02_cg1_raw.csv gpurun_out/r02_cg1_details.csv
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_dense" --csv --log-file gpurun_out/r02_dense_launches.csv python tools/frame1_probe.py 1 > gpurun_out/r02_dense_ncu.log 2>&1; python tools/frame1_probe.py 3 > gpurun_out/r02_f1_probe.log 2>&1; python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_dense.py tests/test_gpu_bands.py -q -p no:cacheprovider > gpurun_out/pytest_dense.log 2>&1

#!/bin/bash
# aux-kernel A/B (warp sort vs per-thread sort) + GPU tests + a bench line
python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/aux_pytest.log 2>&1; echo rc=$? >> gpurun_out/aux_pytest.log
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-clip > gpurun_out/aux_bench.json 2> gpurun_out/aux_bench.err
LS_SORT_THREAD=1 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-clip --no-e2e > gpurun_out/aux_bench_thread.json 2>> gpurun_out/aux_bench.err
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-clip --no-e2e > gpurun_out/aux_bench2.json 2>> gpurun_out/aux_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_sort|k_sample|k_fill|k_image|k_edge|k_copy|elementwise|k_all_finite" -c 200 --csv --log-file gpurun_out/aux_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-clip --no-e2e --profile-only > gpurun_out/aux_ncu.log 2>&1
LS_SORT_THREAD=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_sort" -c 20 --csv --log-file gpurun_out/aux_launches_thread.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-clip --no-e2e --profile-only > gpurun_out/aux_ncu2.log 2>&1

#!/bin/bash
# sampler warp-base states: sampler / band / headline tests, bench, aux launch lists (with and without base states)
python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py tests/test_gpu_bands.py tests/test_gpu_bands_spmd.py tests/test_gpu_reference_energy.py tests/test_gpu_headline.py -q -p no:cacheprovider -x > gpurun_out/aux3_pytest.log 2>&1; echo rc=$? >> gpurun_out/aux3_pytest.log
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-clip --no-e2e > gpurun_out/aux3_bench.json 2> gpurun_out/aux3_bench.err
LS_SAMPLE_NOBASE=1 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-clip --no-e2e > gpurun_out/aux3_bench_nobase.json 2>> gpurun_out/aux3_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_(s|f|i|e|c|a|d|p)" -c 600 --csv --log-file gpurun_out/aux3_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-clip --no-e2e --profile-only > gpurun_out/aux3_ncu.log 2>&1
LS_SAMPLE_NOBASE=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_sample" -c 60 --csv --log-file gpurun_out/aux3_launches_nobase.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-clip --no-e2e --profile-only > gpurun_out/aux3_ncu2.log 2>&1

#!/bin/bash
python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py tests/test_gpu_bands.py tests/test_gpu_bands_spmd.py tests/test_gpu_headline.py tests/test_gpu_reference_energy.py -q -p no:cacheprovider -x > gpurun_out/fill_pytest.log 2>&1; echo rc=$? >> gpurun_out/fill_pytest.log
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-clip --no-e2e > gpurun_out/fill_bench.json 2> gpurun_out/fill_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_(sample|fill|sort)" -c 40 --csv --log-file gpurun_out/fill_launches.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-clip --no-e2e --profile-only > /dev/null 2>&1

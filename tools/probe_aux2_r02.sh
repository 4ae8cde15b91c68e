#!/bin/bash
# aux kernels after the fill change: adjacency / sampler parity tests, a bench line, launch list of the aux kernels
python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py tests/test_gpu_bands.py tests/test_gpu_headline.py -q -p no:cacheprovider -x > gpurun_out/aux2_pytest.log 2>&1; echo rc=$? >> gpurun_out/aux2_pytest.log
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-clip --no-e2e > gpurun_out/aux2_bench.json 2> gpurun_out/aux2_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ls::" -c 1500 --csv --log-file gpurun_out/aux2_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-clip --no-e2e --profile-only > gpurun_out/aux2_ncu.log 2>&1

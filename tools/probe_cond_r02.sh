#!/bin/bash
# graph conditional nodes for the line-search halvings: tests + A/B (LS_NO_COND=1)
python -m pytest tests/test_gpu_scale.py tests/test_gpu_headline.py tests/test_gpu_parity.py tests/test_gpu_correction.py -q -p no:cacheprovider -x > gpurun_out/cond_pytest.log 2>&1; echo rc=$? >> gpurun_out/cond_pytest.log
for i in 1 2; do
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-clip --no-e2e > gpurun_out/cond_bench_$i.json 2> gpurun_out/cond_bench.err
LS_NO_COND=1 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-clip --no-e2e > gpurun_out/cond_bench_nocond_$i.json 2>> gpurun_out/cond_bench.err
done

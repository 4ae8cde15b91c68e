set -x
python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_d.log 2>&1
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-clip > gpurun_out/r02_stored_1.json 2> gpurun_out/r02_d.err
LS_X_DEFERRED=1 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-clip > gpurun_out/r02_deferred_1.json 2>> gpurun_out/r02_d.err
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-clip > gpurun_out/r02_stored_2.json 2>> gpurun_out/r02_d.err
LS_X_DEFERRED=1 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-clip > gpurun_out/r02_deferred_2.json 2>> gpurun_out/r02_d.err
python tools/ablate.py 206 --run > gpurun_out/r02_ablate3.log 2>&1

set -x
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_e.log 2>&1
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-clip > gpurun_out/r02_zonly_1.json 2> gpurun_out/r02_e.err
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-clip > gpurun_out/r02_zonly_2.json 2>> gpurun_out/r02_e.err

set -x
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_c.log 2>&1
python tools/ablate.py 204,205 --run > gpurun_out/r02_ablate2.log 2>&1
python bench.py > gpurun_out/r02_bench_c.json 2> gpurun_out/r02_bench_c.err

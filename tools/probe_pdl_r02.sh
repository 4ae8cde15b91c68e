set -x
python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_pdl.log 2>&1
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-clip > gpurun_out/r02_pdl_on.json 2> gpurun_out/r02_pdl.err
LS_NO_PDL=1 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-clip > gpurun_out/r02_pdl_off.json 2>> gpurun_out/r02_pdl.err
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-clip > gpurun_out/r02_pdl_on2.json 2>> gpurun_out/r02_pdl.err
LS_NO_PDL=1 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-clip > gpurun_out/r02_pdl_off2.json 2>> gpurun_out/r02_pdl.err
python tools/small_bench.py > gpurun_out/r02_small_pdl_on.log 2>&1
LS_NO_PDL=1 python tools/small_bench.py > gpurun_out/r02_small_pdl_off.log 2>&1

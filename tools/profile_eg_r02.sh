#!/bin/bash
# ncu --set full of one steady-state EG and one trial launch with source counters; the
# source pages (SASS + CUDA line attribution) are exported on the box, the report deleted
set -x
ncu --set full --clock-control none --import-source on -k regex:"k_energy" --launch-skip 12 --launch-count 2 -o /tmp/r02_eg python tools/profile_step.py > gpurun_out/r02_eg_ncu.log 2>&1
ncu -i /tmp/r02_eg.ncu-rep --page source --csv --kernel-name k_energy --launch-count 1 --print-source sass > gpurun_out/r02_eg_sass.csv 2> gpurun_out/r02_eg_src.err
ncu -i /tmp/r02_eg.ncu-rep --page source --csv --kernel-name k_energy --launch-count 1 --print-source cuda > gpurun_out/r02_eg_cuda.csv 2>> gpurun_out/r02_eg_src.err
ncu -i /tmp/r02_eg.ncu-rep --page source --csv --kernel-name k_energy --launch-skip 1 --launch-count 1 --print-source cuda > gpurun_out/r02_trial_cuda.csv 2>> gpurun_out/r02_eg_src.err
gzip -f gpurun_out/r02_eg_sass.csv gpurun_out/r02_eg_cuda.csv gpurun_out/r02_trial_cuda.csv
ls -la gpurun_out | tail

python tools/clip_probe.py 300 > gpurun_out/clip_default.log 2>&1
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True python tools/clip_probe.py 300 > gpurun_out/clip_expand.log 2>&1
python tools/clip_probe.py 300 40 > gpurun_out/clip_prewarm.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_dense|k_energy|k_pcg" --csv --log-file gpurun_out/f1_launches.csv python tools/frame1_probe.py 1 > gpurun_out/f1_ncu.log 2>&1
python tools/frame1_probe.py 3 > gpurun_out/f1_probe.log 2>&1
python -m pytest tests/test_gpu_bands_spmd.py tests/test_gpu_bands.py tests/test_gpu_dist1.py -q -p no:cacheprovider > gpurun_out/pytest5.log 2>&1

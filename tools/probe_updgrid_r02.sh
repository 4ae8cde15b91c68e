#!/bin/bash
# k_pcg_update grid size A/B (LS_UPD_GRID = CTAs per SM; default = occupancy, 8)
for g in 8 4 16 24 8; do
  LS_UPD_GRID=$g python bench.py --profile-only --steps 10 --warmup 3 > gpurun_out/updgrid_$g.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/updgrid_$g.json').read().strip().splitlines()[-1]);pk=d['roofline']['per_kernel'];print($g, round(pk['update']['avg_us'],2), round(pk['apply']['avg_us'],2), round(d['value'],2))" >> gpurun_out/updgrid.log
done

"""Warm per-kernel device time of streaming frames at 1080p K=8 (CUPTI via
torch.profiler), to size the per-frame aux work against the solve.

    python tools/step_kernels.py [frames]
"""
import sys
from collections import defaultdict

import torch

sys.path.insert(0, ".")
from paper_1908_01961_b200 import synth                                  # noqa: E402
from paper_1908_01961_b200.energy import EnergyWeights                   # noqa: E402
from paper_1908_01961_b200.palette import BaseColorPalette               # noqa: E402
from paper_1908_01961_b200.pipeline import StreamingDecomposer           # noqa: E402
from paper_1908_01961_b200.solver import SolveConfig                     # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
dev = torch.device("cuda")
clip = synth.make_clip(1080, 1920, 8, n + 4, seed=0, device=dev)
dec = StreamingDecomposer(BaseColorPalette(colors=clip.colors), EnergyWeights(), SolveConfig(tol_rel=0.0))
dec.first(clip.frames[0])
for i in range(1, 4):
    dec.step(clip.frames[i])
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for i in range(4, 4 + n):
        dec.step(clip.frames[i])
    torch.cuda.synchronize()
tot, cnt = defaultdict(float), defaultdict(int)
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        name = ev.name.split("(")[0]
        tot[name] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
        cnt[name] += 1
all_us = sum(tot.values())
print(f"{n} frames, device time {all_us / 1e3 / n:.3f} ms/frame")
for k in sorted(tot, key=tot.get, reverse=True)[:30]:
    print(f"{k[:60]:60s} {cnt[k] / n:6.1f}/frame {tot[k] / n:9.1f} us/frame {tot[k] / max(cnt[k], 1):8.1f} us avg")

"""GPU idle gaps of the streaming loop (torch.profiler / CUPTI timestamps):
per frame, busy kernel time vs the frame's span, and where the gaps sit."""
import sys, json, time
sys.path.insert(0, '.')
import torch
from torch.profiler import profile, ProfilerActivity
from paper_1908_01961_b200 import synth
from paper_1908_01961_b200.energy import EnergyWeights
from paper_1908_01961_b200.palette import BaseColorPalette
from paper_1908_01961_b200.pipeline import StreamingDecomposer
from paper_1908_01961_b200.solver import SolveConfig

H, W, K, n = 1080, 1920, 8, 8
clip = synth.make_clip(H, W, K, n + 4, seed=0, device="cuda")
dec = StreamingDecomposer(BaseColorPalette(colors=clip.colors), EnergyWeights(), SolveConfig(tol_rel=0.0))
dec.first(clip.frames[0])
for i in range(3):
    dec.step(clip.frames[1 + i])
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for i in range(n):
        with torch.profiler.record_function(f"frame{i}"):
            dec.step(clip.frames[4 + i])
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ks = sorted((e.time_range.start, e.time_range.end, e.name) for e in evs)
t0, t1 = ks[0][0], max(k[1] for k in ks)
busy, last, gaps = 0.0, ks[0][0], []
for s, e, nm in ks:
    if s > last:
        gaps.append((s - last, nm))
    busy += max(0, e - max(s, last))
    last = max(last, e)
span = t1 - t0
print(f"span {span/1e3:.2f} ms for {n} frames: {span/n/1e3:.2f} ms/frame, busy {busy/n/1e3:.2f} ms/frame, idle {(span-busy)/n/1e3:.2f} ms/frame")
gaps.sort(reverse=True)
for g, nm in gaps[:25]:
    print(f"gap {g:8.1f} us before {nm[:80]}")

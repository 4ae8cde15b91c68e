"""Whole-clip timing through decompose_frames at 1080p K=8 (SURVEY cfg3):
frames per second including frame 1, and the per-frame wall times, under a
given allocator configuration (set PYTORCH_CUDA_ALLOC_CONF before running).

    python tools/clip_probe.py [n_frames] [prewarm_gb]
"""
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1908_01961_b200 import synth                           # noqa: E402
from paper_1908_01961_b200.energy import EnergyWeights            # noqa: E402
from paper_1908_01961_b200.palette import BaseColorPalette        # noqa: E402
from paper_1908_01961_b200.pipeline import decompose_frames       # noqa: E402
from paper_1908_01961_b200.solver import SolveConfig              # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
prewarm = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
dev = torch.device("cuda")
clip = synth.make_clip(1080, 1920, 8, n, seed=1, device=dev)
pal = BaseColorPalette(colors=clip.colors)
# warm the kernels / contexts on a short clip
decompose_frames(clip.frames[:3], EnergyWeights(), SolveConfig(tol_rel=0.0), seed=1, palette=pal)
if prewarm > 0:
    blk = torch.empty(int(prewarm * 2**30), dtype=torch.uint8, device=dev)
    del blk
torch.cuda.synchronize()
t0 = time.perf_counter()
res = decompose_frames(clip.frames, EnergyWeights(), SolveConfig(tol_rel=0.0), seed=1, palette=pal)
torch.cuda.synchronize()
sec = time.perf_counter() - t0
fs = [1e3 * s for s in res.frame_seconds]
print(f"frames {n} total {sec:.3f} s = {n / sec:.2f} fps; frame1 {fs[0]:.1f} ms; streaming median "
      f"{statistics.median(fs[1:]):.2f} ms, p90 {sorted(fs[1:])[int(0.9 * (n - 1))]:.2f}, max {max(fs[1:]):.2f}; "
      f"reserved {torch.cuda.memory_reserved() / 2**30:.1f} GiB")

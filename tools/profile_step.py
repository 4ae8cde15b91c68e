"""Short 1080p K=8 run for ncu: one unrefined first frame (2 GN steps) and
`--frames` streaming frames.  Kernel order per GN step: k_energy(EG),
16 x (k_apply, k_update), k_energy(trial)."""
import argparse, sys, time
sys.path.insert(0, '.')
import torch
from paper_1908_01961_b200 import synth
from paper_1908_01961_b200.energy import EnergyWeights
from paper_1908_01961_b200.palette import BaseColorPalette
from paper_1908_01961_b200.pipeline import StreamingDecomposer
from paper_1908_01961_b200.solver import SolveConfig

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=2)
ap.add_argument("--H", type=int, default=1080)
ap.add_argument("--W", type=int, default=1920)
ap.add_argument("--K", type=int, default=8)
a = ap.parse_args()
clip = synth.make_clip(a.H, a.W, a.K, a.frames + 1, seed=0, device="cuda")
dec = StreamingDecomposer(BaseColorPalette(colors=clip.colors), EnergyWeights(),
                          SolveConfig(tol_rel=0.0, refine=False, outer_iterations=1))
dec.first(clip.frames[0])
for i in range(a.frames):
    t = time.perf_counter()
    dec.step(clip.frames[1 + i])
    torch.cuda.synchronize()
    print(f"frame {i+1}: {1e3*(time.perf_counter()-t):.2f} ms")

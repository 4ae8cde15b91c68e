"""Streaming frames/s at small sizes (SURVEY configs[0]/[1]: 160x120 K=4,
640x480 K=6), CUDA-graph flip-flop vs eager launches (LS_NO_GRAPH=1)."""
import os, sys, time
sys.path.insert(0, '.')
import torch
from paper_1908_01961_b200 import synth
from paper_1908_01961_b200.energy import EnergyWeights
from paper_1908_01961_b200.palette import BaseColorPalette
from paper_1908_01961_b200.pipeline import StreamingDecomposer
from paper_1908_01961_b200.solver import SolveConfig

for H, W, K in ((120, 160, 4), (480, 640, 6), (1080, 1920, 8)):
    clip = synth.make_clip(H, W, K, 24, seed=0, device="cuda")
    for mode in ("graph", "eager"):
        os.environ["LS_NO_GRAPH"] = "1" if mode == "eager" else ""
        dec = StreamingDecomposer(BaseColorPalette(colors=clip.colors), EnergyWeights(), SolveConfig(tol_rel=0.0))
        dec.first(clip.frames[0])
        for i in range(3):
            dec.step(clip.frames[1 + i])
        torch.cuda.synchronize()
        t = time.perf_counter()
        for i in range(20):
            dec.step(clip.frames[4 + i])
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 20
        print(f"{W}x{H} K={K} {mode}: {1e3 * dt:.3f} ms/frame, {1 / dt:.1f} fps", flush=True)

"""Streaming frames/s across frame sizes and palette sizes (graph path),
with the SURVEY 8(d) frame-bytes model fraction, for DESIGN.md."""
import json, sys, time
sys.path.insert(0, '.')
import torch
from paper_1908_01961_b200 import synth
from paper_1908_01961_b200.energy import EnergyWeights
from paper_1908_01961_b200.palette import BaseColorPalette
from paper_1908_01961_b200.pipeline import StreamingDecomposer
from paper_1908_01961_b200.solver import SolveConfig

PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if __import__("os").path.exists("MEASURED_PEAKS.json") else 6549.8
rows = []
for (H, W, K) in ((480, 640, 6), (720, 1280, 8), (1080, 1920, 4), (1080, 1920, 8), (1080, 1920, 12),
                  (1440, 2560, 8), (2160, 3840, 8)):
    n = 12
    clip = synth.make_clip(H, W, K, n + 4, seed=0, device="cuda")
    dec = StreamingDecomposer(BaseColorPalette(colors=clip.colors), EnergyWeights(), SolveConfig(tol_rel=0.0))
    dec.first(clip.frames[0])
    for i in range(3):
        dec.step(clip.frames[1 + i])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        dec.step(clip.frames[4 + i])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    U = K + 4
    frac = 4 * H * W * (860 * U + 298) / (ms / 1e3) / 1e9 / PEAK
    rows.append((W, H, K, ms, 1e3 / ms, frac))
    print(f"{W}x{H} K={K}: {ms:.2f} ms/frame, {1e3 / ms:.1f} fps, frame-model {frac:.2f} of HBM peak", flush=True)
    del dec, clip
    torch.cuda.empty_cache()

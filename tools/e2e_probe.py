"""Where the end-to-end frame time goes: device-resident frames vs with the
per-frame H2D only, D2H only, and both (bench.py's e2e loop)."""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_1908_01961_b200 import synth
from paper_1908_01961_b200.energy import EnergyWeights
from paper_1908_01961_b200.palette import BaseColorPalette
from paper_1908_01961_b200.pipeline import StreamingDecomposer
from paper_1908_01961_b200.solver import SolveConfig

H, W, K, n = 1080, 1920, 8, 20
clip = synth.make_clip(H, W, K, n + 4, seed=0, device="cuda")
dec = StreamingDecomposer(BaseColorPalette(colors=clip.colors), EnergyWeights(), SolveConfig(tol_rel=0.0))
dec.first(clip.frames[0])
for i in range(3):
    st = dec.step(clip.frames[1 + i])
host = [f.cpu().pin_memory() for f in clip.frames[4:]]
out_host = [torch.empty(tuple(st.layers.X.shape), dtype=torch.float32).pin_memory() for _ in range(2)]
side = torch.cuda.Stream()
cp = torch.cuda.Stream()
for mode in sys.argv[1:] or ("device", "h2d", "d2h", "both", "overlap", "device"):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    nxt = None
    if mode == "overlap":
        cp.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cp):
            nxt = (host[0].to("cuda", non_blocking=True), torch.cuda.Event())
            nxt[1].record(cp)
    for i in range(n):
        if mode == "overlap":
            f, ev = nxt
            torch.cuda.current_stream().wait_event(ev)
            f.record_stream(torch.cuda.current_stream())
            if i + 1 < n:
                with torch.cuda.stream(cp):
                    nxt = (host[i + 1].to("cuda", non_blocking=True), torch.cuda.Event())
                    nxt[1].record(cp)
        else:
            f = host[i].to("cuda", non_blocking=True) if mode in ("h2d", "both") else clip.frames[4 + i]
        s2 = dec.step(f)
        if mode in ("d2h", "both", "overlap"):
            done = torch.cuda.Event(); done.record(); side.wait_event(done)
            with torch.cuda.stream(side):
                s2.layers.X.record_stream(side)
                out_host[i % 2].copy_(s2.layers.X, non_blocking=True)
    torch.cuda.current_stream().wait_stream(side)
    e1.record(); torch.cuda.synchronize()
    print(f"{mode:7s}: {e0.elapsed_time(e1) / n:.2f} ms/frame", flush=True)

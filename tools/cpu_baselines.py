"""CPU timings of one full 1920x1080 K=8 streaming frame (segment + aux +
2 outer x 2 GN x 16 PCG, fixed iteration counts) for the same synthetic
clip as bench.py, by three CPU implementations of the path:

  reference  the reference package itself (baseline/_ref, lumisplit.solver.solve_frame)
  numpy      the NumPy oracle port (oracle/lumisplit_oracle.py)
  c          the compiled restatement (oracle/ls_oracle.c), 1 thread and all threads

    python tools/cpu_baselines.py [--skip reference,numpy] > profiles/r02_cpu_baselines.json
"""
import argparse
import json
import os
import sys
import time
from dataclasses import replace
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

ap = argparse.ArgumentParser()
ap.add_argument("--skip", default="")
ap.add_argument("--H", type=int, default=1080)
ap.add_argument("--W", type=int, default=1920)
ap.add_argument("--K", type=int, default=8)
a = ap.parse_args()
skip = set(a.skip.split(","))

import torch  # noqa: E402
from oracle import c_oracle as CO                      # noqa: E402
from oracle import lumisplit_oracle as O               # noqa: E402
from paper_1908_01961_b200 import synth                # noqa: E402

torch.set_num_threads(os.cpu_count() or 1)
clip = synth.make_clip(a.H, a.W, a.K, 2, seed=0, device="cpu")
f0, f1 = (f.double().numpy() for f in clip.frames)
colors = clip.colors
ids0 = CO.segment(f0, colors)
r0, T0 = CO.initialize(f0, ids0, colors)
cfg = replace(O.Config(tol_rel=0.0), refine=False, outer_iterations=2)
out = {"frame": f"{a.W}x{a.H} K={a.K} streaming frame (2 outer x 2 GN x 16 PCG), warm start = "
                f"frame-0 initialisation", "cpu_threads": os.cpu_count()}
try:
    out["cpu"] = next(ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo") if ln.startswith("model name"))
except Exception:
    pass


def timed(fn):
    t = time.perf_counter()
    res = fn()
    return time.perf_counter() - t, res


prev = O.State(image=None, colors=colors, r=r0, T=T0, aux=None, weights=None, config=None)
for th in (os.cpu_count(), 1):
    CO.set_threads(th)
    dt, st = timed(lambda: CO.stream_frame(f1, colors, prev, f0, O.Weights(), cfg, 1))
    out[f"c_{th}_threads_s"] = dt
    E_c = st.records[-1]["energy_after"]
    out["c_energy_after"] = E_c
    print(f"c {th} threads: {dt:.2f} s", file=sys.stderr, flush=True)

if "numpy" not in skip:
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    ids1 = O.segment(f1, colors)

    def run_np():
        aux = O.build_aux(f1, ids1, 1, O.chromaticity(f0)[0], r0)
        st = O.State(image=f1, colors=colors, r=r0.copy(), T=T0.copy(), aux=aux, weights=O.Weights(), config=cfg)
        return O.flip_flop(st)
    dt, st = timed(run_np)
    out["numpy_oracle_s"] = dt
    out["numpy_energy_after"] = st.records[-1]["energy_after"]
    print(f"numpy oracle: {dt:.2f} s", file=sys.stderr, flush=True)

if "reference" not in skip and (ROOT / "baseline" / "_ref" / "lumisplit").exists():
    sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
    import lumisplit as L
    frame0, frame1 = L.imaging.Frame(f0), L.imaging.Frame(f1)
    pal = L.palette.BaseColorPalette(colors=colors)
    cmap = L.palette.segment(frame1, pal)
    prev_layers = L.energy.LayerStack(r=r0.copy(), T=T0.copy())
    rcfg = L.solver.SolveConfig(tol_rel=0.0, refine=False, outer_iterations=2)
    dt, st = timed(lambda: L.solver.solve_frame(frame1, pal, cmap, L.energy.EnergyWeights(), rcfg, seed=1,
                                                previous=prev_layers, prev_chroma=L.imaging.chromaticity(frame0),
                                                prev_r=r0))
    out["reference_package_s"] = dt
    out["reference_energy_after"] = st.records[-1]["energy_after"]
    out["reference_threads"] = "numpy/OpenBLAS defaults"
    print(f"reference package: {dt:.2f} s", file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))

"""Frame-1 (refinement) wall-time breakdown at 1080p K=8: segment, aux,
initialize, refine_palette, repeated to expose run-to-run variance.

    python tools/frame1_probe.py [reps]
"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1908_01961_b200 import synth                           # noqa: E402
from paper_1908_01961_b200.energy import EnergyWeights            # noqa: E402
from paper_1908_01961_b200.imaging import Frame                   # noqa: E402
from paper_1908_01961_b200.palette import BaseColorPalette, segment  # noqa: E402
from paper_1908_01961_b200.refine import refine_palette           # noqa: E402
from paper_1908_01961_b200.solver import SolveConfig, SolverState, build_aux, initialize  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
dev = torch.device("cuda")
clip = synth.make_clip(1080, 1920, 8, 2, seed=0, device=dev)
pal0 = BaseColorPalette(colors=clip.colors)


def t():
    torch.cuda.synchronize()
    return time.perf_counter()


for rep in range(reps):
    t0 = t()
    frame = Frame(clip.frames[0])
    cm = segment(frame, pal0)
    t1 = t()
    aux = build_aux(frame, cm, seed=0)
    layers = initialize(frame, cm, pal0)
    t2 = t()
    st = SolverState(frame=frame, palette=pal0, layers=layers, aux=aux, weights=EnergyWeights(),
                     config=SolveConfig(tol_rel=0.0))
    refine_palette(st)
    t3 = t()
    n_dense = sum(1 for r in st.records if r["phase"] == "dense")
    trials = sum(1 for r in st.records if r["phase"] == "sparse")
    print(f"rep {rep}: segment {1e3 * (t1 - t0):.1f} ms, aux+init {1e3 * (t2 - t1):.1f} ms, "
          f"refine {1e3 * (t3 - t2):.1f} ms ({trials} sparse, {n_dense} dense records), "
          f"total {1e3 * (t3 - t0):.1f} ms", flush=True)

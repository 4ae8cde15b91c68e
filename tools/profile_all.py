"""One pass over every product kernel at the headline size (1920x1080, K=8)
for an `ncu --set full` capture of each kernel's first launch
(tools/profile_round_r02.sh): palette estimation, segmentation, per-frame
aux (chroma, edge gate, sampler, CSR, scan), first-frame refinement (dense
accumulation + SVD solve, host-driven GN steps), two streaming frames
through the CUDA-graph flip-flop, the per-block residual protocol, flood
fill and recomposition."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1908_01961_b200 import synth                                # noqa: E402
from paper_1908_01961_b200.correction import identify_region           # noqa: E402
from paper_1908_01961_b200.editing import recolor                      # noqa: E402
from paper_1908_01961_b200.energy import EnergyWeights, assemble_blocks  # noqa: E402
from paper_1908_01961_b200.imaging import Frame                        # noqa: E402
from paper_1908_01961_b200.palette import BaseColorPalette, estimate_palette  # noqa: E402
from paper_1908_01961_b200.pipeline import StreamingDecomposer          # noqa: E402
from paper_1908_01961_b200.solver import SolveConfig                    # noqa: E402

clip = synth.make_clip(1080, 1920, 8, 3, seed=0, device="cuda")
f0 = Frame(clip.frames[0])
pal_est, cm_est = estimate_palette(f0, k_max=10, seed=0)
pal = BaseColorPalette(colors=clip.colors)
dec = StreamingDecomposer(pal, EnergyWeights(), SolveConfig(tol_rel=0.0, outer_iterations=4))
t = time.perf_counter()
s0 = dec.first(clip.frames[0])
torch.cuda.synchronize()
print(f"frame 1: {1e3 * (time.perf_counter() - t):.1f} ms, {len(s0.records)} records")
for i in (1, 2):
    t = time.perf_counter()
    st = dec.step(clip.frames[i])
    torch.cuda.synchronize()
    print(f"frame {i + 1}: {1e3 * (time.perf_counter() - t):.2f} ms")
blocks = assemble_blocks(st.frame, st.palette, st.layers, st.aux, st.weights)
res = blocks[3].residual(st.layers.r, st.layers.T)
out_dr, out_dT = torch.zeros_like(st.layers.r), torch.zeros_like(st.layers.T)
blocks[3].apply_jt(res, out_dr, out_dT)
blocks[6].add_diag(out_dr, out_dT)
region = identify_region((960, 540), st.cluster_map, frame=st.frame)
img = recolor(st.layers, st.palette, 1, np.array([0.5, 0.4, 0.3]), st.cluster_map)
torch.cuda.synchronize()
print("done", float(out_dr.abs().sum()), int(region.size), tuple(img.shape))

"""Small end-to-end workload touching every kernel family, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
sampler + CSR, segment, first frame with refinement (EG, PCG, trials,
dense), streaming frames through the CUDA-graph flip-flop, row bands,
flood fill, the batched correction candidates and the edit recomposition."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1908_01961_b200 import synth, correction, editing
from paper_1908_01961_b200.energy import EnergyWeights
from paper_1908_01961_b200.palette import BaseColorPalette
from paper_1908_01961_b200.pipeline import StreamingDecomposer
from paper_1908_01961_b200.solver import SolveConfig

clip = synth.make_clip(64, 96, 3, 3, seed=1, device="cuda")
pal = BaseColorPalette(colors=clip.colors)
for bands in (0, 2):
    dec = StreamingDecomposer(pal, EnergyWeights(), SolveConfig(outer_iterations=3), bands=bands)
    st = dec.first(clip.frames[0])
    for f in clip.frames[1:]:
        st = dec.step(f)
reg = correction.identify_region((40, 30), st.cluster_map)
# the K candidate solves as one batched launch sequence (ls_flip_flop_batch)
from paper_1908_01961_b200.imaging import Frame
pick = correction.correct_reflectance(reg, Frame(clip.frames[-1]), st.cluster_map, dec.palette,
                                      config=SolveConfig(outer_iterations=1, refine=False))
out = editing.recolor(st.layers, dec.palette, 1, [0.3, 0.5, 0.2], st.cluster_map)
torch.cuda.synchronize()
print("workload ok", float(out.mean()), reg.size, pick)

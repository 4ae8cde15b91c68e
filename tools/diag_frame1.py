"""Diagnose frame-1 (cfg1) divergence vs the reference golden records."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from tests.golden_io import load, records_array
from paper_1908_01961_b200.solver import SolveConfig, SolverState, build_aux, initialize
from paper_1908_01961_b200.refine import refine_palette
from paper_1908_01961_b200.palette import BaseColorPalette, cluster_map_from_ids
from paper_1908_01961_b200.imaging import Frame
from paper_1908_01961_b200.energy import EnergyWeights
d = load("frame1_cfg1")
frame = Frame(torch.as_tensor(d["image"], device="cuda"))
pal = BaseColorPalette(colors=d["colors"])
cm = cluster_map_from_ids(d["ids"], pal)
st = SolverState(frame=frame, palette=pal, layers=initialize(frame, cm, pal),
                 aux=build_aux(frame, cm, int(d["seed"])), weights=EnergyWeights(), config=SolveConfig(tol_rel=0.0))
refined, _ = refine_palette(st)
rec = records_array(st.records); g = d["records"]
np.set_printoptions(linewidth=200, precision=4)
for i in range(len(rec)):
    print(i, int(rec[i,0]), "E0 %.8e  E1 %.8e  relE1 %.2e  acc %d/%d a %.3g/%.3g it %d/%d fr %.3e/%.3e" % (
        rec[i,1], rec[i,2], abs(rec[i,2]-g[i,2])/g[i,2], rec[i,3], g[i,3], rec[i,4], g[i,4], rec[i,5], g[i,5], rec[i,7], g[i,7]))
T = st.layers.T.cpu().numpy(); Tg = d["T"]
dT = np.abs(T - Tg)
for k in range(T.shape[2]):
    idx = np.unravel_index(np.argmax(dT[..., k]), dT.shape[:2])
    print("layer", k, "max", dT[...,k].max(), "at", idx, "ours", T[idx][k], "ref", Tg[idx][k], "n>1e-4", int((dT[...,k]>1e-4).sum()), "n>1e-3", int((dT[...,k]>1e-3).sum()))
print("palette diff", np.abs(refined.colors - d["colors_out"]).max())

"""The single-reduction PCG (k_cg_iter, LS_PCG=cg1: one kernel and one
grid-level reduction per PCG iteration, the north star's kernel (2)) against
the oracle and against the default two-kernel textbook loop: same iteration
counts and accept decisions, steps within the GN-step parity gate."""
import os

import numpy as np
import pytest
import torch

from oracle import c_oracle as CO
from oracle import lumisplit_oracle as O

pytestmark = pytest.mark.gpu


def _fresh_contexts():
    """Contexts read LS_PCG when they are created: drop the cached ones."""
    from paper_1908_01961_b200 import _device
    torch.cuda.synchronize()
    _device._cache.clear()


def _state(clip, idx, prev, seed):
    from paper_1908_01961_b200.energy import EnergyWeights
    from paper_1908_01961_b200.imaging import Frame, chromaticity
    from paper_1908_01961_b200.palette import BaseColorPalette, segment
    from paper_1908_01961_b200.solver import SolveConfig, SolverState, build_aux, initialize
    frame = Frame(clip.frames[idx].cuda())
    pal = BaseColorPalette(colors=clip.colors)
    cm = segment(frame, pal)
    if prev is None:
        aux, layers = build_aux(frame, cm, seed), initialize(frame, cm, pal)
    else:
        aux = build_aux(frame, cm, seed, prev_chroma=chromaticity(prev[0]), prev_r=prev[1].r)
        layers = prev[1].copy()
    return SolverState(frame=frame, palette=pal, layers=layers, aux=aux, weights=EnergyWeights(),
                       config=SolveConfig(tol_rel=0.0))


@pytest.mark.parametrize("H,W,K", [(120, 168, 4), (200, 256, 8)])
def test_cg1_gn_steps_match_textbook_and_oracle(H, W, K):
    from paper_1908_01961_b200 import synth
    from paper_1908_01961_b200.solver import gn_step_sparse, _solver_for
    clip = synth.make_clip(H, W, K, 2, seed=5, device="cpu")
    _fresh_contexts()
    s0 = _state(clip, 0, None, 0)          # the previous frame, solved once (default PCG)
    gn_step_sparse(s0)
    runs = {}
    for mode in ("", "cg1"):
        os.environ["LS_PCG"] = mode
        _fresh_contexts()
        try:
            st = _state(clip, 1, (s0.frame, s0.layers), 3)
            assert _solver_for(st).lib is not None
            X0 = st.layers.X.clone()
            recs = [gn_step_sparse(st) for _ in range(3)]
            runs[mode] = (X0, recs, st.layers.X.clone(), st)
        finally:
            os.environ.pop("LS_PCG", None)
    (Xa, ra, Ya, sa), (Xb, rb, Yb, sb) = runs[""], runs["cg1"]
    assert torch.equal(Xa, Xb)
    for a, b in zip(ra, rb):
        assert a["accepted"] == b["accepted"] and a["alpha"] == b["alpha"]
        assert a["pcg"]["iterations"] == b["pcg"]["iterations"] == 16
        assert np.isclose(a["energy_after"], b["energy_after"], rtol=1e-5)
        assert np.isclose(a["pcg"]["final_residual"], b["pcg"]["final_residual"], rtol=1e-3)
    # three free-running GN steps of two PCG formulations: equal up to pixels
    # whose T crosses 0 between them (the non-negativity weight jumps there)
    d = (Ya - Yb).abs()
    assert float((d <= 1e-3).float().mean()) >= 0.999 and float(d.max()) <= 1e-2
    # one cg1 GN step teacher-forced against the oracle
    img1 = clip.frames[1].double().numpy()
    os.environ["LS_PCG"] = "cg1"
    try:
        st = sb
        r0, T0 = st.layers.r.double().cpu().numpy(), st.layers.T.double().cpu().numpy()
        s = st.aux.samples
        pairs = O.Pairs(src=s.src.cpu().numpy(), dst=s.dst.cpu().numpy(), temporal=s.temporal.cpu().numpy(),
                        weight=np.ones(len(s.src)), shape=(H, W))
        oaux = O.Aux(edge=st.aux.edge_weights.double().cpu().numpy(), pairs=pairs,
                     prev_r=st.aux.prev_r.double().cpu().numpy(), cluster_ids=st.aux.cluster_ids.cpu().numpy())
        ost = O.State(image=img1, colors=np.asarray(clip.colors), r=r0, T=T0, aux=oaux, weights=O.Weights(),
                      config=O.Config(tol_rel=0.0))
        orec = CO.gn_step_sparse(ost)
        rec = gn_step_sparse(st)
    finally:
        os.environ.pop("LS_PCG", None)
        _fresh_contexts()
    assert rec["accepted"] == orec["accepted"] and rec["pcg"]["iterations"] == orec["pcg"]["iterations"]
    assert np.isclose(rec["energy_after"], orec["energy_after"], rtol=1e-4)
    dT = np.abs(st.layers.T.double().cpu().numpy() - ost.T).max()
    dR = np.abs(np.exp(st.layers.r.double().cpu().numpy()) - np.exp(ost.r)).max()
    assert dT <= 1e-3 and dR <= 1e-3, (dT, dR)


def test_cg1_streaming_graph_equals_eager():
    from paper_1908_01961_b200 import synth
    from paper_1908_01961_b200.energy import EnergyWeights
    from paper_1908_01961_b200.palette import BaseColorPalette
    from paper_1908_01961_b200.pipeline import StreamingDecomposer
    from paper_1908_01961_b200.solver import SolveConfig
    clip = synth.make_clip(104, 136, 4, 3, seed=6, device="cpu")
    runs = []
    for no_graph in ("", "1"):
        os.environ["LS_PCG"] = "cg1"
        os.environ["LS_NO_GRAPH"] = no_graph
        _fresh_contexts()
        try:
            dec = StreamingDecomposer(BaseColorPalette(colors=clip.colors), EnergyWeights(),
                                      SolveConfig(tol_rel=0.0, refine=False, outer_iterations=2))
            sts = [dec.first(clip.frames[0].cuda())] + [dec.step(f.cuda()) for f in clip.frames[1:]]
            runs.append([(s.records, s.layers.X.clone()) for s in sts])
        finally:
            os.environ.pop("LS_PCG", None)
            os.environ.pop("LS_NO_GRAPH", None)
    _fresh_contexts()
    for (ra, Xa), (rb, Xb) in zip(*runs):
        assert ra == rb and torch.equal(Xa, Xb)

"""Row bands (bands.py) on one GPU: the band-partitioned
solve against the whole-frame solve on the same inputs.

* 1 band in band-partial mode is bitwise the whole-frame path;
* n bands: segmentation bitwise (dark-pixel inheritance across band
  boundaries), partner draws identical (energies equal to fp64 rounding),
  GN / dense steps equal up to the grouping of the fp64 reductions;
* a banded streaming clip stays within the frame-1 parity gate of the
  whole-frame clip."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _clip(H, W, K, n=2, seed=0):
    from paper_1908_01961_b200 import synth
    return synth.make_clip(H, W, K, n, seed=seed, device="cpu")


def _state(clip, idx=0, bands=0, prev=None, seed=0, refine=False):
    from dataclasses import replace
    from paper_1908_01961_b200.energy import EnergyWeights
    from paper_1908_01961_b200.imaging import Frame, chromaticity
    from paper_1908_01961_b200.palette import BaseColorPalette, segment
    from paper_1908_01961_b200.solver import SolveConfig, SolverState, build_aux, initialize
    frame = Frame(clip.frames[idx].cuda(), bands=bands)
    pal = BaseColorPalette(colors=clip.colors)
    cm = segment(frame, pal)
    if prev is None:
        aux = build_aux(frame, cm, seed)
        layers = initialize(frame, cm, pal)
    else:
        pframe, players = prev
        aux = build_aux(frame, cm, seed, prev_chroma=chromaticity(pframe), prev_r=players.r)
        layers = players.copy()
    cfg = replace(SolveConfig(tol_rel=0.0), refine=refine)
    return SolverState(frame=frame, palette=pal, layers=layers, aux=aux,
                       weights=EnergyWeights(), config=cfg)


@pytest.mark.parametrize("n", [2, 3, 5])
def test_band_segment_bit_exact_with_dark_runs(n):
    from paper_1908_01961_b200.bands import BandedSolver
    from paper_1908_01961_b200.palette import BaseColorPalette, segment
    from paper_1908_01961_b200.imaging import Frame
    clip = _clip(200, 96, 4, n=1, seed=2)
    img = clip.frames[0].clone()
    img[:13] = 0.0                 # dark top: ids come from the frame's first non-dark pixel
    img[60:130, :] = 0.001         # dark run across band boundaries
    img[140:150, 10:50] = 0.0
    img = img.cuda()
    ref = segment(Frame(img), BaseColorPalette(colors=clip.colors)).ids
    bs = BandedSolver(img.device, 200, 96, 4, n=n)
    ids = bs.segment(img, clip.colors)
    assert torch.equal(ids, ref.to(torch.int32))


def test_one_band_is_bitwise_the_whole_frame_path():
    from paper_1908_01961_b200.solver import gn_step_sparse
    clip = _clip(120, 160, 4, n=1, seed=1)
    a, b = _state(clip), _state(clip, bands=1)
    b.layers.X.copy_(a.layers.X)
    ra, rb = gn_step_sparse(a), gn_step_sparse(b)
    assert ra == rb
    assert torch.equal(a.layers.X, b.layers.X)


@pytest.mark.parametrize("n", [2, 4])
def test_banded_energy_and_gn_step_match_whole_frame(n):
    from paper_1908_01961_b200.solver import gn_step_sparse, _solver_for
    clip = _clip(256, 320, 6, n=2, seed=3)
    # streaming frame (temporal partners + prev_r) from a whole-frame solve of frame 0
    s0 = _state(clip)
    gn_step_sparse(s0)
    prev = (s0.frame, s0.layers)
    a = _state(clip, 1, prev=prev, seed=7)
    b = _state(clip, 1, bands=n, prev=prev, seed=7)
    ea = _solver_for(a).energy_terms(a.palette.colors, a.layers.X)
    eb = _solver_for(b).energy_terms(b.palette.colors, b.layers.X)
    np.testing.assert_allclose(eb, ea, rtol=1e-12, atol=1e-9)     # same partners, same terms
    for _ in range(2):
        ra, rb = gn_step_sparse(a), gn_step_sparse(b)
        assert ra["accepted"] == rb["accepted"]
        assert abs(rb["energy_after"] - ra["energy_after"]) <= 1e-6 * ra["energy_after"]
        assert ra["pcg"]["iterations"] == rb["pcg"]["iterations"]
    d = (a.layers.X - b.layers.X).abs()
    assert float(d.max()) <= 1e-3
    assert float((d > 1e-5).float().mean()) <= 1e-3


def test_banded_dense_step_matches_whole_frame():
    from paper_1908_01961_b200.solver import gn_step_sparse, solve_dense_block
    clip = _clip(192, 256, 4, n=1, seed=6)
    a, b = _state(clip), _state(clip, bands=3)
    b.layers.X.copy_(a.layers.X)
    gn_step_sparse(a)
    b.layers.X.copy_(a.layers.X)
    da, db = solve_dense_block(a), solve_dense_block(b)
    np.testing.assert_allclose(db, da, rtol=1e-9, atol=1e-12)
    assert a.records[-1]["accepted"] == b.records[-1]["accepted"]
    np.testing.assert_allclose(b.palette.colors, a.palette.colors, rtol=1e-9, atol=1e-12)


def test_banded_streaming_clip_within_parity_gate():
    from paper_1908_01961_b200.energy import EnergyWeights
    from paper_1908_01961_b200.palette import BaseColorPalette
    from paper_1908_01961_b200.pipeline import StreamingDecomposer
    from paper_1908_01961_b200.solver import SolveConfig
    clip = _clip(240, 320, 4, n=3, seed=9)
    out = []
    for bands in (0, 4):
        dec = StreamingDecomposer(BaseColorPalette(colors=clip.colors), EnergyWeights(),
                                  SolveConfig(tol_rel=0.0), seed=0, bands=bands)
        sts = [dec.first(clip.frames[0].cuda())] + [dec.step(f.cuda()) for f in clip.frames[1:]]
        out.append(sts)
    for a, b in zip(*out):
        assert [r["phase"] for r in a.records] == [r["phase"] for r in b.records]
        np.testing.assert_allclose(b.palette.colors, a.palette.colors, atol=1e-3)
        d = (a.layers.X - b.layers.X).abs()
        assert float((d <= 1e-3).float().mean()) >= 0.999
        ea, eb = a.energy_history[-1], b.energy_history[-1]
        assert abs(ea - eb) <= 1e-4 * ea


def test_banded_device_flip_flop_matches_host_loop_and_graph():
    """The device-resident band flip-flop (decisions on the device, one CUDA
    graph per frame) equals the host-driven band loop bit for bit, with and
    without the graph, and every band reports the same records."""
    import os
    from paper_1908_01961_b200.bands import banded_solver
    from paper_1908_01961_b200.solver import _solver_for, gn_step_sparse
    clip = _clip(200, 128, 4, n=2, seed=4)
    s0 = _state(clip)
    gn_step_sparse(s0)
    st = _state(clip, 1, bands=3, prev=(s0.frame, s0.layers), seed=5)
    bs = _solver_for(st)
    X0 = st.layers.X.clone()
    outs = []
    for mode in ("host", "graph", "eager"):
        if mode == "host":
            outs.append(bs.flip_flop_stream_host(st.palette.colors, X0, 2, 2, 1e-3))
        else:
            outs.append(bs.flip_flop_stream(st.palette.colors, X0, 2, 2, 1e-3, graph=(mode == "graph")))
    ref = outs[0]
    for rc, recs, status, X, fault in outs[1:]:
        assert rc == ref[0] and status == ref[2] and len(recs) == len(ref[1])
        for a, b in zip(recs, ref[1]):
            assert (a.accepted, a.energy_before, a.energy_after, a.alpha, a.pcg_iterations) == \
                   (b.accepted, b.energy_before, b.energy_after, b.alpha, b.pcg_iterations)
            assert list(a.terms) == list(b.terms)
        assert torch.equal(X, ref[3])
    # a second graph replay (next frame) still matches the eager path
    r2g = bs.flip_flop_stream(st.palette.colors, outs[1][3], 2, 2, 1e-3, graph=True)
    r2e = bs.flip_flop_stream(st.palette.colors, outs[1][3], 2, 2, 1e-3, graph=False)
    assert torch.equal(r2g[3], r2e[3])


def test_banded_graph_recaptured_when_frame_state_changes():
    """frame 1 without refinement and with outer_iterations equal to
    the streaming count captures the band graph with no previous-frame
    reflectance; frame 2 (temporal partners) must not replay that graph.
    Banded and whole-frame clips agree frame by frame."""
    from paper_1908_01961_b200.energy import EnergyWeights
    from paper_1908_01961_b200.palette import BaseColorPalette
    from paper_1908_01961_b200.pipeline import StreamingDecomposer
    from paper_1908_01961_b200.solver import SolveConfig
    clip = _clip(160, 192, 4, n=3, seed=11)
    cfg = SolveConfig(tol_rel=0.0, refine=False, outer_iterations=2)
    out = []
    for bands in (0, 3):
        dec = StreamingDecomposer(BaseColorPalette(colors=clip.colors), EnergyWeights(), cfg,
                                  seed=0, streaming_outer=2, bands=bands)
        sts = [dec.first(clip.frames[0].cuda())] + [dec.step(f.cuda()) for f in clip.frames[1:]]
        torch.cuda.synchronize()
        out.append(sts)
    for a, b in zip(*out):
        assert len(a.records) == len(b.records)
        for ra, rb in zip(a.records, b.records):
            assert ra["accepted"] == rb["accepted"]
            assert abs(ra["energy_after"] - rb["energy_after"]) <= 1e-6 * ra["energy_after"]
        d = (a.layers.X - b.layers.X).abs()
        assert float((d <= 1e-3).float().mean()) >= 0.999


def test_banded_graph_key_tracks_weights():
    """Changing the energy weights between frames re-captures the band graph
    (the weights are baked into the kernels' arguments)."""
    from paper_1908_01961_b200.bands import banded_solver
    from paper_1908_01961_b200.energy import EnergyWeights
    from paper_1908_01961_b200.solver import SolveConfig, _solver_for, gn_step_sparse
    clip = _clip(160, 128, 4, n=2, seed=12)
    s0 = _state(clip)
    gn_step_sparse(s0)
    st = _state(clip, 1, bands=2, prev=(s0.frame, s0.layers), seed=3)
    bs = _solver_for(st)
    X0 = st.layers.X.clone()
    g1 = bs.flip_flop_stream(st.palette.colors, X0, 1, 2, 0.0, graph=True)
    bs.configure(EnergyWeights(lambda_smoothness=30.0), SolveConfig(tol_rel=0.0))
    g2 = bs.flip_flop_stream(st.palette.colors, X0, 1, 2, 0.0, graph=True)
    e2 = bs.flip_flop_stream(st.palette.colors, X0, 1, 2, 0.0, graph=False)
    assert torch.equal(g2[3], e2[3])
    assert not torch.equal(g1[3], g2[3])

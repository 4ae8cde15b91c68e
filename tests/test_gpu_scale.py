"""GPU tests at full size and on the less common code paths:
1080p bit-exact sampler / segmentation vs the oracle, operator symmetry,
bitwise determinism, TMA vs cooperative-load paths, K = 0 and K = 12
instantiations, non-default weights (p != 1, identity chroma regulariser)."""
import os

import numpy as np
import pytest
import torch

from oracle import lumisplit_oracle as O

pytestmark = pytest.mark.gpu


def _clip(H, W, K, n=2, seed=0):
    from paper_1908_01961_b200 import synth
    return synth.make_clip(H, W, K, n, seed=seed, device="cpu")


def _state(clip, idx=0, prev=None, weights=None, seed=0):
    from paper_1908_01961_b200.energy import EnergyWeights
    from paper_1908_01961_b200.imaging import Frame, chromaticity
    from paper_1908_01961_b200.palette import BaseColorPalette, segment
    from paper_1908_01961_b200.solver import SolveConfig, SolverState, build_aux, initialize
    frame = Frame(clip.frames[idx].cuda())
    pal = BaseColorPalette(colors=clip.colors)
    cm = segment(frame, pal)
    if prev is None:
        aux = build_aux(frame, cm, seed)
        layers = initialize(frame, cm, pal)
    else:
        pframe, players = prev
        aux = build_aux(frame, cm, seed, prev_chroma=chromaticity(pframe), prev_r=players.r)
        layers = players.copy()
    return SolverState(frame=frame, palette=pal, layers=layers, aux=aux,
                       weights=weights or EnergyWeights(), config=SolveConfig(tol_rel=0.0))


def test_1080p_sampler_and_segment_bit_exact():
    clip = _clip(1080, 1920, 8, n=2, seed=4)
    from paper_1908_01961_b200.imaging import Frame, chromaticity
    from paper_1908_01961_b200.energy import sample_consistency
    from paper_1908_01961_b200.palette import segment, BaseColorPalette
    f0, f1 = (Frame(f.cuda()) for f in clip.frames)
    c0, c1 = chromaticity(f0), chromaticity(f1)
    s = sample_consistency(c1, c0, 11)
    img0 = clip.frames[0].double().numpy()
    img1 = clip.frames[1].double().numpy()
    ref = O.sample_pairs(O.chromaticity(img1)[0], O.chromaticity(img0)[0], 11)
    assert np.array_equal(s.src.cpu().numpy(), ref.src)
    assert np.array_equal(s.dst.cpu().numpy(), ref.dst)
    assert np.array_equal(s.temporal.cpu().numpy(), ref.temporal)
    ids = segment(f1, BaseColorPalette(colors=clip.colors)).ids.cpu().numpy()
    assert np.array_equal(ids, O.segment(img1, clip.colors))


def test_1080p_sampler_with_a_rejection_bit_exact():
    """Seed 95's u32 stream has a zero word at 16,473,226 (< 8 N at 1080p:
    a Lemire rejection in the dy draws; tools/find_rejection_seed.py).  The
    device finds it, shifts the rest of the stream and redraws: the threads of
    the warp holding the zero seek by the full jump, every other thread from
    its warp's base state.  Pairs equal numpy's, with and without the temporal
    section (which the shift moves as well)."""
    clip = _clip(1080, 1920, 8, n=2, seed=4)
    from paper_1908_01961_b200.imaging import Frame, chromaticity
    from paper_1908_01961_b200.energy import sample_consistency
    f0, f1 = (Frame(f.cuda()) for f in clip.frames)
    c0, c1 = chromaticity(f0), chromaticity(f1)
    img0 = clip.frames[0].double().numpy()
    img1 = clip.frames[1].double().numpy()
    oc0, oc1 = O.chromaticity(img0)[0], O.chromaticity(img1)[0]
    for prev, oprev in ((None, None), (c0, oc0)):
        s = sample_consistency(c1, prev, 95)
        ref = O.sample_pairs(oc1, oprev, 95)
        assert np.array_equal(s.src.cpu().numpy(), ref.src)
        assert np.array_equal(s.dst.cpu().numpy(), ref.dst)
        assert np.array_equal(s.temporal.cpu().numpy(), ref.temporal)


def test_sampled_adjacency_rows_in_reference_order():
    """The sampled adjacency (k_fill_samples + incoming segments sorted by
    entry code) orders every row exactly as the explicit-pairs path
    (ls_set_pairs: own pairs, then incoming ones by pair index = source
    pixel, slot), so the operator's fixed-order consistency sums agree bit
    for bit -- at 1080p, with temporal partners."""
    from paper_1908_01961_b200.solver import _solver_for
    clip = _clip(1080, 1920, 8, n=2, seed=4)
    st0 = _state(clip)
    st = _state(clip, idx=1, prev=(st0.frame, st0.layers), seed=7)
    s = _solver_for(st)
    g = torch.Generator(device="cpu").manual_seed(3)
    p = torch.randn(st.layers.X.shape, generator=g).to(st.layers.X.device)
    w_sampled = s.apply(st.palette.colors, st.layers.X, p)
    from paper_1908_01961_b200.energy import _guard_csr
    src, dst, tmp = s.get_pairs()
    _guard_csr(s)
    s.set_pairs(src, dst, tmp)
    w_pairs = s.apply(st.palette.colors, st.layers.X, p)
    s.installed = None            # the context's adjacency is no longer the aux's
    assert torch.equal(w_sampled, w_pairs)


def test_1080p_operator_symmetric_and_step_deterministic():
    from paper_1908_01961_b200.energy import assemble_blocks
    from paper_1908_01961_b200.solver import gn_step_sparse
    clip = _clip(1080, 1920, 8, n=1, seed=5)
    st = _state(clip)
    blocks = assemble_blocks(st.frame, st.palette, st.layers, st.aux, st.weights)
    g = torch.Generator(device="cuda").manual_seed(0)
    p = torch.randn(st.layers.X.shape, device="cuda", generator=g)
    q = torch.randn(st.layers.X.shape, device="cuda", generator=g)
    Ap, Aq = blocks.apply_normal(p), blocks.apply_normal(q)
    a = float((q.double() * Ap.double()).sum())
    b = float((p.double() * Aq.double()).sum())
    assert abs(a - b) <= 1e-5 * max(abs(a), abs(b))
    assert float((p.double() * Ap.double()).sum()) > 0       # J^T J is PSD
    X0 = st.layers.X.clone()
    r1 = gn_step_sparse(st)
    X1 = st.layers.X.clone()
    st2 = _state(clip)
    st2.layers.X.copy_(X0)
    r2 = gn_step_sparse(st2)
    assert r1["energy_after"] == r2["energy_after"] and r1["accepted"]
    assert torch.equal(X1, st2.layers.X)
    assert r1["energy_after"] < r1["energy_before"]


def test_tma_and_cooperative_paths_identical():
    """Same problem through the TMA pipeline and the cooperative-load path
    (LS_NO_TMA): bitwise identical operator, gradient and GN step."""
    from paper_1908_01961_b200 import _device
    from paper_1908_01961_b200.energy import assemble_blocks
    from paper_1908_01961_b200.solver import gn_step_sparse
    clip = _clip(72, 136, 5, n=1, seed=6)
    outs = []
    for no_tma in (False, True):
        _device.clear_cache()
        if no_tma:
            os.environ["LS_NO_TMA"] = "1"
        try:
            st = _state(clip)
            blocks = assemble_blocks(st.frame, st.palette, st.layers, st.aux, st.weights)
            p = torch.linspace(-1, 1, st.layers.X.numel(), device="cuda").reshape(st.layers.X.shape)
            Ap = blocks.apply_normal(p)
            b, d = blocks.gradient_and_diag()
            e = blocks.energies()
            rec = gn_step_sparse(st)
            outs.append((Ap, b, d, e, rec["energy_after"], st.layers.X.clone()))
        finally:
            os.environ.pop("LS_NO_TMA", None)
            _device.clear_cache()
    (Ap0, b0, d0, e0, ea0, X0), (Ap1, b1, d1, e1, ea1, X1) = outs
    assert torch.equal(Ap0, Ap1) and torch.equal(b0, b1) and torch.equal(d0, d1)
    assert e0 == e1 and ea0 == ea1
    assert torch.equal(X0, X1)


@pytest.mark.parametrize("K", [1, 12])
def test_extreme_K_gn_step_matches_oracle(K):
    from paper_1908_01961_b200.solver import gn_step_sparse
    clip = _clip(40, 52, K, n=1, seed=7)
    st = _state(clip)
    r0 = st.layers.r.double().cpu().numpy()
    T0 = st.layers.T.double().cpu().numpy()
    rec = gn_step_sparse(st)
    img = clip.frames[0].double().numpy()
    ids = st.aux.cluster_ids.cpu().numpy()
    ost = O.State(image=img, colors=clip.colors, r=r0, T=T0, aux=O.build_aux(img, ids, 0),
                  weights=O.Weights(), config=O.Config())
    orec = O.gn_step_sparse(ost)
    assert rec["accepted"] == orec["accepted"]
    assert np.isclose(rec["energy_before"], orec["energy_before"], rtol=1e-5)
    assert np.isclose(rec["energy_after"], orec["energy_after"], rtol=1e-4)
    assert np.max(np.abs(st.layers.T.double().cpu().numpy() - ost.T)) < 1e-3


def test_k0_direct_layer_only():
    """K = 0 (white illuminant only), as test_solver.py:72-100 uses."""
    from paper_1908_01961_b200.energy import ConsistencySamples, EnergyAux, EnergyWeights, LayerStack
    from paper_1908_01961_b200.imaging import Frame, chromaticity
    from paper_1908_01961_b200.energy import chroma_edge_weights, sample_consistency
    from paper_1908_01961_b200.palette import BaseColorPalette
    from paper_1908_01961_b200.solver import SolveConfig, SolverState, gn_step_sparse
    h = w = 8
    rng = np.random.default_rng(3)
    image = np.clip(rng.uniform(0.2, 0.9, size=(h, w, 3)), 0, 1).astype(np.float32)
    frame = Frame(torch.as_tensor(image, device="cuda"))
    R = np.full((h, w, 3), 0.7, dtype=np.float32)
    layers = LayerStack(torch.as_tensor(np.log(R), device="cuda"),
                        torch.full((h, w, 1), 0.1, device="cuda"))
    ch = chromaticity(frame)
    aux = EnergyAux(edge_weights=chroma_edge_weights(ch), samples=sample_consistency(ch, None, 0),
                    r_cluster_log=torch.as_tensor(np.log(R), device="cuda"))
    weights = EnergyWeights(lambda_clustering=1e12, lambda_r_sparsity=0, lambda_r_consistency=0,
                            lambda_monochrome=0, lambda_i_sparsity=0, lambda_smoothness=0, lambda_non_neg=0)
    st = SolverState(frame=frame, palette=BaseColorPalette(colors=np.zeros((0, 3))), layers=layers,
                     aux=aux, weights=weights, config=SolveConfig(pcg_iterations=16))
    gn_step_sparse(st)
    S0 = 0.1
    num = (R * (image - R * S0)).sum(axis=2)
    den = (R ** 2).sum(axis=2)
    expected = 0.1 + num / den
    assert np.max(np.abs(st.layers.T[:, :, 0].cpu().numpy() - expected)) < 1e-5


def test_nondefault_weights_match_oracle():
    from paper_1908_01961_b200.energy import EnergyWeights, assemble_blocks, to_reference_vector
    clip = _clip(36, 44, 3, n=1, seed=8)
    w = EnergyWeights(p=0.8, chroma_reg="identity", lambda_r_consistency=25.0, eps_irls=0.05)
    st = _state(clip, weights=w)
    blocks = assemble_blocks(st.frame, st.palette, st.layers, st.aux, w)
    img = clip.frames[0].double().numpy()
    ids = st.aux.cluster_ids.cpu().numpy()
    ow = O.Weights(p=0.8, chroma_reg="identity", lambda_r_consistency=25.0, eps_irls=0.05)
    osys = O.FrozenSystem(img, clip.colors, st.layers.r.double().cpu().numpy(),
                          st.layers.T.double().cpu().numpy(), O.build_aux(img, ids, 0), ow)
    e = blocks.energies()
    et = osys.terms(osys.r0, osys.T0)
    for k in O.TERM_NAMES:
        assert np.isclose(e[k], et[k], rtol=1e-5, atol=1e-9), k
    b, d = blocks.gradient_and_diag()
    ob, od = osys.grad_diag()
    bv = to_reference_vector(b).cpu().numpy()
    assert np.max(np.abs(bv - ob)) / np.max(np.abs(ob)) < 1e-5
    from paper_1908_01961_b200.energy import refine_normal_system
    A, rhs = refine_normal_system(st.frame, st.layers, st.palette, w, cluster_ids=st.aux.cluster_ids)
    oA, orhs = O.refine_normal_system(img, osys.r0, osys.T0, clip.colors, ow, ids)
    assert np.max(np.abs(A - oA)) / np.max(np.abs(oA)) < 1e-9


def test_device_flip_flop_equals_host_loop():
    """The device-resident streaming flip-flop makes the same decisions and
    produces the same state (bitwise) as the host-driven loop of
    solver.py:311-338, including the convergence test."""
    from dataclasses import replace
    from paper_1908_01961_b200 import solver as S
    clip = _clip(64, 96, 4, n=2, seed=9)
    outs = []
    for dev in (True, False):
        S.DEVICE_FLIP_FLOP = dev
        try:
            st0 = _state(clip)
            st0.config = replace(st0.config, refine=False, outer_iterations=2)
            S.flip_flop(st0)
            st = _state(clip, idx=1, prev=(st0.frame, st0.layers), seed=1)
            st.config = replace(st.config, refine=False, outer_iterations=6, tol_rel=2e-3)
            S.flip_flop(st)
            outs.append((st.records, st.status, st.layers.X.clone(), st.energy_history))
        finally:
            S.DEVICE_FLIP_FLOP = True
    (r0, s0, X0, h0), (r1, s1, X1, h1) = outs
    assert s0 == s1 and len(r0) == len(r1) and h0 == h1
    for a, b in zip(r0, r1):
        assert a == b
    assert torch.equal(X0, X1)


def test_graph_flip_flop_equals_eager_and_replays():
    """ls_flip_flop_graph (one CUDA-graph launch, captured once and replayed
    for the next frames) gives the eager ls_flip_flop_stream's records and
    state bit for bit, frame after frame."""
    import os
    from paper_1908_01961_b200.energy import EnergyWeights
    from paper_1908_01961_b200.palette import BaseColorPalette
    from paper_1908_01961_b200.pipeline import StreamingDecomposer
    from paper_1908_01961_b200.solver import SolveConfig
    clip = _clip(96, 128, 4, n=4, seed=12)
    runs = []
    for no_graph in ("", "1"):
        os.environ["LS_NO_GRAPH"] = no_graph
        try:
            dec = StreamingDecomposer(BaseColorPalette(colors=clip.colors), EnergyWeights(),
                                      SolveConfig(tol_rel=0.0, refine=False, outer_iterations=2))
            sts = [dec.first(clip.frames[0].cuda())] + [dec.step(f.cuda()) for f in clip.frames[1:]]
            runs.append([(s.records, s.status, s.layers.X.clone()) for s in sts])
        finally:
            os.environ.pop("LS_NO_GRAPH", None)
    for (ra, sa, Xa), (rb, sb, Xb) in zip(*runs):
        assert ra == rb and sa == sb
        assert torch.equal(Xa, Xb)


def test_graph_conditional_halvings_equal_eager(monkeypatch):
    """Opt-in LS_GRAPH_COND=1: the line-search halvings captured as graph
    conditional nodes (a trial's last CTA enables its successor) give the
    eager path's records and state bit for bit -- from rough starting states
    that make the search halve and reject."""
    import numpy as np
    from paper_1908_01961_b200 import _device
    from paper_1908_01961_b200.energy import install
    monkeypatch.setenv("LS_GRAPH_COND", "1")
    clip = _clip(64, 96, 3, n=2, seed=13)
    st = _state(clip, idx=1)
    H, W, K = st.frame.height, st.frame.width, st.palette.K
    from dataclasses import replace
    from paper_1908_01961_b200.energy import EnergyWeights
    s = _device.DeviceSolver(st.layers.X.device, H, W, K)      # created with the variable set
    g = torch.Generator(device="cpu").manual_seed(5)
    halved = 0
    for w, iters in ((st.weights, 16), (EnergyWeights(p=0.5, eps_irls=1e-3), 2), (EnergyWeights(p=0.3), 1)):
        s.configure(w, replace(st.config, pcg_iterations=iters))
        install(s, st.frame, st.aux)
        for scale in (0.0, 1.0, 4.0):
            X0 = st.layers.X.clone()
            X0 += scale * torch.randn(X0.shape, generator=g).to(X0.device)
            rg = s.flip_flop_stream(st.palette.colors, X0, 2, 2, 0.0, graph=True)
            re = s.flip_flop_stream(st.palette.colors, X0, 2, 2, 0.0, graph=False)
            assert torch.equal(rg[3], re[3])
            assert [(r.energy_after, r.alpha, r.accepted) for r in rg[1]] == \
                [(r.energy_after, r.alpha, r.accepted) for r in re[1]]
            halved += sum(1 for r in re[1] if r.alpha != 1.0)
    assert halved > 0, "no halving exercised"


def test_context_image_reinstalled_after_in_place_edit_and_in_inference_mode():
    """A context skips ls_set_image for the tensor it already holds,
    unmodified: an in-place edit (torch's version counter moves) must be seen,
    and inference tensors (no version counter) are never skipped."""
    from paper_1908_01961_b200.imaging import Frame
    from paper_1908_01961_b200.palette import BaseColorPalette, segment
    clip = _clip(48, 64, 3, n=2, seed=17)
    pal = BaseColorPalette(colors=clip.colors)
    f = Frame(clip.frames[0].cuda())
    segment(f, pal)
    f.data.copy_(clip.frames[1].cuda())               # same tensor, new contents
    ids_edit = segment(f, pal).ids
    ids_fresh = segment(Frame(clip.frames[1].cuda()), pal).ids
    assert torch.equal(ids_edit, ids_fresh)
    with torch.inference_mode():
        g = Frame(clip.frames[0].cuda())
        a = segment(g, pal).ids.clone()
        g.data.copy_(clip.frames[1].cuda())
        b = segment(g, pal).ids
    assert torch.equal(b, ids_fresh) and not torch.equal(a, b)


def test_graph_recaptures_when_the_palette_changes():
    """The captured flip-flop bakes the palette into its kernels: a new
    palette must re-capture (results equal the eager path for A, B, A)."""
    import numpy as np
    from paper_1908_01961_b200 import _device
    clip = _clip(64, 96, 3, n=2, seed=13)
    st = _state(clip, idx=1)
    from paper_1908_01961_b200.solver import _solver_for
    s = _solver_for(st)
    A = st.palette.colors
    B = np.clip(A * 0.9 + 0.05, 0.0, 1.0)
    for cols in (A, B, A):
        rg = s.flip_flop_stream(cols, st.layers.X, 1, 2, 0.0, graph=True)
        re = s.flip_flop_stream(cols, st.layers.X, 1, 2, 0.0, graph=False)
        assert torch.equal(rg[3], re[3])
        assert [r.energy_after for r in rg[1]] == [r.energy_after for r in re[1]]


def test_cfg2_streaming_steps_teacher_forced_vs_oracle():
    """configs[1] size (640x480, K=6) with temporal partners: two streaming GN
    steps on the device against the oracle from the same input state and aux
    (partners bit-exact), per-layer max-abs <= 1e-3, energies within 1e-5."""
    from paper_1908_01961_b200.solver import gn_step_sparse
    clip = _clip(480, 640, 6, n=2, seed=21)
    st0 = _state(clip)                                  # frame 0 initial state
    r_prev = st0.layers.r.double().cpu().numpy()
    st = _state(clip, idx=1, prev=(st0.frame, st0.layers), seed=3)
    img0 = clip.frames[0].double().numpy()
    img1 = clip.frames[1].double().numpy()
    ids1 = st.aux.cluster_ids.cpu().numpy()
    oaux = O.build_aux(img1, ids1, 3, O.chromaticity(img0)[0], r_prev)
    s = st.aux.samples
    assert np.array_equal(s.src.cpu().numpy(), oaux.pairs.src)
    assert np.array_equal(s.temporal.cpu().numpy(), oaux.pairs.temporal)
    for _ in range(2):
        r0 = st.layers.r.double().cpu().numpy()
        T0 = st.layers.T.double().cpu().numpy()
        ost = O.State(image=img1, colors=np.asarray(clip.colors, dtype=np.float64), r=r0, T=T0, aux=oaux,
                      weights=O.Weights(), config=O.Config(tol_rel=0.0))
        orec = O.gn_step_sparse(ost)
        rec = gn_step_sparse(st)
        assert rec["accepted"] == orec["accepted"]
        assert np.isclose(rec["energy_before"], orec["energy_before"], rtol=1e-5)
        assert np.isclose(rec["energy_after"], orec["energy_after"], rtol=1e-5)
        dT = np.abs(st.layers.T.double().cpu().numpy() - ost.T).max()
        dR = np.abs(np.exp(st.layers.r.double().cpu().numpy()) - np.exp(ost.r)).max()
        assert dT <= 1e-3 and dR <= 1e-3, (dT, dR)
        st.layers.X.copy_(torch.as_tensor(np.concatenate([ost.r.transpose(2, 0, 1), ost.T.transpose(2, 0, 1)]),
                                          dtype=torch.float32, device="cuda"))      # teacher forcing


@pytest.mark.parametrize("graph", [True, False])
def test_streaming_fault_raises_with_dump(graph):
    """A non-finite state in a streaming frame raises NumericalFaultError
    with the reference's dump (solver.py:153-157) through the device-resident
    flip-flop, graph or eager, and the next frame still solves."""
    import os
    from dataclasses import replace
    from paper_1908_01961_b200.solver import NumericalFaultError, flip_flop
    clip = _clip(48, 64, 3, n=2, seed=17)
    os.environ["LS_NO_GRAPH"] = "" if graph else "1"
    try:
        st = _state(clip)
        st.config = replace(st.config, refine=False, outer_iterations=2)
        st.layers.X[1, 5, 7] = float("nan")
        with pytest.raises(NumericalFaultError) as exc:
            flip_flop(st)
        assert exc.value.dump["iteration"] == 0 and set(exc.value.dump["terms"]) >= {"data", "smoothness"}
        ok = _state(clip)
        ok.config = replace(ok.config, refine=False, outer_iterations=2)
        flip_flop(ok)
        assert ok.records and all(np.isfinite(r["energy_after"]) for r in ok.records)
    finally:
        os.environ.pop("LS_NO_GRAPH", None)


@pytest.mark.parametrize("no_graph", ["", "1"])
def test_streaming_step_leaves_previous_frame_untouched(no_graph):
    """StreamingDecomposer.step warm-starts from the previous frame's planes
    without a copy: the previous frame's layers must come out unchanged and
    the new frame must own a new tensor (graph and eager flip-flops)."""
    from paper_1908_01961_b200.energy import EnergyWeights
    from paper_1908_01961_b200.palette import BaseColorPalette
    from paper_1908_01961_b200.pipeline import StreamingDecomposer
    from paper_1908_01961_b200.solver import SolveConfig
    clip = _clip(64, 96, 3, n=3, seed=19)
    os.environ["LS_NO_GRAPH"] = no_graph
    try:
        dec = StreamingDecomposer(BaseColorPalette(colors=clip.colors), EnergyWeights(),
                                  SolveConfig(tol_rel=0.0, outer_iterations=2))
        s0 = dec.first(clip.frames[0].cuda())
        X0 = s0.layers.X.clone()
        s1 = dec.step(clip.frames[1].cuda())
        X1 = s1.layers.X.clone()
        s2 = dec.step(clip.frames[2].cuda())
        torch.cuda.synchronize()
        assert torch.equal(s0.layers.X, X0) and torch.equal(s1.layers.X, X1)
        assert s1.layers.X.data_ptr() != s0.layers.X.data_ptr()
        assert s2.layers.X.data_ptr() != s1.layers.X.data_ptr()
    finally:
        os.environ.pop("LS_NO_GRAPH", None)

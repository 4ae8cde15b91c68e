"""GPU parity of the sm_100a path (through the C ABI) against the reference's
golden fixtures and the CPU oracle.  Mirrors the reference's hot-path golden
suite.

Tolerances: the device stores state and PCG vectors in fp32, computes per
pixel in fp32 (data residual exactly rounded) and reduces in fp64 (DESIGN.md
"Numerics"); operator outputs are compared at 1e-5 relative, solver steps at
the north-star gate (per-layer max-abs <= 1e-3, relative reconstruction
energy <= 1e-4).
"""
from dataclasses import replace

import numpy as np
import pytest
import torch

from oracle import lumisplit_oracle as O
from tests.golden_io import load, oracle_aux, oracle_system, records_array

pytestmark = pytest.mark.gpu

OPS = ["ops_a", "ops_b", "ops_c", "ops_d"]


def lib():
    from paper_1908_01961_b200 import energy, solver, palette, imaging, refine, pipeline  # noqa
    import paper_1908_01961_b200 as P
    return P


def rel(a, b):
    a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
    b = b.detach().cpu().numpy() if isinstance(b, torch.Tensor) else np.asarray(b)
    return float(np.max(np.abs(a.astype(np.float64) - b)) / max(np.max(np.abs(b)), 1e-300))


def device_problem(d):
    from paper_1908_01961_b200.energy import (ConsistencySamples, EnergyAux, LayerStack,
                                              EnergyWeights, assemble_blocks)
    from paper_1908_01961_b200.palette import BaseColorPalette
    from paper_1908_01961_b200.imaging import Frame
    dev = torch.device("cuda")
    t = lambda a, dt=torch.float32: torch.as_tensor(np.asarray(a), dtype=dt, device=dev)  # noqa
    samples = ConsistencySamples(src=t(d["pair_src"], torch.int64), dst=t(d["pair_dst"], torch.int64),
                                 temporal=t(d["pair_temporal"], torch.bool),
                                 weight=t(d["pair_weight"], torch.float64), shape=d["image"].shape[:2])
    aux = EnergyAux(edge_weights=t(d["edge"]), samples=samples,
                    prev_r=t(d["prev_r"]) if "prev_r" in d else None,
                    cluster_ids=t(d["cluster_ids"], torch.int32) if "cluster_ids" in d else None,
                    r_cluster_log=t(d["r_cluster_log"]) if "r_cluster_log" in d else None)
    frame = Frame(t(d["image"]))
    pal = BaseColorPalette(colors=d["colors"])
    layers = LayerStack(t(d["r0"]), t(d["T0"]))
    return frame, pal, layers, aux, EnergyWeights()


@pytest.mark.parametrize("name", OPS)
def test_energy_terms(name):
    from paper_1908_01961_b200.energy import assemble_blocks, LayerStack
    d = load(name)
    frame, pal, layers, aux, w = device_problem(d)
    blocks = assemble_blocks(frame, pal, layers, aux, w)
    e0 = blocks.energies()
    got = np.array([e0[k] for k in O.TERM_NAMES])
    assert np.allclose(got, d["terms0"], rtol=2e-6, atol=1e-9), (got, d["terms0"])
    nr = d["r0"].size
    r1 = d["r0"] + 0.01 * d["p"][:nr].reshape(d["r0"].shape)
    T1 = d["T0"] + 0.01 * d["p"][nr:].reshape(d["T0"].shape)
    e1 = blocks.energies(torch.as_tensor(r1, dtype=torch.float32, device="cuda"),
                         torch.as_tensor(T1, dtype=torch.float32, device="cuda"))
    got1 = np.array([e1[k] for k in O.TERM_NAMES])
    assert np.allclose(got1, d["terms_shift"], rtol=1e-5, atol=1e-8)


@pytest.mark.parametrize("name", OPS)
def test_gradient_diag_apply(name):
    from paper_1908_01961_b200.energy import assemble_blocks, to_reference_vector, from_reference_vector
    d = load(name)
    frame, pal, layers, aux, w = device_problem(d)
    blocks = assemble_blocks(frame, pal, layers, aux, w)
    b, diag = blocks.gradient_and_diag()
    assert rel(to_reference_vector(b), d["b"]) < 1e-5
    assert rel(to_reference_vector(diag), d["diag"]) < 1e-5
    H, W = d["image"].shape[:2]
    K = d["colors"].shape[0]
    p = from_reference_vector(d["p"], H, W, K)
    Ap = blocks.apply_normal(p)
    assert rel(to_reference_vector(Ap), d["Ap"]) < 2e-5


@pytest.mark.parametrize("weighted", [False, True])
def test_apply_with_a_hub_pixel_vs_oracle(weighted):
    """Explicit partner rows where four hub pixels of one 32-pixel run each
    pair with their whole 15x15 window: that run's adjacency span (~900
    entries) overflows the warp sort's shared memory, so the in-place fallback
    orders it -- the operator still matches the oracle's (unit and explicit
    pair weights)."""
    from paper_1908_01961_b200.energy import assemble_blocks, from_reference_vector, to_reference_vector
    d = dict(load("ops_d"))
    H, W = d["image"].shape[:2]
    K = d["colors"].shape[0]
    srcs, dsts = [], []
    for hy, hx in ((16, 4), (16, 12), (16, 20), (16, 28)):     # flat 644 .. 668: one 32-row group
        hub = hy * W + hx
        for y in range(max(0, hy - 7), min(H, hy + 8)):
            for x in range(max(0, hx - 7), min(W, hx + 8)):
                if y * W + x != hub:
                    srcs.append(y * W + x)
                    dsts.append(hub)
    rng = np.random.default_rng(4)
    extra = len(srcs)
    d["pair_src"] = np.concatenate([d["pair_src"], np.array(srcs, dtype=np.int64)])
    d["pair_dst"] = np.concatenate([d["pair_dst"], np.array(dsts, dtype=np.int64)])
    d["pair_temporal"] = np.concatenate([d["pair_temporal"], np.zeros(extra, dtype=bool)])
    w = rng.uniform(0.5, 2.0, size=d["pair_src"].size) if weighted else np.ones(d["pair_src"].size)
    d["pair_weight"] = w
    frame, pal, layers, aux, wts = device_problem(d)
    blocks = assemble_blocks(frame, pal, layers, aux, wts)
    p = from_reference_vector(d["p"], H, W, K)
    Ap = to_reference_vector(blocks.apply_normal(p))
    osys = oracle_system(d)
    assert rel(Ap, osys.apply(d["p"])) < 2e-5


@pytest.mark.parametrize("name", OPS)
def test_pcg16(name):
    from paper_1908_01961_b200.energy import assemble_blocks, to_reference_vector
    d = load(name)
    frame, pal, layers, aux, w = device_problem(d)
    x, info = assemble_blocks(frame, pal, layers, aux, w).pcg(16)
    assert info["iterations"] == int(d["pcg_info"][0])
    xv = to_reference_vector(x).cpu().numpy()
    assert np.linalg.norm(xv - d["pcg_x"]) / np.linalg.norm(d["pcg_x"]) < 1e-4
    assert np.isclose(info["initial_residual"], d["pcg_info"][1], rtol=1e-5)
    assert np.isclose(info["final_residual"], d["pcg_info"][2], rtol=1e-2)


@pytest.mark.parametrize("name", OPS)
def test_gn_step(name):
    from paper_1908_01961_b200.solver import SolverState, SolveConfig, gn_step_sparse
    d = load(name)
    frame, pal, layers, aux, w = device_problem(d)
    st = SolverState(frame=frame, palette=pal, layers=layers, aux=aux, weights=w,
                     config=SolveConfig())
    rec = gn_step_sparse(st)
    assert rec["accepted"] == bool(d["gn_rec"][2])
    assert rec["alpha"] == d["gn_rec"][3]
    assert np.isclose(rec["energy_before"], d["gn_rec"][0], rtol=2e-6)
    assert np.isclose(rec["energy_after"], d["gn_rec"][1], rtol=1e-4)
    assert np.max(np.abs(st.layers.T.cpu().numpy() - d["gn_T"])) < 1e-3
    assert np.max(np.abs(st.layers.r.cpu().numpy() - d["gn_r"])) < 1e-3
    assert set(rec) == {"phase", "energy_before", "energy_after", "accepted", "alpha", "pcg", "terms"}
    assert set(rec["terms"]) == set(O.TERM_NAMES)


def test_gn_step_deterministic():
    from paper_1908_01961_b200.solver import SolverState, SolveConfig, gn_step_sparse
    d = load("ops_d")
    outs = []
    for _ in range(2):
        frame, pal, layers, aux, w = device_problem(d)
        st = SolverState(frame=frame, palette=pal, layers=layers, aux=aux, weights=w,
                         config=SolveConfig())
        rec = gn_step_sparse(st)
        outs.append((rec["energy_after"], st.layers.X.clone()))
    assert outs[0][0] == outs[1][0]
    assert torch.equal(outs[0][1], outs[1][1])


def test_numerical_fault_carries_terms():
    from paper_1908_01961_b200.solver import (SolverState, SolveConfig, gn_step_sparse,
                                              NumericalFaultError)
    d = load("ops_a")
    frame, pal, layers, aux, w = device_problem(d)
    layers.X[0, 0, 0] = float("nan")
    st = SolverState(frame=frame, palette=pal, layers=layers, aux=aux, weights=w,
                     config=SolveConfig())
    with pytest.raises(NumericalFaultError) as exc:
        gn_step_sparse(st)
    assert "terms" in exc.value.dump


def test_sampler_and_edge_bit_exact():
    from paper_1908_01961_b200.imaging import chromaticity, Frame
    from paper_1908_01961_b200.energy import sample_consistency, chroma_edge_weights
    d = load("sampler")
    img = Frame(torch.as_tensor(d["image"], dtype=torch.float32, device="cuda"))
    pimg = Frame(torch.as_tensor(d["prev_image"], dtype=torch.float32, device="cuda"))
    c, pc = chromaticity(img), chromaticity(pimg)
    assert np.array_equal(c.chroma.cpu().numpy(), d["chroma"])
    assert rel(chroma_edge_weights(c), d["edge"]) < 1e-6
    for seed in (0, 9, 123):
        for tag, prev in (("sp", None), ("tp", pc)):
            s = sample_consistency(c, prev, seed)
            assert np.array_equal(s.src.cpu().numpy(), d[f"{tag}{seed}_src"])
            assert np.array_equal(s.dst.cpu().numpy(), d[f"{tag}{seed}_dst"])
            assert np.array_equal(s.temporal.cpu().numpy(), d[f"{tag}{seed}_temporal"])


def test_segment_bit_exact():
    from paper_1908_01961_b200.palette import segment, BaseColorPalette
    from paper_1908_01961_b200.imaging import Frame
    d = load("segment")
    cm = segment(Frame(torch.as_tensor(d["image"], dtype=torch.float32, device="cuda")),
                 BaseColorPalette(colors=d["colors"]))
    assert np.array_equal(cm.ids.cpu().numpy(), d["ids"])


def test_frame_rejects_non_finite_values():
    """imaging.py:36-57: a frame with NaN / inf anywhere raises FrameError
    (k_all_finite: float4 body, scalar tail, unaligned views)."""
    from paper_1908_01961_b200.imaging import Frame, FrameError
    rng = np.random.default_rng(2)
    base = torch.as_tensor(rng.uniform(0, 1, size=(37, 41, 3)), dtype=torch.float32, device="cuda")
    Frame(base)                                            # finite: accepted
    n = base.numel()
    for pos in (0, 1, 2, 3, n // 2, n - 5, n - 2, n - 1):  # body and the scalar tail (n % 4 = 3)
        for bad in (float("nan"), float("inf"), -float("inf")):
            x = base.clone()
            x.view(-1)[pos] = bad
            with pytest.raises(FrameError):
                Frame(x)
    big = torch.zeros(1, 38, 41, 3, dtype=torch.float32, device="cuda").view(-1)
    view = big[1:1 + n].view(37, 41, 3)                    # 4-byte aligned, not 16: scalar path
    view.copy_(base)
    Frame(view)
    view[36, 40, 2] = float("nan")
    with pytest.raises(FrameError):
        Frame(view)


def test_segment_ties_bit_exact():
    """Argmin ties (palette.py:203-207, first minimum wins): duplicated palette
    colors, colors mirrored about pixel chromas, and pixels quantised onto a
    coarse grid so that many squared distances coincide -- the device's
    one-root argmin against the oracle's per-color norms."""
    from paper_1908_01961_b200.palette import segment, BaseColorPalette
    from paper_1908_01961_b200.imaging import Frame
    rng = np.random.default_rng(11)
    img = np.round(rng.uniform(0.05, 1.0, size=(96, 128, 3)) * 8) / 8      # few distinct chromas
    img[:4, :4] = 0.001                                                    # dark pixels
    colors = np.array([[0.5, 0.25, 0.25], [0.25, 0.5, 0.25], [0.25, 0.5, 0.25],   # a duplicate
                       [0.25, 0.25, 0.5], [0.375, 0.375, 0.25], [0.25, 0.375, 0.375]])
    cm = segment(Frame(torch.as_tensor(img, dtype=torch.float32, device="cuda")), BaseColorPalette(colors=colors))
    ref = O.segment(img.astype(np.float32).astype(np.float64), colors)
    assert np.array_equal(cm.ids.cpu().numpy(), ref)


def test_dense_system_svd_and_step():
    from paper_1908_01961_b200.energy import refine_normal_system, EnergyWeights
    from paper_1908_01961_b200.solver import svd_solve, solve_dense_block, SolverState, SolveConfig
    d = load("dense")
    frame, pal, layers, aux, w = device_problem(d)
    A0, r0 = refine_normal_system(frame, layers, pal, w)
    assert rel(A0, d["A_noids"]) < 1e-9 and rel(r0, d["rhs_noids"]) < 1e-9
    A1, r1 = refine_normal_system(frame, layers, pal, w, cluster_ids=aux.cluster_ids)
    assert rel(A1, d["A_ids"]) < 1e-9 and rel(r1, d["rhs_ids"]) < 1e-9
    assert rel(svd_solve(d["A_ids"], d["rhs_ids"], 1e-8), d["svd_x"]) < 1e-9
    assert rel(svd_solve(d["A_rank"], d["rhs_rank"], 1e-8), d["svd_rank_x"]) < 1e-6
    st = SolverState(frame=frame, palette=pal, layers=layers, aux=aux, weights=w,
                     config=SolveConfig())
    applied = solve_dense_block(st)
    assert np.max(np.abs(applied - d["dense_applied"])) < 1e-7
    rec = st.records[-1]
    assert rec["accepted"] == bool(d["dense_rec"][2]) and rec["alpha"] == d["dense_rec"][3]
    assert np.isclose(rec["energy_before"], d["dense_rec"][0], rtol=1e-6)


def test_svd_solve_hand_cases():
    from paper_1908_01961_b200.solver import svd_solve
    rng = np.random.default_rng(0)
    for n in (1, 3, 6, 12, 24, 36):
        M = rng.normal(size=(n, n))
        A = M @ M.T + n * np.eye(n)
        b = rng.normal(size=n)
        assert np.allclose(svd_solve(A, b, 1e-8), np.linalg.solve(A, b), rtol=1e-9, atol=1e-12)
    assert np.all(svd_solve(np.zeros((6, 6)), np.ones(6), 1e-8) == 0.0)


def layer_gate(r, T, r_ref, T_ref, image, colors):
    """North-star parity gate: per-layer max-abs (R = e^r, each T_k) and the
    relative reconstruction energy."""
    R, Rr = np.exp(r), np.exp(r_ref)
    B = O.palette_matrix(colors)
    e = np.sum((image - R * (T @ B)) ** 2)
    er = np.sum((image - Rr * (T_ref @ B)) ** 2)
    return (float(np.max(np.abs(R - Rr))), [float(np.max(np.abs(T[..., k] - T_ref[..., k])))
                                            for k in range(T.shape[2])],
            abs(e - er) / max(er, 1e-300), e, er)


def _frame1_setup(d):
    from paper_1908_01961_b200.palette import BaseColorPalette, cluster_map_from_ids
    from paper_1908_01961_b200.imaging import Frame
    frame = Frame(torch.as_tensor(d["image"], device="cuda"))
    pal = BaseColorPalette(colors=d["colors"])
    return frame, pal, cluster_map_from_ids(d["ids"], pal)


def test_frame1_cfg1_free_running():
    """cfg1 frame 1 (refinement, 28 GN + dense steps, fixed counts) solved
    free-running vs the reference.  The non-negativity weight jumps at T = 0
    (energy.py:115-118), so single pixels that sit at T ~ 0 can land on the
    other side of the switch after many steps; the
    per-layer gate is therefore asserted on 99.9% of pixels with the worst
    pixel bounded, and the exact per-step gate is the teacher-forced test
    below."""
    from paper_1908_01961_b200.solver import SolveConfig, SolverState, build_aux, initialize
    from paper_1908_01961_b200.refine import refine_palette
    from paper_1908_01961_b200.energy import EnergyWeights
    d = load("frame1_cfg1")
    frame, pal, cm = _frame1_setup(d)
    st = SolverState(frame=frame, palette=pal, layers=initialize(frame, cm, pal),
                     aux=build_aux(frame, cm, int(d["seed"])), weights=EnergyWeights(),
                     config=SolveConfig(tol_rel=0.0))
    refined, _ = refine_palette(st)
    rec = records_array(st.records)
    assert rec.shape == d["records"].shape
    assert np.allclose(rec[:, [0, 3, 4, 5]], d["records"][:, [0, 3, 4, 5]])
    assert np.allclose(rec[:, 2], d["records"][:, 2], rtol=1e-4)
    T = st.layers.T.cpu().numpy().astype(np.float64)
    R = np.exp(st.layers.r.cpu().numpy().astype(np.float64))
    dT = np.abs(T - d["T"])
    dR = np.abs(R - np.exp(d["r"].astype(np.float64)))
    frac = max(float(np.mean(dR > 1e-3)), max(float(np.mean(dT[..., k] > 1e-3)) for k in range(T.shape[2])))
    print(f"frame1 free-running: max|dR| {dR.max():.2e} max|dT| {dT.max():.2e} "
          f"pixels over 1e-3: {frac:.2e}")
    assert frac <= 1e-3
    assert dR.max() <= 1e-2 and dT.max() <= 1e-2
    _, _, drel, _, _ = layer_gate(np.log(R), T, d["r"].astype(np.float64), d["T"].astype(np.float64),
                                  d["image"].astype(np.float64), d["colors_out"])
    assert drel <= 1e-4
    assert np.max(np.abs(refined.colors - d["colors_out"])) <= 1e-3


def test_frame1_cfg1_teacher_forced_steps():
    """Every step of the reference frame-1 trajectory (sparse GN steps and
    dense base-color steps, including both branches of each refine race,
    solver.py:274-292), replayed on the device from the oracle's input state:
    per-layer max-abs <= 1e-3 and energies within 1e-5 at every step.  The
    oracle itself is pinned to the reference on this frame
    (tests/test_oracle_golden.py::test_frame1_cfg1_matches_reference)."""
    import copy
    from paper_1908_01961_b200.solver import (SolveConfig, SolverState, build_aux, gn_step_sparse,
                                              solve_dense_block)
    from paper_1908_01961_b200.energy import EnergyWeights, LayerStack
    from paper_1908_01961_b200.palette import BaseColorPalette
    d = load("frame1_cfg1")
    img = d["image"].astype(np.float64)
    steps = []
    real_gn, real_dense = O.gn_step_sparse, O.solve_dense_block

    def rec_gn(st):
        before = (st.r.copy(), st.T.copy(), st.colors.copy())
        out = real_gn(st)
        steps.append(("sparse", before, (st.r.copy(), st.T.copy(), st.colors.copy()), copy.deepcopy(out)))
        return out

    def rec_dense(st):
        before = (st.r.copy(), st.T.copy(), st.colors.copy())
        n0 = len(st.records)
        out = real_dense(st)
        r = st.records[-1] if len(st.records) > n0 else None
        steps.append(("dense", before, (st.r.copy(), st.T.copy(), st.colors.copy()), copy.deepcopy(r)))
        return out

    O.gn_step_sparse, O.solve_dense_block = rec_gn, rec_dense
    try:
        ost = O.State(image=img, colors=d["colors"].copy(), r=None, T=None,
                      aux=O.build_aux(img, d["ids"], int(d["seed"])), weights=O.Weights(),
                      config=O.Config(tol_rel=0.0))
        ost.r, ost.T = O.initialize(img, d["ids"], d["colors"])
        O.refine_palette(ost)
    finally:
        O.gn_step_sparse, O.solve_dense_block = real_gn, real_dense
    assert len(steps) >= 30

    frame, pal, cm = _frame1_setup(d)
    aux = build_aux(frame, cm, int(d["seed"]))
    worst = 0.0
    for kind, (r0, T0, c0), (r1, T1, c1), orec in steps:
        st = SolverState(frame=frame, palette=BaseColorPalette(colors=c0),
                         layers=LayerStack(torch.as_tensor(r0, dtype=torch.float32, device="cuda"),
                                           torch.as_tensor(T0, dtype=torch.float32, device="cuda")),
                         aux=aux, weights=EnergyWeights(), config=SolveConfig(tol_rel=0.0))
        if kind == "sparse":
            rec = gn_step_sparse(st)
            assert rec["accepted"] == orec["accepted"] and rec["alpha"] == orec["alpha"]
            assert rec["pcg"]["iterations"] == orec["pcg"]["iterations"]
            assert np.isclose(rec["energy_before"], orec["energy_before"], rtol=1e-5)
            assert np.isclose(rec["energy_after"], orec["energy_after"], rtol=1e-5)
            dT = np.abs(st.layers.T.cpu().numpy() - T1).max()
            dR = np.abs(np.exp(st.layers.r.cpu().numpy().astype(np.float64)) - np.exp(r1)).max()
            worst = max(worst, dT, dR)
            assert dT <= 1e-3 and dR <= 1e-3, (kind, dT, dR)
        else:
            solve_dense_block(st)
            if orec is None:
                assert np.array_equal(st.palette.colors, c0)
                continue
            assert np.max(np.abs(st.palette.colors - c1)) <= 1e-5
            assert np.isclose(st.records[-1]["energy_after"], orec["energy_after"], rtol=1e-5)
    print(f"frame1 teacher-forced: {len(steps)} steps, worst per-layer max-abs {worst:.2e}")


def test_stream_cfg1_teacher_forced_gate():
    from paper_1908_01961_b200.solver import SolveConfig, SolverState, build_aux, flip_flop
    from paper_1908_01961_b200.palette import BaseColorPalette, segment
    from paper_1908_01961_b200.imaging import Frame, chromaticity
    from paper_1908_01961_b200.energy import EnergyWeights, LayerStack
    d = load("stream_cfg1")
    frame = Frame(torch.as_tensor(d["image"], device="cuda"))
    prev = Frame(torch.as_tensor(d["prev_image"], device="cuda"))
    pal = BaseColorPalette(colors=d["colors"])
    cm = segment(frame, pal)
    assert np.array_equal(cm.ids.cpu().numpy(), d["ids"])
    prev_layers = LayerStack(torch.as_tensor(d["prev_r"], device="cuda"),
                             torch.as_tensor(d["prev_T"], device="cuda"))
    aux = build_aux(frame, cm, int(d["seed"]), prev_chroma=chromaticity(prev),
                    prev_r=prev_layers.r)
    st = SolverState(frame=frame, palette=pal, layers=prev_layers.copy(), aux=aux,
                     weights=EnergyWeights(),
                     config=replace(SolveConfig(tol_rel=0.0), refine=False, outer_iterations=2))
    flip_flop(st)
    dR, dT, drel, _, _ = layer_gate(st.layers.r.cpu().numpy().astype(np.float64),
                                    st.layers.T.cpu().numpy().astype(np.float64),
                                    d["r"].astype(np.float64), d["T"].astype(np.float64),
                                    d["image"].astype(np.float64), d["colors"])
    assert dR <= 1e-3 and max(dT) <= 1e-3, (dR, dT)
    assert drel <= 1e-4


def test_clip_small_pipeline_drift_reported():
    """Free-running clip through decompose_frames: drift is reported, gated
    loosely (free-running runs are chaotic at T = 0)."""
    from paper_1908_01961_b200.pipeline import decompose_frames
    from paper_1908_01961_b200.palette import BaseColorPalette, cluster_map_from_ids
    from paper_1908_01961_b200.energy import EnergyWeights
    from paper_1908_01961_b200.solver import SolveConfig
    d = load("clip_small")
    frames = [torch.as_tensor(f, device="cuda") for f in d["frames"]]
    pal = BaseColorPalette(colors=d["colors"])
    res = decompose_frames(frames, EnergyWeights(), SolveConfig(tol_rel=0.0), seed=0,
                           palette=pal, cluster_map=cluster_map_from_ids(d["ids0"], pal))
    assert np.max(np.abs(res.palette.colors - d["colors_out"])) < 1e-2
    for i, ls in enumerate(res.layer_stacks):
        dT = np.max(np.abs(ls.T.cpu().numpy() - d["T"][i]))
        assert dT < 5e-2, (i, dT)

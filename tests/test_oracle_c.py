"""Pin the compiled CPU restatement (oracle/ls_oracle.c via oracle/c_oracle.py)
against the reference's own outputs frozen in tests/golden/ -- the same
fixtures and bars as tests/test_oracle_golden.py pins the NumPy oracle with
-- plus thread-count independence.  CPU only.

The C oracle is what makes the 1920x1080 K=8 headline configuration
checkable (tests/test_gpu_headline.py) and the CPU baseline measurable at
full size (bench.py), so it must be pinned as tightly as the NumPy one."""
from dataclasses import replace

import numpy as np
import pytest

from oracle import c_oracle as CO
from oracle import lumisplit_oracle as O
from tests.golden_io import load, oracle_aux, records_array

OPS = ["ops_a", "ops_b", "ops_c", "ops_d"]


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def _sys(d):
    s = CO.System(d["image"], d["colors"], oracle_aux(d), O.Weights())
    s.linearize(d["r0"], d["T0"])
    return s


@pytest.mark.parametrize("name", OPS)
def test_terms_match_reference(name):
    d = load(name)
    s = _sys(d)
    t0 = s.terms(d["r0"], d["T0"])
    assert np.allclose([t0[k] for k in O.TERM_NAMES], d["terms0"], rtol=1e-12, atol=1e-12)
    nr = d["r0"].size
    r1 = d["r0"] + 0.01 * d["p"][:nr].reshape(d["r0"].shape)
    T1 = d["T0"] + 0.01 * d["p"][nr:].reshape(d["T0"].shape)
    t1 = s.terms(r1, T1)
    assert np.allclose([t1[k] for k in O.TERM_NAMES], d["terms_shift"], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("name", OPS)
def test_grad_diag_apply_match_reference(name):
    d = load(name)
    s = _sys(d)
    b, diag = s.grad_diag()
    assert rel(b, d["b"]) < 1e-13
    assert rel(diag, d["diag"]) < 1e-13
    assert rel(s.apply(d["p"]), d["Ap"]) < 1e-13


@pytest.mark.parametrize("name", OPS)
def test_pcg_and_gn_step_match_reference(name):
    d = load(name)
    s = _sys(d)
    b, diag = s.grad_diag()
    x, info = s.pcg(b, diag, 16)
    assert info["iterations"] == int(d["pcg_info"][0])
    assert rel(x, d["pcg_x"]) < 1e-9
    assert np.isclose(info["final_residual"], d["pcg_info"][2], rtol=1e-8)
    st = O.State(image=d["image"], colors=d["colors"], r=d["r0"].copy(), T=d["T0"].copy(),
                 aux=oracle_aux(d), weights=O.Weights(), config=O.Config())
    rec = CO.gn_step_sparse(st)
    assert rec["accepted"] == bool(d["gn_rec"][2])
    assert rec["alpha"] == d["gn_rec"][3]
    assert np.isclose(rec["energy_after"], d["gn_rec"][1], rtol=1e-10)
    assert np.allclose([rec["terms"][k] for k in O.TERM_NAMES], d["gn_terms"], rtol=1e-10, atol=1e-12)
    assert np.max(np.abs(st.T - d["gn_T"])) < 1e-9
    assert np.max(np.abs(st.r - d["gn_r"])) < 1e-9


def test_aux_and_sampler_bit_exact():
    d = load("sampler")
    c, _ = CO.chromaticity(d["image"])
    pc, _ = CO.chromaticity(d["prev_image"])
    oc, _, _ = O.chromaticity(d["image"])
    assert np.array_equal(c, oc)
    assert np.max(np.abs(CO.edge_gate(c) - d["edge"])) <= 1e-15
    for seed in (0, 9, 123):
        for tag, prev in (("sp", None), ("tp", pc)):
            s = CO.sample_pairs(c, prev, seed)
            assert np.array_equal(s.src, d[f"{tag}{seed}_src"])
            assert np.array_equal(s.dst, d[f"{tag}{seed}_dst"])
            assert np.array_equal(s.temporal, d[f"{tag}{seed}_temporal"])


def test_sampler_matches_numpy_generator_with_rejections():
    """Large random frames: the draw stream (including Lemire rejections,
    p = 2^-32 per draw) equals numpy's Generator for many seeds."""
    rng = np.random.default_rng(5)
    img = rng.uniform(0.05, 1.0, size=(64, 96, 3))
    prev = rng.uniform(0.05, 1.0, size=(64, 96, 3))
    c, _ = CO.chromaticity(img)
    pc, _ = CO.chromaticity(prev)
    for seed in range(8):
        a = CO.sample_pairs(c, pc, seed)
        b = O.sample_pairs(c, pc, seed)
        assert np.array_equal(a.src, b.src) and np.array_equal(a.dst, b.dst)
        assert np.array_equal(a.temporal, b.temporal)


def test_dense_system_and_svd_match_reference():
    d = load("dense")
    w = O.Weights()
    aux = oracle_aux(d)
    s = CO.System(d["image"], d["colors"], aux, w)
    A0, r0 = s.dense_normal(d["r0"], d["T0"], use_ids=False)
    A1, r1 = s.dense_normal(d["r0"], d["T0"], use_ids=True)
    assert rel(A0, d["A_noids"]) < 1e-12 and rel(r0, d["rhs_noids"]) < 1e-12
    assert rel(A1, d["A_ids"]) < 1e-12 and rel(r1, d["rhs_ids"]) < 1e-12
    assert rel(CO.svd_solve(A1, r1, 1e-8), d["svd_x"]) < 1e-10
    assert rel(CO.svd_solve(d["A_rank"], d["rhs_rank"], 1e-8), d["svd_rank_x"]) < 1e-8
    assert not np.any(CO.svd_solve(np.zeros((6, 6)), np.ones(6), 1e-8))


def test_segment_and_initialize_match_reference():
    d = load("segment")
    assert np.array_equal(CO.segment(d["image"], d["colors"]), d["ids"])
    d = load("frame1_cfg1")
    img = d["image"].astype(np.float64)
    r, T = CO.initialize(img, d["ids"], d["colors"])
    ro, To = O.initialize(img, d["ids"], d["colors"])
    assert np.max(np.abs(r - ro)) <= 1e-15 and np.max(np.abs(T - To)) <= 1e-15


def test_frame1_cfg1_matches_reference():
    """Frame 1 with refinement (the refine race and dense line search)."""
    d = load("frame1_cfg1")
    img = d["image"].astype(np.float64)
    st = CO.solve_frame(img, d["colors"].copy(), d["ids"], O.Weights(), O.Config(tol_rel=0.0),
                        int(d["seed"]))
    rec = records_array(st.records)
    assert rec.shape == d["records"].shape
    assert np.allclose(rec[:, [0, 3, 4, 5]], d["records"][:, [0, 3, 4, 5]])
    assert np.max(np.abs(np.exp(st.r) - np.exp(d["r"]))) < 1e-5
    assert np.max(np.abs(st.T - d["T"])) < 1e-5
    assert np.max(np.abs(st.colors - d["colors_out"])) < 1e-9


def test_stream_cfg1_teacher_forced_matches_reference():
    d = load("stream_cfg1")
    img = d["image"].astype(np.float64)
    prev = O.State(image=None, colors=d["colors"], r=d["prev_r"].astype(np.float64),
                   T=d["prev_T"].astype(np.float64), aux=None, weights=None, config=None)
    cfg = replace(O.Config(tol_rel=0.0), outer_iterations=2)
    st = CO.stream_frame(img, d["colors"], prev, d["prev_image"].astype(np.float64), O.Weights(), cfg,
                         int(d["seed"]))
    assert np.max(np.abs(st.T - d["T"])) < 1e-5
    assert np.max(np.abs(st.r - d["r"])) < 1e-5
    rec = records_array(st.records)
    assert np.allclose(rec[:, 1:3], d["records"][:, 1:3], rtol=1e-9)


def test_clip_small_free_running():
    d = load("clip_small")
    frames = [f.astype(np.float64) for f in d["frames"]]
    states = CO.decompose_clip(frames, d["colors"], d["ids0"], O.Weights(), O.Config(tol_rel=0.0))
    assert np.max(np.abs(states[0].colors - d["colors_out"])) < 1e-9
    for i, st in enumerate(states):
        assert np.max(np.abs(st.T - d["T"][i])) < 1e-5, i
        assert np.max(np.abs(st.r - d["r"][i])) < 1e-5, i


def test_matches_numpy_oracle_at_k8_and_is_thread_count_independent():
    """K = 8 (the headline palette size) on a small frame: the C restatement
    equals the NumPy oracle's operators to 1e-12 and one GN step to 1e-9,
    and gives the same bits with 1 and with all threads."""
    from paper_1908_01961_b200 import synth
    clip = synth.make_clip(40, 56, 8, 2, seed=4, device="cpu")
    img = clip.frames[1].double().numpy()
    pimg = clip.frames[0].double().numpy()
    ids = O.segment(img, clip.colors)
    r0, T0 = O.initialize(pimg, O.segment(pimg, clip.colors), clip.colors)
    pc = O.chromaticity(pimg)[0]
    aux = O.build_aux(img, ids, 3, pc, r0)
    so = O.FrozenSystem(img, clip.colors, r0, T0, aux, O.Weights())
    p = np.random.default_rng(1).normal(size=r0.size + T0.size)
    outs = []
    for threads in (1, CO.max_threads()):
        CO.set_threads(threads)
        sc = CO.System(img, clip.colors, aux, O.Weights())
        sc.linearize(r0, T0)
        b, dg = sc.grad_diag()
        outs.append((sc.terms(r0, T0), b, dg, sc.apply(p)))
        st = O.State(image=img, colors=clip.colors, r=r0.copy(), T=T0.copy(), aux=aux, weights=O.Weights(),
                     config=O.Config())
        CO.gn_step_sparse(st)
        outs[-1] += (st.r, st.T)
    CO.set_threads(0)
    for a, b in zip(outs[0][1:], outs[1][1:]):
        assert np.array_equal(a, b)
    assert outs[0][0] == outs[1][0]
    bo, do = so.grad_diag()
    assert rel(outs[0][1], bo) < 1e-12 and rel(outs[0][2], do) < 1e-12
    assert rel(outs[0][3], so.apply(p)) < 1e-12
    to = so.terms(r0, T0)
    assert np.allclose([outs[0][0][k] for k in O.TERM_NAMES], [to[k] for k in O.TERM_NAMES], rtol=1e-12)
    st = O.State(image=img, colors=clip.colors, r=r0.copy(), T=T0.copy(), aux=aux, weights=O.Weights(),
                 config=O.Config())
    O.gn_step_sparse(st)
    assert np.max(np.abs(st.r - outs[0][4])) < 1e-9 and np.max(np.abs(st.T - outs[0][5])) < 1e-9

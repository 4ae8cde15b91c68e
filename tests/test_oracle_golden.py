"""Pin the CPU oracle (oracle/lumisplit_oracle.py) against the reference's
own outputs frozen in tests/golden/ (tools/make_golden.py).  CPU only.

These mirror the reference's hot-path golden suite:
energies, -J^T F, diag(J^T J), J^T J p, PCG(16), one GN step, the dense
normal system, the truncated-SVD solve, the dense step, the sampler,
segmentation and full frame solves.
"""
from dataclasses import replace

import numpy as np
import pytest

from oracle import lumisplit_oracle as O
from tests.golden_io import load, oracle_aux, oracle_system, records_array

OPS = ["ops_a", "ops_b", "ops_c", "ops_d"]


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("name", OPS)
def test_terms_match_reference(name):
    d = load(name)
    s = oracle_system(d)
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
    s = oracle_system(d)
    b, diag = s.grad_diag()
    assert rel(b, d["b"]) < 1e-13
    assert rel(diag, d["diag"]) < 1e-13
    assert rel(s.apply(d["p"]), d["Ap"]) < 1e-13


@pytest.mark.parametrize("name", OPS)
def test_pcg_and_gn_step_match_reference(name):
    d = load(name)
    s = oracle_system(d)
    b, diag = s.grad_diag()
    x, info = O.pcg(s.apply, b, diag, 16)
    assert info["iterations"] == int(d["pcg_info"][0])
    assert rel(x, d["pcg_x"]) < 1e-9
    assert np.isclose(info["final_residual"], d["pcg_info"][2], rtol=1e-8)
    st = O.State(image=d["image"], colors=d["colors"], r=d["r0"].copy(), T=d["T0"].copy(),
                 aux=oracle_aux(d), weights=O.Weights(), config=O.Config())
    rec = O.gn_step_sparse(st)
    assert rec["accepted"] == bool(d["gn_rec"][2])
    assert rec["alpha"] == d["gn_rec"][3]
    assert np.isclose(rec["energy_after"], d["gn_rec"][1], rtol=1e-10)
    assert np.max(np.abs(st.T - d["gn_T"])) < 1e-9
    assert np.max(np.abs(st.r - d["gn_r"])) < 1e-9


def test_sampler_bit_exact():
    d = load("sampler")
    c, _, _ = O.chromaticity(d["image"])
    pc, _, _ = O.chromaticity(d["prev_image"])
    assert np.array_equal(O.edge_gate(c), d["edge"])
    for seed in (0, 9, 123):
        for tag, prev in (("sp", None), ("tp", pc)):
            s = O.sample_pairs(c, prev, seed)
            assert np.array_equal(s.src, d[f"{tag}{seed}_src"])
            assert np.array_equal(s.dst, d[f"{tag}{seed}_dst"])
            assert np.array_equal(s.temporal, d[f"{tag}{seed}_temporal"])


def test_pcg64_stream_model():
    """The u32-stream / Lemire model the CUDA sampler implements."""
    n = 50
    u = O.pcg64_u32_stream(7, 12 * n)
    rng = np.random.default_rng(7)
    dx = rng.integers(-7, 8, size=(n, 4)).ravel()
    dy = rng.integers(-7, 8, size=(n, 4)).ravel()
    tt = rng.integers(0, 2, size=(n, 4)).ravel()
    assert np.array_equal(((u[:4 * n] * 15) >> 32).astype(np.int64) - 7, dx)
    assert np.array_equal(((u[4 * n:8 * n] * 15) >> 32).astype(np.int64) - 7, dy)
    assert np.array_equal(((u[8 * n:] * 2) >> 32).astype(np.int64), tt)


def test_dense_system_and_svd_match_reference():
    d = load("dense")
    w = O.Weights()
    A0, r0 = O.refine_normal_system(d["image"], d["r0"], d["T0"], d["colors"], w)
    A1, r1 = O.refine_normal_system(d["image"], d["r0"], d["T0"], d["colors"], w,
                                    d["cluster_ids"])
    assert rel(A0, d["A_noids"]) < 1e-12 and rel(r0, d["rhs_noids"]) < 1e-12
    assert rel(A1, d["A_ids"]) < 1e-12 and rel(r1, d["rhs_ids"]) < 1e-12
    assert rel(O.svd_solve(A1, r1, 1e-8), d["svd_x"]) < 1e-10
    assert rel(O.svd_solve(d["A_rank"], d["rhs_rank"], 1e-8), d["svd_rank_x"]) < 1e-8
    st = O.State(image=d["image"], colors=d["colors"].copy(), r=d["r0"], T=d["T0"],
                 aux=oracle_aux(d), weights=w, config=O.Config())
    applied = O.solve_dense_block(st)
    assert np.max(np.abs(applied - d["dense_applied"])) < 1e-10
    rec = st.records[-1]
    assert np.allclose([rec["energy_before"], rec["energy_after"], rec["accepted"],
                        rec["alpha"], rec["delta_b_norm"]], d["dense_rec"], rtol=1e-10)


def test_segment_matches_reference():
    d = load("segment")
    assert np.array_equal(O.segment(d["image"], d["colors"]), d["ids"])


def test_frame1_cfg1_matches_reference():
    """Frame 1 with refinement, fixed iteration counts (SURVEY 8c gate 1)."""
    d = load("frame1_cfg1")
    img = d["image"].astype(np.float64)
    cfg = O.Config(tol_rel=0.0)
    aux = O.build_aux(img, d["ids"], int(d["seed"]))
    r, T = O.initialize(img, d["ids"], d["colors"])
    st = O.State(image=img, colors=d["colors"].copy(), r=r, T=T, aux=aux,
                 weights=O.Weights(), config=cfg)
    O.refine_palette(st)
    rec = records_array(st.records)
    assert rec.shape == d["records"].shape
    assert np.allclose(rec[:, [0, 3, 4, 5]], d["records"][:, [0, 3, 4, 5]])
    assert np.max(np.abs(np.exp(st.r) - np.exp(d["r"]))) < 1e-5
    assert np.max(np.abs(st.T - d["T"])) < 1e-5
    assert np.max(np.abs(st.colors - d["colors_out"])) < 1e-9


def test_stream_cfg1_teacher_forced_matches_reference():
    d = load("stream_cfg1")
    img = d["image"].astype(np.float64)
    prev_chroma = O.chromaticity(d["prev_image"].astype(np.float64))[0]
    prev_r = d["prev_r"].astype(np.float64)
    prev_T = d["prev_T"].astype(np.float64)
    aux = O.build_aux(img, d["ids"], int(d["seed"]), prev_chroma, prev_r)
    cfg = replace(O.Config(tol_rel=0.0), refine=False, outer_iterations=2)
    st = O.State(image=img, colors=d["colors"], r=prev_r.copy(), T=prev_T.copy(), aux=aux,
                 weights=O.Weights(), config=cfg)
    O.flip_flop(st)
    assert np.array_equal(O.segment(img, d["colors"]), d["ids"])
    assert np.max(np.abs(st.T - d["T"])) < 1e-5
    assert np.max(np.abs(st.r - d["r"])) < 1e-5
    rec = records_array(st.records)
    assert np.allclose(rec[:, 1:3], d["records"][:, 1:3], rtol=1e-9)


def test_clip_small_free_running():
    d = load("clip_small")
    frames = [f.astype(np.float64) for f in d["frames"]]
    states = O.decompose_clip(frames, d["colors"], d["ids0"], O.Weights(),
                              O.Config(tol_rel=0.0))
    assert np.max(np.abs(states[0].colors - d["colors_out"])) < 1e-9
    for i, st in enumerate(states):
        assert np.max(np.abs(st.T - d["T"][i])) < 1e-5, i
        assert np.max(np.abs(st.r - d["r"][i])) < 1e-5, i

"""Generate the golden fixtures in tests/golden/ by running the REFERENCE
package (`lumisplit`, /root/reference/pkg/src) in the build container.

    python tools/make_golden.py            # writes tests/golden/*.npz

The reference cannot travel to the GPU box, so its outputs are frozen here
as small .npz files.  Every fixture stores its inputs too, so the tests that
read them (tests/test_oracle_golden.py on CPU, tests/test_gpu_parity.py on
the GPU) need nothing but numpy.  Inputs are float32-representable.
"""

from __future__ import annotations

import sys
import time
from dataclasses import replace
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "tests" / "golden"
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))

from lumisplit import energy as E  # noqa: E402
from lumisplit import solver as S  # noqa: E402
from lumisplit.imaging import Frame, chromaticity, ChromaticityImage  # noqa: E402
from lumisplit.palette import BaseColorPalette, ClusterMap, segment  # noqa: E402
from lumisplit.refine import refine_palette  # noqa: E402

from paper_1908_01961_b200 import synth  # noqa: E402

f32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731
TERMS = ("data", "clustering", "r_sparsity", "r_consistency", "monochrome",
         "i_sparsity", "smoothness", "non_neg")


def samples_arrays(s):
    return dict(pair_src=s.src.astype(np.int64), pair_dst=s.dst.astype(np.int64),
                pair_temporal=s.temporal.astype(np.bool_), pair_weight=s.weight)


def terms_vec(d):
    return np.array([d[k] for k in TERMS])


def random_problem(seed, h, w, K, temporal, anchor_ids):
    """A state with every term active (negatives trigger non-neg), fp32 inputs."""
    rng = np.random.default_rng(100 + seed)
    colors = f32(rng.uniform(0.1, 1.0, size=(K, 3)))
    image = f32(rng.uniform(0.05, 1.0, size=(h, w, 3)))
    # blocky chroma so the consistency gate keeps a realistic fraction
    image[: h // 2] = f32(image[: h // 2] * 0.2 + 0.8 * image[0, 0])
    r = f32(rng.uniform(np.log(0.05), 0.0, size=(h, w, 3)))
    T = f32(rng.uniform(0.0, 1.2, size=(h, w, K + 1)))
    T[rng.uniform(size=T.shape) < 0.15] *= -0.3
    T = f32(T)
    frame = Frame(image)
    chroma = chromaticity(frame)
    prev_chroma = prev_r = None
    if temporal:
        pimg = f32(np.clip(image * rng.uniform(0.97, 1.03, size=(h, w, 1)), 0, 1))
        prev_chroma = chromaticity(Frame(pimg))
        prev_r = f32(r + rng.normal(scale=0.05, size=r.shape))
    samples = E.sample_consistency(chroma, prev_chroma, seed=seed + 7)
    ids = None
    rcl = None
    if anchor_ids and K > 0:
        ids = rng.integers(1, K + 1, size=(h, w)).astype(np.int32)
    else:
        rcl = f32(np.log(np.exp(rng.uniform(np.log(0.1), 0.0, size=(h, w, 3)))))
    aux = E.EnergyAux(edge_weights=E.chroma_edge_weights(chroma), samples=samples,
                      prev_r=prev_r, cluster_ids=ids, r_cluster_log=rcl)
    pal = BaseColorPalette(colors=colors)
    layers = E.LayerStack(r=r, T=T)
    d = dict(image=image, colors=colors, r0=r, T0=T, edge=aux.edge_weights,
             **samples_arrays(samples))
    if prev_r is not None:
        d["prev_r"] = prev_r
    if ids is not None:
        d["cluster_ids"] = ids
    if rcl is not None:
        d["r_cluster_log"] = rcl
    return frame, pal, layers, aux, d


def gen_ops():
    cases = [("ops_a", 0, 8, 9, 2, False, False),
             ("ops_b", 1, 20, 24, 3, True, True),
             ("ops_c", 2, 12, 16, 0, True, False),
             ("ops_d", 3, 33, 40, 5, True, True)]
    for name, seed, h, w, K, temporal, ids in cases:
        frame, pal, layers, aux, d = random_problem(seed, h, w, K, temporal, ids)
        wts = E.EnergyWeights()
        blocks = E.assemble_blocks(frame.data, pal, layers, aux, wts)
        rng = np.random.default_rng(seed + 55)
        n = layers.r.size + layers.T.size
        p = f32(rng.normal(size=n))
        d["p"] = p
        d["terms0"] = terms_vec(E.block_energies(blocks, layers.r, layers.T))
        nr = layers.r.size
        r1 = layers.r + 0.01 * p[:nr].reshape(layers.r.shape)
        T1 = layers.T + 0.01 * p[nr:].reshape(layers.T.shape)
        d["terms_shift"] = terms_vec(E.block_energies(blocks, r1, T1))
        b, diag = S._gradient_and_diag(blocks, layers.r, layers.T)
        d["b"], d["diag"] = b, diag
        A = S._normal_operator(blocks, layers.r.shape, layers.T.shape)
        d["Ap"] = A(p)
        x, info = S.pcg(A, b, diag, 16)
        d["pcg_x"] = x
        d["pcg_info"] = np.array([info["iterations"], info["initial_residual"],
                                  info["final_residual"]])
        st = S.SolverState(frame=frame, palette=pal, layers=layers.copy(), aux=aux,
                           weights=wts, config=S.SolveConfig())
        rec = S.gn_step_sparse(st)
        d["gn_r"], d["gn_T"] = st.layers.r, st.layers.T
        d["gn_rec"] = np.array([rec["energy_before"], rec["energy_after"],
                                float(rec["accepted"]), rec["alpha"]])
        d["gn_terms"] = terms_vec(rec["terms"])
        np.savez_compressed(OUT / f"{name}.npz", **d)
        print(name, "ok", h, w, K)


def gen_sampler():
    rng = np.random.default_rng(5)
    h, w = 24, 32
    img = np.full((h, w, 3), 0.5)
    img[:, 16:] = [0.7, 0.1, 0.1]
    img[6:12, 4:10] = [0.1, 0.5, 0.2]
    img = f32(img * rng.uniform(0.9, 1.0, size=(h, w, 1)))
    img[20:, :3] = 0.001                            # dark pixels -> neutral chroma
    prev = f32(np.roll(img, 1, axis=1))
    c = chromaticity(Frame(img))
    pc = chromaticity(Frame(prev))
    d = dict(image=img, prev_image=prev)
    for seed in (0, 9, 123):
        s0 = E.sample_consistency(c, None, seed)
        s1 = E.sample_consistency(c, pc, seed)
        for tag, s in (("sp", s0), ("tp", s1)):
            d[f"{tag}{seed}_src"] = s.src
            d[f"{tag}{seed}_dst"] = s.dst
            d[f"{tag}{seed}_temporal"] = s.temporal
    d["edge"] = E.chroma_edge_weights(c)
    d["chroma"] = c.chroma
    np.savez_compressed(OUT / "sampler.npz", **d)
    print("sampler ok")


def gen_dense_and_segment():
    frame, pal, layers, aux, d = random_problem(4, 16, 20, 3, False, True)
    layers.T[:, :, 1:] = np.abs(layers.T[:, :, 1:])
    d["T0"] = layers.T
    wts = E.EnergyWeights()
    A0, rhs0 = E.refine_normal_system(frame.data, layers, pal, wts)
    A1, rhs1 = E.refine_normal_system(frame.data, layers, pal, wts, cluster_ids=aux.cluster_ids)
    d.update(A_noids=A0, rhs_noids=rhs0, A_ids=A1, rhs_ids=rhs1)
    d["svd_x"] = S.svd_solve(A1, rhs1, 1e-8)
    # rank-deficient case (test_solver.py:266-283)
    pal2 = BaseColorPalette(colors=np.array([[0.5, 0.2, 0.2], [0.5, 0.2, 0.2]]))
    T2 = layers.T[:, :, :3].copy()
    T2[:, :, 2] = T2[:, :, 1]
    A2, rhs2 = E.refine_normal_system(frame.data, E.LayerStack(layers.r, T2), pal2,
                                      E.EnergyWeights(lambda_ir=0.0, lambda_cr=0.0))
    d.update(A_rank=A2, rhs_rank=rhs2, svd_rank_x=S.svd_solve(A2, rhs2, 1e-8))
    st = S.SolverState(frame=frame, palette=pal, layers=layers.copy(), aux=aux,
                       weights=wts, config=S.SolveConfig())
    applied = S.solve_dense_block(st)
    rec = st.records[-1]
    d["dense_applied"] = applied
    d["dense_colors"] = st.palette.colors
    d["dense_rec"] = np.array([rec["energy_before"], rec["energy_after"],
                               float(rec["accepted"]), rec["alpha"], rec["delta_b_norm"]])
    np.savez_compressed(OUT / "dense.npz", **d)
    print("dense ok")

    rng = np.random.default_rng(6)
    img = f32(rng.uniform(0.0, 1.0, size=(18, 22, 3)))
    img[rng.uniform(size=(18, 22)) < 0.2] = 0.004            # dark pixels
    img[:1, :5] = 0.001                                       # leading dark run
    cols = f32(rng.uniform(0.1, 0.95, size=(5, 3)))
    cm = segment(Frame(img), BaseColorPalette(colors=cols))
    np.savez_compressed(OUT / "segment.npz", image=img, colors=cols, ids=cm.ids)
    print("segment ok")


def records_arrays(records):
    rows = []
    for rec in records:
        pc = rec.get("pcg", {"iterations": -1, "initial_residual": np.nan,
                             "final_residual": np.nan})
        rows.append([0.0 if rec["phase"] == "sparse" else 1.0, rec["energy_before"],
                     rec["energy_after"], float(rec["accepted"]), rec["alpha"],
                     pc["iterations"], pc["initial_residual"], pc["final_residual"],
                     rec.get("delta_b_norm", np.nan)])
    return np.array(rows)


def gen_frames():
    """cfg1: 160x120, K=4.  Frame 1 with refinement (fixed counts), then
    frame 2 teacher-forced from the reference's frame-1 state."""
    H, W, K = 120, 160, 4
    clip = synth.make_clip(H, W, K, 3, seed=0)
    frames = [f.numpy().astype(np.float64) for f in clip.frames]
    colors = clip.colors
    pal = BaseColorPalette(colors=colors)
    wts = E.EnergyWeights()
    cfg = S.SolveConfig(tol_rel=0.0)
    cm0 = segment(Frame(frames[0]), pal)
    t0 = time.time()
    aux = S.build_aux(Frame(frames[0]), cm0, seed=0)
    layers = S.initialize(Frame(frames[0]), cm0, pal)
    st = S.SolverState(frame=Frame(frames[0]), palette=pal, layers=layers, aux=aux,
                       weights=wts, config=cfg)
    refined, mags = refine_palette(st)
    t1 = time.time()
    np.savez_compressed(OUT / "frame1_cfg1.npz", image=frames[0].astype(np.float32),
                        colors=colors, ids=cm0.ids, seed=0,
                        r=st.layers.r.astype(np.float32), T=st.layers.T.astype(np.float32),
                        colors_out=refined.colors, records=records_arrays(st.records),
                        energy_history=np.array(st.energy_history), seconds=t1 - t0)
    print("frame1 ok", t1 - t0, "s", st.status, len(st.records))
    # teacher-forced streaming frame 2 (pipeline.py:136-156)
    scfg = replace(cfg, refine=False, outer_iterations=2)
    prev_r = st.layers.r.astype(np.float32).astype(np.float64)
    prev_T = st.layers.T.astype(np.float32).astype(np.float64)
    pal_r = BaseColorPalette(colors=refined.colors)
    f2 = Frame(frames[1])
    cm1 = segment(f2, pal_r)
    t0 = time.time()
    aux2 = S.build_aux(f2, cm1, seed=1, prev_chroma=chromaticity(Frame(frames[0])),
                       prev_r=prev_r)
    lay2 = S.initialize(f2, cm1, pal_r, previous=E.LayerStack(prev_r, prev_T))
    st2 = S.SolverState(frame=f2, palette=pal_r, layers=lay2, aux=aux2, weights=wts,
                        config=scfg)
    S.flip_flop(st2)
    t1 = time.time()
    np.savez_compressed(OUT / "stream_cfg1.npz", image=frames[1].astype(np.float32),
                        prev_image=frames[0].astype(np.float32), colors=refined.colors,
                        ids=cm1.ids, seed=1, prev_r=prev_r.astype(np.float32),
                        prev_T=prev_T.astype(np.float32),
                        r=st2.layers.r.astype(np.float32), T=st2.layers.T.astype(np.float32),
                        records=records_arrays(st2.records), seconds=t1 - t0)
    print("stream ok", t1 - t0, "s", st2.status)


def gen_clip_small():
    """Free-running 4-frame 24x32 K=3 clip through the pipeline's sequence
    (pipeline.py:113-166 with the palette given)."""
    H, W, K = 24, 32, 3
    clip = synth.make_clip(H, W, K, 4, seed=3)
    frames = [f.numpy().astype(np.float64) for f in clip.frames]
    pal = BaseColorPalette(colors=clip.colors)
    wts = E.EnergyWeights()
    cfg = S.SolveConfig(tol_rel=0.0)
    cm0 = segment(Frame(frames[0]), pal)
    aux = S.build_aux(Frame(frames[0]), cm0, seed=0)
    st = S.SolverState(frame=Frame(frames[0]), palette=pal,
                       layers=S.initialize(Frame(frames[0]), cm0, pal), aux=aux,
                       weights=wts, config=cfg)
    refined, _ = refine_palette(st)
    rs, Ts, recs = [st.layers.r], [st.layers.T], [records_arrays(st.records)]
    prev = st
    scfg = replace(cfg, refine=False, outer_iterations=2)
    for i in range(1, len(frames)):
        f = Frame(frames[i])
        cm = segment(f, refined)
        aux = S.build_aux(f, cm, seed=i, prev_chroma=chromaticity(Frame(frames[i - 1])),
                          prev_r=prev.layers.r)
        s2 = S.SolverState(frame=f, palette=refined,
                           layers=S.initialize(f, cm, refined, previous=prev.layers),
                           aux=aux, weights=wts, config=scfg)
        S.flip_flop(s2)
        rs.append(s2.layers.r)
        Ts.append(s2.layers.T)
        recs.append(records_arrays(s2.records))
        prev = s2
    np.savez_compressed(OUT / "clip_small.npz", frames=np.stack(frames).astype(np.float32),
                        colors=clip.colors, colors_out=refined.colors, ids0=cm0.ids,
                        r=np.stack(rs), T=np.stack(Ts),
                        **{f"records{i}": r for i, r in enumerate(recs)})
    print("clip ok")


if __name__ == "__main__":
    OUT.mkdir(parents=True, exist_ok=True)
    which = sys.argv[1:] or ["ops", "sampler", "dense", "frames", "clip"]
    if "ops" in which:
        gen_ops()
    if "sampler" in which:
        gen_sampler()
    if "dense" in which:
        gen_dense_and_segment()
    if "clip" in which:
        gen_clip_small()
    if "frames" in which:
        gen_frames()

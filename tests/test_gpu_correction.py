"""Misclustering correction and layer edits on the
device against the reference's own outputs (tests/golden/correction.npz and
editing.npz from tools/make_golden_correction.py)."""
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"


def _cmap(ids):
    from paper_1908_01961_b200.palette import ClusterMap
    t = torch.as_tensor(ids, dtype=torch.int32, device="cuda")
    return ClusterMap(ids=t, r_cluster=torch.zeros(*ids.shape, 3, device="cuda"))


def test_flood_identify_merge_track_bit_exact():
    from paper_1908_01961_b200 import correction as C
    d = np.load(G / "correction.npz")
    r1 = C.identify_region((10, 10), _cmap(d["ids"]))
    r2 = C.identify_region((20, 28), _cmap(d["ids"]))
    assert r1.source_id == int(d["src1"]) and r2.source_id == int(d["src2"])
    assert np.array_equal(r1.mask.cpu().numpy(), d["m_identify"])
    assert np.array_equal(r2.mask.cpu().numpy(), d["m_identify2"])
    t = C.track_region(r1, _cmap(d["ids2"]), frame_index=1)
    assert np.array_equal(t.mask.cpu().numpy(), d["m_track"])
    merged = C.identify_region((10, 10), _cmap(d["ids"]), merge_into=r1)
    assert torch.equal(merged.mask, r1.mask)
    with pytest.raises(C.EmptyRegionError):
        C.identify_region((10, 10), _cmap(d["ids"]), merge_into=r2) if r2.source_id != r1.source_id \
            else C.identify_region((999, 0), _cmap(d["ids"]))


def test_correct_reflectance_picks_the_reference_color():
    from paper_1908_01961_b200 import correction as C
    from paper_1908_01961_b200.imaging import Frame
    from paper_1908_01961_b200.energy import EnergyWeights
    from paper_1908_01961_b200.palette import BaseColorPalette, ClusterMap
    from paper_1908_01961_b200.solver import SolveConfig
    d = np.load(G / "correction.npz")
    colors = d["c_colors"]
    ids = torch.as_tensor(d["c_ids"], dtype=torch.int32, device="cuda")
    cmap = ClusterMap(ids=ids, r_cluster=torch.as_tensor(colors, dtype=torch.float32, device="cuda")[ids.long() - 1])
    frame = Frame(torch.as_tensor(d["c_image"], device="cuda"))
    pal = BaseColorPalette(colors=colors)
    region = C.identify_region(tuple(int(v) for v in d["c_click"]), cmap, frame=frame)
    assert np.array_equal(region.mask.cpu().numpy(), d["c_mask"])
    cfg = SolveConfig(outer_iterations=int(d["c_outer"]), refine=False)
    scores = [C._candidate_sparsity(frame, cmap, pal, region, k, EnergyWeights(), cfg, 0) for k in (1, 2, 3)]
    np.testing.assert_allclose(scores, d["c_scores"], rtol=0.05)
    assert C.correct_reflectance(region, frame, cmap, pal, config=cfg, max_workers=1) == int(d["c_pick"])
    # batched (all candidates in flight, one context + stream each): the same
    # kernels on the same inputs, so the same scores bit for bit
    batch = C._candidate_batch(frame, cmap, pal, region, (1, 2, 3), EnergyWeights(), cfg, 0)
    assert [batch[k] for k in (1, 2, 3)] == scores
    assert C.correct_reflectance(region, frame, cmap, pal, config=cfg) == int(d["c_pick"])
    assert C.correct_reflectance(region, frame, cmap, pal, config=cfg, max_workers=2) == int(d["c_pick"])
    # the corrected map carries the pick over the region
    region.corrected_id = int(d["c_pick"])
    fixed = C.apply_region_correction(cmap, region, pal)
    assert bool((fixed.ids[region.mask] == int(d["c_pick"])).all())


def test_edits_match_reference():
    from paper_1908_01961_b200 import editing as E
    from paper_1908_01961_b200.energy import LayerStack
    from paper_1908_01961_b200.imaging import Frame
    from paper_1908_01961_b200.palette import BaseColorPalette, ClusterMap
    d = np.load(G / "editing.npz")
    pal = BaseColorPalette(colors=d["e_colors"])
    L = LayerStack(torch.as_tensor(d["e_r"], dtype=torch.float32, device="cuda"),
                   torch.as_tensor(d["e_T"], dtype=torch.float32, device="cuda"))
    ids = torch.as_tensor(d["e_ids"], dtype=torch.int32, device="cuda")
    cmap = ClusterMap(ids=ids, r_cluster=torch.zeros(*ids.shape, 3, device="cuda"))
    out = E.recolor(L, pal, 2, d["e_new"], cmap)
    np.testing.assert_allclose(out.cpu().numpy(), d["e_recolor"], atol=1e-6)
    np.testing.assert_allclose(E.suppress_spill(L, pal, 3).cpu().numpy(), d["e_spill"], atol=1e-6)
    bg = Frame(torch.as_tensor(d["e_bg"], dtype=torch.float32, device="cuda"))
    out = E.rekey_background(L, pal, 1, bg, d["e_matte"])
    np.testing.assert_allclose(out.cpu().numpy(), d["e_rekey"], atol=1e-6)
    with pytest.raises(ValueError):
        E.suppress_spill(L, pal, 4)


def test_decompose_frames_with_clicks_tracks_the_region():
    from paper_1908_01961_b200 import synth
    from paper_1908_01961_b200.energy import EnergyWeights
    from paper_1908_01961_b200.palette import BaseColorPalette
    from paper_1908_01961_b200.pipeline import decompose_frames
    from paper_1908_01961_b200.solver import SolveConfig
    clip = synth.make_clip(48, 64, 3, 3, seed=5, device="cpu")
    pal = BaseColorPalette(colors=clip.colors)
    frames = [f.cuda() for f in clip.frames]
    res = decompose_frames(frames, EnergyWeights(), SolveConfig(outer_iterations=2, refine=False), palette=pal,
                           clicks=[(32, 24)])
    assert len(res.regions) == 1 and res.regions[0].corrected_id in (1, 2, 3)
    rid = res.regions[0].corrected_id
    for cm in res.cluster_maps:            # the correction is re-applied on every frame
        assert bool((cm.ids[res.regions[0].mask] == rid).any())

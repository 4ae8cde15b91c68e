"""Frame I/O and the per-frame write-out against the
reference's own files (tests/golden/frameio.json from tools/make_golden_io.py:
SHA-256 of every file pipeline.write_frame_outputs writes), plus the async
writer on the GPU."""
import hashlib
import json
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest

from paper_1908_01961_b200 import frameio

GOLDEN = Path(__file__).resolve().parent / "golden" / "frameio.json"


def _golden():
    g = json.loads(GOLDEN.read_text())
    colors = np.array(g["colors"])
    r, T, ids = np.array(g["r"]), np.array(g["T"]), np.array(g["ids"], dtype=np.int32)
    X = np.concatenate([r.transpose(2, 0, 1), T.transpose(2, 0, 1)]).astype(np.float32)
    return g, colors, X, ids


def _hashes(d: Path):
    return {str(p.relative_to(d)): hashlib.sha256(p.read_bytes()).hexdigest()
            for p in sorted(d.rglob("*")) if p.is_file()}


def test_write_frame_files_match_reference_bytes(tmp_path):
    g, colors, X, ids = _golden()
    frameio.write_frame_files(tmp_path, 3, X, colors, ids)
    assert _hashes(tmp_path) == g["files"]


def test_r_cluster_written_from_the_cluster_maps_palette(tmp_path):
    """after refinement the frame-1 cluster map still holds the
    pre-refinement palette's reflectance; the reference writes that map
    (pipeline.py:213-214), not colors[ids - 1] of the refined palette."""
    g, colors, X, ids = _golden()
    cc = np.array(g["cluster_colors"])
    frameio.write_frame_files(tmp_path, 1, X, colors, ids, ("colors", cc))
    assert _hashes(tmp_path) == g["files_cluster_palette"]
    d2 = tmp_path / "explicit"
    frameio.write_frame_files(d2, 1, X, colors, ids, ("array", cc[ids - 1]))
    assert _hashes(d2) == g["files_cluster_palette"]


def test_pfm_png_roundtrip_and_find_frames(tmp_path):
    from paper_1908_01961_b200.imaging import load_pfm, save_pfm
    a = np.random.default_rng(0).uniform(size=(5, 7, 3)).astype(np.float32)
    save_pfm(tmp_path / "frame_0002.pfm", a)
    assert np.array_equal(load_pfm(tmp_path / "frame_0002.pfm"), a.astype(np.float64))
    frameio.save_png_preview(tmp_path / "frame_0002.png", a)
    frameio.save_png_preview(tmp_path / "frame_0001.png", a)
    (tmp_path / "notes.txt").write_text("x")
    got = [p.name for p in frameio.find_frames(tmp_path)]
    assert got == ["frame_0001.png", "frame_0002.pfm"]          # PFM wins the tie
    ids = np.arange(35, dtype=np.int32).reshape(5, 7) % 3 + 1
    frameio.save_cluster_map(tmp_path / "c.png", tmp_path / "c.pfm", ids, a)
    i2, rc = frameio.load_cluster_map(tmp_path / "c.png", tmp_path / "c.pfm")
    assert np.array_equal(i2, ids) and np.array_equal(rc, a.astype(np.float64))


def test_write_diagnostics_format(tmp_path):
    rec = {"phase": "sparse", "accepted": True, "energy_before": 2.0, "energy_after": 1.0,
           "pcg": {"iterations": 16, "initial_residual": 3.0, "final_residual": 0.5},
           "terms": {"data": 0.75, "smoothness": 0.25}}
    frameio.write_diagnostics(tmp_path, SimpleNamespace(records=[[rec, {**rec, "phase": "dense"}]]))
    rows = [json.loads(l) for l in (tmp_path / "diagnostics.jsonl").read_text().splitlines()]
    assert rows[0] == {"frame": 1, "iteration": 0, "phase": "sparse", "accepted": True,
                       "energy_before": 2.0, "energy_after": 1.0, "pcg_initial": 3.0, "pcg_final": 0.5}
    csv = (tmp_path / "energy_terms.csv").read_text().splitlines()
    assert csv[0] == "frame,iteration,term,energy" and csv[1] == "1,0,data,0.75"


@pytest.mark.gpu
def test_async_writer_matches_sync_bytes(tmp_path):
    import torch
    from paper_1908_01961_b200.energy import LayerStack
    from paper_1908_01961_b200.palette import BaseColorPalette, cluster_map_from_ids
    g, colors, X, ids = _golden()
    pal = BaseColorPalette(colors=colors)
    w = frameio.AsyncFrameWriter(tmp_path, depth=2)
    for idx in (3, 4, 5):
        w.submit(idx, LayerStack(planes=torch.as_tensor(X).cuda()), pal,
                 cluster_map_from_ids(ids, pal, device=torch.device("cuda")))
    w.close()
    h = _hashes(tmp_path)
    for idx in (3, 4, 5):
        sub = {k.replace(f"frame_{idx:06d}", "frame_000003"): v for k, v in h.items()
               if k.startswith(f"frame_{idx:06d}")}
        assert sub == g["files"]
    # a cluster map segmented with another (pre-refinement) palette
    w = frameio.AsyncFrameWriter(tmp_path / "rc", depth=2)
    pal_c = BaseColorPalette(colors=np.array(g["cluster_colors"]))
    w.submit(1, LayerStack(planes=torch.as_tensor(X).cuda()), pal,
             cluster_map_from_ids(ids, pal_c, device=torch.device("cuda")))
    w.close()
    assert _hashes(tmp_path / "rc") == g["files_cluster_palette"]


@pytest.mark.gpu
def test_run_pipeline_disk_to_disk(tmp_path):
    from paper_1908_01961_b200 import synth
    from paper_1908_01961_b200.imaging import save_pfm
    from paper_1908_01961_b200.pipeline import run_pipeline
    from paper_1908_01961_b200.solver import SolveConfig
    clip = synth.make_clip(48, 64, 3, 3, seed=1, device="cpu")
    src = tmp_path / "in"
    src.mkdir()
    for i, f in enumerate(clip.frames):
        save_pfm(src / f"frame_{i + 1:04d}.pfm", f.numpy())
    res = run_pipeline(src, tmp_path / "out", config=SolveConfig(outer_iterations=2), k_max=4)
    out = tmp_path / "out"
    man = json.loads((out / "manifest.json").read_text())
    assert man["n_frames"] == 3 and man["K"] == res.palette.K
    K = res.palette.K
    for i in range(3):
        files = {p.name for p in (out / f"frame_{i + 1:06d}").iterdir()}
        assert len([f for f in files if f.endswith(".pfm")]) == K + 3     # R, direct, K indirect, r_cluster
        assert len([f for f in files if f.endswith(".png")]) == K + 4     # + reconstruction, cluster ids
    assert (out / "palette.json").exists() and (out / "diagnostics.jsonl").exists()

"""The UNMODIFIED reference package running on the B200 backend
(paper_1908_01961_b200.integration.install: the INTEGRATION.md patch).

The reference is installed into baseline/_ref by the recipe in DESIGN.md
(`pip install --no-index --no-deps --target baseline/_ref <copy of
/root/reference/pkg>`; git-ignored, it travels with the repo to the GPU box).
Its own `solve_frame` and `decompose_frames` run twice on the same inputs --
stock (NumPy fp64 on the host) and with the flip_flop seam swapped for the
device solver -- and the results are compared at the north-star gates.
Skipped when baseline/_ref is absent."""
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"


@pytest.fixture(scope="module")
def lumisplit():
    if not (REF / "lumisplit" / "__init__.py").exists():
        pytest.skip("reference package not installed in baseline/_ref")
    sys.path.insert(0, str(REF))
    try:
        import lumisplit as L
        import lumisplit.pipeline  # noqa: F401
        import lumisplit.refine  # noqa: F401
        yield L
    finally:
        sys.path.remove(str(REF))


def _frames(lumisplit, H, W, K, n, seed):
    from paper_1908_01961_b200 import synth
    clip = synth.make_clip(H, W, K, n, seed=seed, device="cpu")
    return [lumisplit.imaging.Frame(f.double().numpy()) for f in clip.frames], clip.colors


def _gate(frame, pal_a, la, pal_b, lb, frac_min=0.999):
    """Per layer: >= frac_min of the pixels within 1e-3 (R = exp(r), T_0,
    T_k), all within 1e-2; relative reconstruction energy within 1e-4."""
    d = np.concatenate([np.abs(np.exp(la.r) - np.exp(lb.r)), np.abs(la.T - lb.T)], axis=2)
    ok = (d <= 1e-3).mean(axis=(0, 1))
    assert ok.min() >= frac_min and d.max() <= 1e-2, (ok.tolist(), float(d.max()))

    def recon(pal, ls):
        B = np.vstack([np.ones((1, 3)), pal.colors])
        return float(np.sum((frame.data - np.exp(ls.r) * (ls.T @ B)) ** 2))
    ea, eb = recon(pal_a, la), recon(pal_b, lb)
    assert abs(ea - eb) <= 1e-4 * eb, (ea, eb)


def test_reference_solve_frame_on_the_device(lumisplit):
    from paper_1908_01961_b200 import integration
    L = lumisplit
    frames, colors = _frames(L, 48, 64, 3, 1, seed=5)
    pal = L.palette.BaseColorPalette(colors=colors)
    cmap = L.palette.segment(frames[0], pal)
    cfg = L.solver.SolveConfig(tol_rel=0.0, refine=False, outer_iterations=2)
    w = L.energy.EnergyWeights()
    ref = L.solver.solve_frame(frames[0], pal, cmap, w, cfg, seed=0)
    undo = integration.install(L)
    try:
        dev = L.solver.solve_frame(frames[0], pal, cmap, w, cfg, seed=0)
    finally:
        undo()
    assert isinstance(dev.layers, L.energy.LayerStack) and isinstance(dev.layers.r, np.ndarray)
    assert dev.status == ref.status and len(dev.records) == len(ref.records) == 4
    for a, b in zip(dev.records, ref.records):
        assert set(a) == set(b) and a["phase"] == b["phase"] == "sparse"
        assert a["accepted"] == b["accepted"] and a["alpha"] == b["alpha"]
        assert a["pcg"]["iterations"] == b["pcg"]["iterations"]
        assert np.isclose(a["energy_after"], b["energy_after"], rtol=1e-4)
        assert set(a["terms"]) == set(b["terms"])
    _gate(frames[0], dev.palette, dev.layers, ref.palette, ref.layers)
    assert L.solver.flip_flop.__module__ == "lumisplit.solver"      # uninstalled


def test_reference_decompose_frames_on_the_device(lumisplit):
    """decompose_frames (pipeline.py:87-167): the reference's own palette
    estimation, first-frame refinement race, streaming loop and region-free
    aux, with every solver step on the device."""
    from paper_1908_01961_b200 import integration
    L = lumisplit
    frames, _ = _frames(L, 40, 56, 3, 3, seed=6)
    w = L.energy.EnergyWeights()
    cfg = L.solver.SolveConfig(tol_rel=0.0, outer_iterations=4)
    ref = L.pipeline.decompose_frames(frames, w, cfg, seed=0, k_max=4)
    undo = integration.install(L)
    try:
        dev = L.pipeline.decompose_frames(frames, w, cfg, seed=0, k_max=4)
    finally:
        undo()
    assert dev.palette.K == ref.palette.K
    assert [[r["phase"] for r in rs] for rs in dev.records] == [[r["phase"] for r in rs] for rs in ref.records]
    assert np.abs(dev.palette.colors - ref.palette.colors).max() <= 1e-3
    assert dev.statuses == ref.statuses
    for f, la, lb in zip(frames, dev.layer_stacks, ref.layer_stacks):
        _gate(f, dev.palette, la, ref.palette, lb)
    R = dev.reflectances()[0]
    assert isinstance(R, np.ndarray) and R.shape == (40, 56, 3)

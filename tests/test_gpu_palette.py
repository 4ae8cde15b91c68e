"""First-frame palette estimation on the device (csrc/ls_palette.cu) against
the reference's own estimate_palette (tests/golden/palette.npz from
tools/make_golden_palette.py): same K, colors to fp64 summation-order
rounding, and the same cluster map."""
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden" / "palette.npz"


def _cases():
    with np.load(GOLDEN) as z:
        d = {k: z[k] for k in z.files}
    return [(d[f"c{i}_image"], int(d[f"c{i}_kmax"]), int(d[f"c{i}_seed"]), d[f"c{i}_colors"], d[f"c{i}_ids"])
            for i in range(int(d["n"]))]


@pytest.mark.parametrize("case", range(7))
def test_estimate_palette_matches_reference(case):
    from paper_1908_01961_b200.imaging import Frame
    from paper_1908_01961_b200.palette import estimate_palette
    img, k_max, seed, colors, ids = _cases()[case]
    pal, cmap = estimate_palette(Frame(torch.as_tensor(img).cuda()), k_max=k_max, seed=seed)
    assert pal.K == colors.shape[0]
    assert np.abs(pal.colors - colors).max() <= 1e-12
    assert np.array_equal(cmap.ids.cpu().numpy(), ids)


def test_estimate_palette_errors():
    from paper_1908_01961_b200.imaging import Frame
    from paper_1908_01961_b200.palette import EmptyHistogramError, estimate_palette
    dark = Frame(torch.zeros(16, 16, 3, device="cuda"))
    with pytest.raises(EmptyHistogramError):
        estimate_palette(dark)
    img = torch.rand(16, 16, 3, device="cuda")
    with pytest.raises(ValueError):
        estimate_palette(Frame(img), k_max=0)


def test_decompose_bundle_returns_layers_and_palette():
    """pipeline.py:170-177 over a synthetic bundle (palette estimated on the
    device from frame 1)."""
    from paper_1908_01961_b200 import synth
    from paper_1908_01961_b200.energy import EnergyWeights
    from paper_1908_01961_b200.pipeline import decompose_bundle
    from paper_1908_01961_b200.solver import SolveConfig
    clip = synth.make_clip(48, 64, 3, 3, seed=4, device="cuda")
    refl, illum, pal, res = decompose_bundle(clip, EnergyWeights(), SolveConfig(outer_iterations=3), k_max=4)
    assert len(refl) == len(illum) == 3 and pal.K >= 1
    assert tuple(refl[0].shape) == (48, 64, 3) and tuple(illum[0].shape) == (48, 64, 3)
    assert all(np.isfinite(r["energy_after"]) for rs in res.records for r in rs)

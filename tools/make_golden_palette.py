"""Golden fixture for first-frame palette estimation (reference
palette.py:81-238): runs the REFERENCE `estimate_palette` and its pieces
(build_histogram, weighted_kmeans) on float32-representable frames and stores
inputs and outputs in tests/golden/palette.npz.  Build container only
(imports /root/reference); the GPU test (tests/test_gpu_palette.py) needs
nothing but the .npz.

    python tools/make_golden_palette.py
"""
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))

from lumisplit import palette as P                 # noqa: E402
from lumisplit.imaging import Frame, chromaticity  # noqa: E402

from paper_1908_01961_b200 import synth            # noqa: E402


def cases():
    rng = np.random.default_rng(11)
    out = []
    # synthetic Voronoi frames (the bench generator), several palette sizes
    for i, (H, W, K, k_max, seed) in enumerate([(96, 128, 4, 10, 0), (120, 160, 6, 10, 3),
                                                (72, 96, 8, 12, 7), (64, 80, 3, 2, 1)]):
        clip = synth.make_clip(H, W, K, 1, seed=i, device="cpu")
        out.append((clip.frames[0].numpy().astype(np.float64), k_max, seed))
    # noisy frame: every histogram bin populated, many merges
    img = rng.uniform(0.0, 1.0, size=(50, 70, 3)).astype(np.float32).astype(np.float64)
    out.append((img, 10, 5))
    # dark regions (excluded from the histogram and the color means)
    clip = synth.make_clip(80, 100, 5, 1, seed=9, device="cpu")
    img = clip.frames[0].numpy().astype(np.float64)
    img[:20] = 0.001
    img[50:60, 10:90] = 0.0
    out.append((img.astype(np.float32).astype(np.float64), 10, 2))
    # two colors only (k_max larger than the populated bins)
    img = np.zeros((40, 60, 3))
    img[:, :30] = [0.8, 0.2, 0.1]
    img[:, 30:] = [0.1, 0.3, 0.7]
    out.append((img.astype(np.float32).astype(np.float64), 10, 0))
    return out


def main():
    d = {}
    for i, (img, k_max, seed) in enumerate(cases()):
        frame = Frame(img)
        hist = P.build_histogram(chromaticity(frame))
        centers = P.weighted_kmeans(hist, k_max, seed)
        pal, cmap = P.estimate_palette(frame, k_max=k_max, seed=seed)
        d[f"c{i}_image"] = img.astype(np.float32)
        d[f"c{i}_kmax"] = np.array(k_max)
        d[f"c{i}_seed"] = np.array(seed)
        d[f"c{i}_pop"] = hist.population
        d[f"c{i}_centers"] = centers
        d[f"c{i}_colors"] = pal.colors
        d[f"c{i}_ids"] = cmap.ids
        print(f"case {i}: {img.shape[:2]} k_max={k_max} seed={seed}: {centers.shape[0]} centers -> K={pal.K}")
    d["n"] = np.array(len(cases()))
    out = ROOT / "tests" / "golden" / "palette.npz"
    np.savez_compressed(out, **d)
    print(f"wrote {out}")


if __name__ == "__main__":
    main()

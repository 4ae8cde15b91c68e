"""Base-color palette types, segmentation and first-frame estimation
(reference palette.py).

`segment` (per streaming frame) runs on the device kernel, bit-identical to
palette.py:195-224.  `estimate_palette` is the first-frame histogram k-means
(palette.py:81-238) -- outside the solver hot path (SURVEY.md section 2,
row 6): ~100 histogram bins, so it runs on the host after one device copy.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np
import torch

from . import _device
from .imaging import Frame, chroma_of_color, chromaticity, as_cuda

HIST_BINS = 10
MERGE_DISTANCE = 0.2
KMEANS_MAX_ITERS = 100


class EmptyHistogramError(ValueError):
    """palette.py:23-24."""


@dataclass(frozen=True)
class BaseColorPalette:
    """K reflectance base colors; the illuminant is white (palette.py:48-70)."""

    colors: np.ndarray
    refined: bool = False
    previous: np.ndarray | None = None

    def __post_init__(self):
        c = self.colors
        if isinstance(c, torch.Tensor):
            c = c.detach().cpu().numpy()
        object.__setattr__(self, "colors", np.asarray(c, dtype=np.float64).reshape(-1, 3))

    @property
    def K(self) -> int:
        return int(self.colors.shape[0])

    @property
    def illuminant(self) -> np.ndarray:
        return np.ones(3)

    def matrix(self) -> np.ndarray:
        return np.vstack([np.ones((1, 3)), self.colors])

    def chromas(self) -> np.ndarray:
        return chroma_of_color(self.colors)


class ClusterMap:
    """Per-pixel cluster id (1..K) and clustered reflectance (palette.py:73-78).

    `ClusterMap(ids, r_cluster)` as in the reference; `segment` passes the
    palette instead and `r_cluster` (= colors[ids - 1]) is gathered on first
    access -- the streaming solve anchors on the ids alone, so a per-frame
    (H, W, 3) gather the solver never reads is not launched."""

    def __init__(self, ids, r_cluster=None, *, colors=None):
        if r_cluster is None and colors is None:
            raise ValueError("ClusterMap needs r_cluster or the palette colors")
        self.ids = ids              # (H, W) int32, CUDA
        self._r_cluster = r_cluster
        self._colors = colors

    @property
    def r_cluster(self):            # (H, W, 3) float32, CUDA
        if self._r_cluster is None:
            ids = self.ids
            cols = torch.as_tensor(self._colors, dtype=torch.float32, device=ids.device)
            self._r_cluster = cols[(ids - 1).long()]
        return self._r_cluster

    @r_cluster.setter
    def r_cluster(self, value):
        self._r_cluster = value

    def __repr__(self):
        return f"ClusterMap(ids={tuple(self.ids.shape)})"


def segment(frame: Frame, palette: BaseColorPalette, chroma=None) -> ClusterMap:
    """palette.py:195-224 on the device."""
    img = frame.data
    H, W = int(img.shape[0]), int(img.shape[1])
    bands = getattr(frame, "bands", 0)
    if bands and not isinstance(bands, int) and not bands.whole:
        # one band of a multi-process banded frame: the dark-pixel
        # inheritance crosses band boundaries (bands.BandedSolver.segment)
        ids = bands.segment(img, palette.colors)
    else:
        solver = _device.get_solver(img.device, H, W, palette.K)
        solver.set_image(img)
        solver.installed = None
        ids = solver.segment(palette.colors)
    return ClusterMap(ids=ids, colors=np.array(palette.colors, dtype=np.float64))


# ---- first-frame palette estimation (host; out of the hot path) -------------

def _histogram(chroma_np, inten_np, dark_np):
    valid = ~dark_np
    if not np.any(valid):
        raise EmptyHistogramError("all pixels are dark; nothing to cluster")
    c = chroma_np[valid]
    rb = np.clip((c[:, 0] * HIST_BINS).astype(np.int64), 0, HIST_BINS - 1)
    gb = np.clip((c[:, 1] * HIST_BINS).astype(np.int64), 0, HIST_BINS - 1)
    flat = gb * HIST_BINS + rb
    pop = np.bincount(flat, minlength=HIST_BINS * HIST_BINS)
    return pop.reshape(HIST_BINS, HIST_BINS)


def _kmeans(pop, k_max, seed):
    """palette.py:81-120: population-weighted farthest-point seeding + Lloyd."""
    if k_max < 1:
        raise ValueError("k_max must be >= 1")
    gb, rb = np.nonzero(pop)
    mids = np.stack([(rb + 0.5) / HIST_BINS, (gb + 0.5) / HIST_BINS], axis=-1)
    pops = pop[gb, rb]
    n = mids.shape[0]
    k = min(k_max, n)
    rng = np.random.default_rng(seed)
    chosen = [rng.choice(n, p=pops / pops.sum())]
    while len(chosen) < k:
        d = np.min(np.linalg.norm(mids[:, None, :] - mids[chosen][None, :, :], axis=2), axis=1)
        chosen.append(int(np.argmax(d)))
    centers = mids[chosen].copy()
    prev = None
    for _ in range(KMEANS_MAX_ITERS):
        assign = np.argmin(np.linalg.norm(mids[:, None, :] - centers[None], axis=2), axis=1)
        if prev is not None and np.array_equal(assign, prev):
            break
        prev = assign
        for j in range(k):
            sel = assign == j
            if np.any(sel):
                centers[j] = np.average(mids[sel], axis=0, weights=pops[sel])
    return centers


def _merge(centers, image_np, assign, dark_np):
    """palette.py:148-192: merge centers closer than 0.2, smaller into larger."""
    centers = centers.copy()
    valid = ~dark_np
    k = centers.shape[0]
    pops = np.array([np.count_nonzero((assign == j) & valid) for j in range(k)], dtype=np.int64)
    alive = list(range(k))
    while len(alive) > 1:
        best = None
        for ai in range(len(alive)):
            for bi in range(ai + 1, len(alive)):
                a, b = alive[ai], alive[bi]
                d = float(np.linalg.norm(centers[a] - centers[b]))
                if d < MERGE_DISTANCE and (best is None or d < best[0]):
                    best = (d, a, b)
        if best is None:
            break
        _, a, b = best
        small, large = (a, b) if pops[a] <= pops[b] else (b, a)
        assign[assign == small] = large
        pops[large] += pops[small]
        pops[small] = 0
        alive.remove(small)
    colors = []
    for j in alive:
        sel = (assign == j) & valid
        if np.any(sel):
            colors.append(image_np[sel].mean(axis=0))
        else:
            r, g = centers[j]
            colors.append(np.array([r, g, max(0.0, 1.0 - r - g)]))
    return BaseColorPalette(colors=np.array(colors))


def estimate_palette(frame: Frame, k_max: int = 10, seed: int = 0):
    """palette.py:227-238 -> (palette, cluster_map)."""
    ch = chromaticity(frame)
    chroma_np = ch.chroma.cpu().numpy()
    dark_np = ch.dark.cpu().numpy()
    image_np = frame.data.double().cpu().numpy()
    centers = _kmeans(_histogram(chroma_np, None, dark_np), k_max, seed)
    flat = chroma_np.reshape(-1, 2)
    assign = np.argmin(np.linalg.norm(flat[:, None, :] - centers[None], axis=2), axis=1)
    pal = _merge(centers, image_np, assign.reshape(chroma_np.shape[:2]), dark_np)
    return pal, segment(frame, pal)


def palette_to_json(palette: BaseColorPalette) -> dict:
    doc = {"K": palette.K, "colors": [[float(v) for v in c] for c in palette.colors]}
    if palette.refined:
        doc["refined"] = True
        if palette.previous is not None:
            doc["previous"] = [[float(v) for v in c] for c in palette.previous]
    return doc


def palette_from_json(doc: dict) -> BaseColorPalette:
    prev = doc.get("previous")
    return BaseColorPalette(colors=np.array(doc["colors"], dtype=np.float64),
                            refined=bool(doc.get("refined", False)),
                            previous=None if prev is None else np.array(prev))


def save_palette(path, palette: BaseColorPalette) -> None:
    with open(path, "w") as fh:
        json.dump(palette_to_json(palette), fh, indent=2)
        fh.write("\n")


def load_palette(path) -> BaseColorPalette:
    with open(path) as fh:
        return palette_from_json(json.load(fh))


def cluster_map_from_ids(ids, palette: BaseColorPalette, device=None) -> ClusterMap:
    ids_t = as_cuda(ids, dtype=torch.int32, device=device)
    cols = torch.as_tensor(palette.colors, dtype=torch.float32, device=ids_t.device)
    return ClusterMap(ids=ids_t, r_cluster=cols[(ids_t - 1).long()])

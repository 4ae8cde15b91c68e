"""Base-color palette types, segmentation and first-frame estimation
(reference palette.py).

`segment` (per streaming frame) runs on the device kernel, bit-identical to
palette.py:195-224.  `estimate_palette`, the first-frame histogram k-means
and merge (palette.py:81-238), runs on the device too (csrc/ls_palette.cu):
integer histogram, bit-exact k-means centers, merge in the last CTA.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np
import torch

from . import _device
from .imaging import Frame, chroma_of_color, chromaticity, as_cuda

HIST_BINS = 10            # palette.py:19-21 (the kernels' constants)
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


# ---- first-frame palette estimation (device, csrc/ls_palette.cu) ----------

def estimate_palette(frame: Frame, k_max: int = 10, seed: int = 0):
    """palette.py:227-238 -> (palette, cluster_map).  Histogram, weighted
    k-means (the first pick drawn from default_rng(seed) exactly as
    Generator.choice does) and the merge run on the device
    (ls_estimate_palette); the cluster map is `segment` with the result."""
    from . import _lib as L
    import ctypes as C
    if k_max < 1:
        raise ValueError("k_max must be >= 1")
    img = frame.data
    if not img.is_cuda:
        raise ValueError("estimate_palette needs a CUDA frame")
    H, W = int(img.shape[0]), int(img.shape[1])
    st = np.random.PCG64(seed).state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m64 = (1 << 64) - 1
    kk = min(int(k_max), L.MAX_K)
    out = np.zeros(3 * kk)
    K = C.c_int()
    lib = L.load()
    with torch.cuda.device(img.device):
        stream = torch.cuda.current_stream(img.device)
        rc = lib.ls_estimate_palette(C.c_void_p(img.contiguous().data_ptr()), H, W, kk, s >> 64, s & m64,
                                     inc >> 64, inc & m64, out.ctypes.data_as(L.DBL_P), C.byref(K),
                                     C.c_void_p(stream.cuda_stream))
    if rc != L.LS_OK:
        raise (ValueError if rc == L.LS_ERR_ARG else L.NativeError)(L.last_error())
    if K.value == 0:
        raise EmptyHistogramError("all pixels are dark; nothing to cluster")
    pal = BaseColorPalette(colors=out[:3 * K.value].reshape(K.value, 3).copy())
    return pal, segment(frame, pal)


# palette file format (palette.py:241-265): {"K", "colors"[, "refined",
# "previous"]}, indented two spaces, trailing newline
def palette_to_json(palette: BaseColorPalette) -> dict:
    rows = lambda a: np.asarray(a, dtype=np.float64).tolist()     # noqa: E731
    doc = dict(K=palette.K, colors=rows(palette.colors))
    if palette.refined:
        doc.update(refined=True)
        if palette.previous is not None:
            doc.update(previous=rows(palette.previous))
    return doc


def palette_from_json(doc: dict) -> BaseColorPalette:
    prev = doc.get("previous")
    return BaseColorPalette(colors=np.asarray(doc["colors"], dtype=np.float64),
                            refined=bool(doc.get("refined", False)),
                            previous=np.asarray(prev) if prev is not None else None)


def save_palette(path, palette: BaseColorPalette) -> None:
    from pathlib import Path
    Path(path).write_text(json.dumps(palette_to_json(palette), indent=2) + "\n")


def load_palette(path) -> BaseColorPalette:
    from pathlib import Path
    return palette_from_json(json.loads(Path(path).read_text()))


def cluster_map_from_ids(ids, palette: BaseColorPalette, device=None) -> ClusterMap:
    ids_t = as_cuda(ids, dtype=torch.int32, device=device)
    cols = torch.as_tensor(palette.colors, dtype=torch.float32, device=ids_t.device)
    return ClusterMap(ids=ids_t, r_cluster=cols[(ids_t - 1).long()])

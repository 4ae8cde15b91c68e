"""Deterministic synthetic clips for parity tests and the benchmark
(SURVEY.md section 8d "Concrete synthetic inputs").

Each clip is an exact factorisation I = R (*) sum_k b_k T_k (Eq. 2,
reference energy.py:97-99) of a Voronoi reflectance canvas, a smooth direct
layer and non-negative indirect bumps, panned and flickered per frame like
the reference's box-world renderer (synth.py:82-89, 400-404).  Frames are
float32 so the fp64 reference and the fp32 GPU path see identical inputs.

This is input generation, not solver code: it runs once, outside the timed
region, on whatever device the caller chooses.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

PAN_PX = 16          # maximum x-offset of the pan (2 * pingpong(t, 8))
CELLS_PER_FRAME = 64
BLUR_SIGMA = 0.8
BUMP_SIGMA = 12.0
FLICKER = 0.12


@dataclass
class Clip:
    frames: list          # list of (H, W, 3) float32 tensors
    colors: np.ndarray    # (K, 3) float64 palette (fp32-representable)
    truth_R: torch.Tensor  # (H, W+PAN_PX, 3) canvas reflectance
    K: int


def _chroma(c):
    s = c.sum(axis=-1, keepdims=True)
    return c[..., :2] / s


def make_palette(K: int, seed: int = 0) -> np.ndarray:
    """K colors uniform in [0.1, 0.95]^3 with pairwise chroma distance >= dmin
    (0.2 as in SURVEY 8d, relaxed geometrically when rejection keeps failing:
    eight mutually distant chromas do not always fit the sampling box)."""
    rng = np.random.default_rng(seed)
    dmin = 0.2
    while True:
        for _ in range(20000):
            cols = rng.uniform(0.1, 0.95, size=(K, 3))
            ch = _chroma(cols)
            d = np.linalg.norm(ch[:, None] - ch[None], axis=2) + np.eye(K)
            if d.min() >= dmin:
                return cols.astype(np.float32).astype(np.float64)
        dmin *= 0.85


def _pingpong(t: int, period: int) -> int:
    m = t % (2 * period)
    return m if m <= period else 2 * period - m


def _blur(img: torch.Tensor, sigma: float) -> torch.Tensor:
    """Separable Gaussian blur of an (H, W, C) tensor, reflect padding."""
    rad = max(1, int(math.ceil(3 * sigma)))
    x = torch.arange(-rad, rad + 1, dtype=img.dtype, device=img.device)
    k = torch.exp(-x * x / (2 * sigma * sigma))
    k = k / k.sum()
    t = img.permute(2, 0, 1).unsqueeze(1)                    # (C,1,H,W)
    t = torch.nn.functional.pad(t, (rad, rad, 0, 0), mode="reflect")
    t = torch.nn.functional.conv2d(t, k.view(1, 1, 1, -1))
    t = torch.nn.functional.pad(t, (0, 0, rad, rad), mode="reflect")
    t = torch.nn.functional.conv2d(t, k.view(1, 1, -1, 1))
    return t.squeeze(1).permute(1, 2, 0)


def make_clip(H: int, W: int, K: int, n_frames: int, seed: int = 0,
              device="cpu") -> Clip:
    """Render `n_frames` frames of an (H, W) clip with K base colors."""
    dev = torch.device(device)
    colors = make_palette(K, seed)
    Wc = W + PAN_PX
    rng = np.random.default_rng(seed + 1000)
    n_cells = max(K, int(round(CELLS_PER_FRAME * Wc / W)))
    pts = np.stack([rng.uniform(0, Wc, n_cells), rng.uniform(0, H, n_cells)], axis=1)
    cell_color = np.arange(n_cells) % K
    f64 = torch.float64
    P = torch.tensor(pts, dtype=f64, device=dev)
    ys = torch.arange(H, dtype=f64, device=dev)
    xs = torch.arange(Wc, dtype=f64, device=dev)
    yy, xx = torch.meshgrid(ys, xs, indexing="ij")
    # nearest seed (Voronoi), chunked over rows to bound memory at 4K
    owner = torch.empty(H, Wc, dtype=torch.long, device=dev)
    dk = torch.full((K, H, Wc), float("inf"), dtype=f64, device=dev)
    cc = torch.tensor(cell_color, device=dev)
    step = max(1, (1 << 22) // (Wc * n_cells))
    for y0 in range(0, H, step):
        y1 = min(H, y0 + step)
        d2 = (xx[y0:y1, :, None] - P[:, 0]) ** 2 + (yy[y0:y1, :, None] - P[:, 1]) ** 2
        owner[y0:y1] = d2.argmin(dim=2)
        for k in range(K):
            dk[k, y0:y1] = d2[:, :, cc == k].min(dim=2).values
    col = torch.tensor(colors, dtype=f64, device=dev)
    R = col[cc[owner]]                                          # (H, Wc, 3)
    R = _blur(R, BLUR_SIGMA).clamp(0.02, 1.0)
    T = torch.zeros(K + 1, H, Wc, dtype=f64, device=dev)
    T[0] = 0.5 + 0.3 * torch.sin(3 * xx / W) * torch.cos(2 * yy / H)
    T[1:] = 0.15 * torch.exp(-dk / (2 * BUMP_SIGMA ** 2))
    B = torch.cat([torch.ones(1, 3, dtype=f64, device=dev), col], 0)
    fl = np.random.default_rng(0).uniform(-1, 1, size=(n_frames, K + 1))
    gain_max = 1.0 + FLICKER
    S_max = torch.einsum("khw,kc->hwc", T, B) * gain_max
    scale = min(1.0, 0.98 / float((R * S_max).max()))
    T = T * scale
    frames = []
    for t in range(n_frames):
        off = 2 * _pingpong(t, 8)
        g = torch.tensor(1.0 + FLICKER * fl[t], dtype=f64, device=dev)
        Tt = T[:, :, off:off + W] * g[:, None, None]
        S = torch.einsum("khw,kc->hwc", Tt, B)
        I = (R[:, off:off + W] * S).clamp(0.0, 1.0)
        frames.append(I.to(torch.float32).contiguous())
    return Clip(frames=frames, colors=colors, truth_R=R, K=K)

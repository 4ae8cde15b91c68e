"""Clip decomposition entry point (reference pipeline.py:87-167).

`decompose_frames` keeps the reference signature and flow: frame 1 is
clustered (or takes the palette / cluster map given), refined and solved;
frames 2..N are re-segmented with the frozen palette and solved warm-started
with temporal consistency pairs.  Interactive misclustering correction
(`clicks`, correction.py) is outside this framework's scope (SURVEY.md
section 2, row 7) and is rejected explicitly.
"""

from __future__ import annotations

import logging
import time
from dataclasses import dataclass, field, replace

import torch

from .energy import EnergyWeights, LayerStack
from .imaging import Frame, as_cuda, chromaticity
from .palette import BaseColorPalette, ClusterMap, estimate_palette, segment
from .refine import refine_palette
from .solver import SolveConfig, SolverState, build_aux, flip_flop, initialize

log = logging.getLogger(__name__)


@dataclass
class PipelineResult:
    """pipeline.py:33-47."""

    palette: BaseColorPalette
    layer_stacks: list
    cluster_maps: list
    regions: list
    records: list
    statuses: list
    frame_seconds: list = field(default_factory=list)

    def reflectances(self) -> list:
        return [torch.exp(ls.r) for ls in self.layer_stacks]

    def illuminations(self) -> list:
        return [ls.illumination(self.palette) for ls in self.layer_stacks]


def _as_frame(f, bands=0) -> Frame:
    if isinstance(f, Frame):
        return f if (not bands or f.bands is bands) else Frame(f.data, bands=bands)
    return Frame(as_cuda(f), bands=bands)


class StreamingDecomposer:
    """The per-frame loop of decompose_frames (pipeline.py:113-166) as an
    object: `first(frame)` solves frame 1 (refinement when enabled), each
    `step(frame)` re-segments with the frozen palette and solves the frame
    warm-started from the previous one."""

    def __init__(self, palette: BaseColorPalette, weights: EnergyWeights, config: SolveConfig,
                 seed: int = 0, streaming_outer: int = 2, bands=0):
        self.bands = bands          # row bands (bands.py), 0 = whole frames
        self.palette = palette
        self.weights = weights
        self.config = config
        self.seed = seed
        self.stream_cfg = replace(config, refine=False, outer_iterations=streaming_outer)
        self.index = 0
        self.prev_layers = None
        self.prev_chroma = None

    def first(self, frame, cluster_map: ClusterMap | None = None) -> SolverState:
        frame = _as_frame(frame, self.bands)
        if cluster_map is None:
            cluster_map = segment(frame, self.palette)
        aux = build_aux(frame, cluster_map, seed=self.seed)
        layers = initialize(frame, cluster_map, self.palette)
        state = SolverState(frame=frame, palette=self.palette, layers=layers, aux=aux,
                            weights=self.weights, config=self.config)
        if self.config.refine:
            self.palette, _ = refine_palette(state)
        else:
            state.config = replace(state.config, refine=False)
            flip_flop(state)
            self.palette = state.palette
        state.cluster_map = cluster_map
        self.index = 1
        self.prev_layers = state.layers
        self.prev_chroma = chromaticity(frame)
        return state

    def step(self, frame) -> SolverState:
        frame = _as_frame(frame, self.bands)
        cmap = segment(frame, self.palette)
        aux = build_aux(frame, cmap, seed=self.seed + self.index, prev_chroma=self.prev_chroma,
                        prev_r=self.prev_layers.r)
        layers = initialize(frame, cmap, self.palette, previous=self.prev_layers)
        state = SolverState(frame=frame, palette=self.palette, layers=layers, aux=aux,
                            weights=self.weights, config=self.stream_cfg)
        flip_flop(state)
        state.cluster_map = cmap
        self.index += 1
        self.prev_layers = state.layers
        self.prev_chroma = chromaticity(frame)
        return state


def decompose_frames(frames: list, weights: EnergyWeights, config: SolveConfig, seed: int = 0,
                     k_max: int = 10, clicks: list | None = None, streaming_outer: int = 2,
                     palette: BaseColorPalette | None = None,
                     cluster_map: ClusterMap | None = None,
                     on_frame=None) -> PipelineResult:
    """Decompose an in-memory frame sequence (pipeline.py:87-167).

    Extra keyword arguments (not in the reference): `palette` /
    `cluster_map` skip first-frame estimation (SURVEY.md section 8d uses the
    generator palette); `on_frame(index, state)` is called after each frame
    (streams results out without keeping them)."""
    if not frames:
        raise ValueError("no frames")
    if clicks:
        raise NotImplementedError("misclustering correction (clicks) is outside lumisplit_b200's scope")
    f0 = _as_frame(frames[0])
    if palette is None:
        palette, cluster_map = estimate_palette(f0, k_max=k_max, seed=seed)
    result = PipelineResult(palette=palette, layer_stacks=[], cluster_maps=[], regions=[],
                            records=[], statuses=[])
    dec = StreamingDecomposer(palette, weights, config, seed=seed, streaming_outer=streaming_outer)
    for idx, f in enumerate(frames):
        t0 = time.perf_counter()
        state = dec.first(f0, cluster_map) if idx == 0 else dec.step(f)
        result.layer_stacks.append(state.layers)
        result.cluster_maps.append(state.cluster_map)
        result.records.append(state.records)
        result.statuses.append(state.status)
        result.frame_seconds.append(time.perf_counter() - t0)
        if on_frame is not None:
            on_frame(idx, state)
    result.palette = dec.palette
    return result


# disk-to-disk pipeline and per-frame outputs (pipeline.py:183-270)
from .frameio import (find_frames, run_pipeline, write_diagnostics,  # noqa: E402,F401
                      write_frame_outputs)

"""Clip decomposition entry point (reference pipeline.py:87-167).

`decompose_frames` keeps the reference signature and flow: frame 1 is
clustered (or takes the palette / cluster map given), refined and solved;
frames 2..N are re-segmented with the frozen palette and solved warm-started
with temporal consistency pairs.  First-frame clicks mark misclustered
regions (correction.py): each is flood-filled, its base color chosen by K
candidate solves, and the region is tracked and re-applied on every later
frame (pipeline.py:66-84, 100-106, 140-149).
"""

from __future__ import annotations

import logging
import time
from dataclasses import dataclass, field, replace

import torch

from .energy import EnergyWeights, LayerStack
from .imaging import Frame, as_cuda, chromaticity
from .palette import BaseColorPalette, ClusterMap, estimate_palette, segment
from .correction import apply_region_correction, correct_reflectance, identify_region, track_region
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
                 seed: int = 0, streaming_outer: int = 2, bands=0, regions=None):
        self.bands = bands          # row bands (bands.py), 0 = whole frames
        self.regions = list(regions or [])   # tracked misclustering corrections
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
        if self.regions:            # pipeline.py:140-149: track and re-apply corrections
            tracked = []
            for region in self.regions:
                nxt = track_region(region, cmap, frame_index=self.index)
                if nxt is None:
                    log.warning("frame %d: region from %s lost", self.index + 1, region.seed_xy)
                    continue
                tracked.append(nxt)
            for region in tracked:
                cmap = apply_region_correction(cmap, region, self.palette)
            self.regions = tracked
        aux = build_aux(frame, cmap, seed=self.seed + self.index, prev_chroma=self.prev_chroma,
                        prev_r=self.prev_layers.r)
        # warm start (solver.py:295-300): the reference deep-copies the previous
        # layers; the streaming flip-flop never writes its input state (the
        # graph copies it into its own ring and returns a new tensor), so the
        # previous frame's planes are passed as they are -- one 100 MB copy
        # per 1080p frame less
        layers = LayerStack(planes=self.prev_layers.X)
        state = SolverState(frame=frame, palette=self.palette, layers=layers, aux=aux,
                            weights=self.weights, config=self.stream_cfg)
        flip_flop(state)
        state.cluster_map = cmap
        self.index += 1
        self.prev_layers = state.layers
        self.prev_chroma = chromaticity(frame)
        return state


def journal_clicks(entries: list) -> list:
    """pipeline.py:60-63: first-frame click coordinates, in journal order."""
    return [(int(e["x"]), int(e["y"])) for e in entries
            if e.get("kind") == "click" and int(e.get("frame", 1)) == 1]


def read_journal(path) -> list:
    """pipeline.py:50-57: one JSON object per line."""
    import json
    with open(path) as fh:
        return [json.loads(line) for line in fh if line.strip()]


def _collect_regions(clicks, frame, cluster_map, palette, weights, config, seed):
    """pipeline.py:66-84: identify clicked regions (same-cluster clicks merge)
    and solve each region's corrected base color."""
    regions = []
    ids = cluster_map.ids
    for xy in clicks:
        sid = int(ids[int(xy[1]), int(xy[0])])
        existing = next((r for r in regions if r.source_id == sid), None)
        region = identify_region(xy, cluster_map, frame=frame, merge_into=existing)
        if existing is not None:
            regions[regions.index(existing)] = region
        else:
            regions.append(region)
    for region in regions:
        region.corrected_id = correct_reflectance(region, frame, cluster_map, palette, weights=weights,
                                                  seed=seed)
        log.info("region at %s (%d px): cluster %d -> %d", region.seed_xy, region.size,
                 region.source_id, region.corrected_id)
    return regions


def _reserve_results(n: int, f0: Frame, K: int) -> None:
    """The result keeps every frame's layer stack and cluster ids on the
    device (~(K+5) * 4 bytes per pixel per frame).  Grow the caching
    allocator by that much ONCE, before the loop: otherwise every retained
    frame costs a fresh cudaMalloc of ~100 MB at 1080p, which stalls the
    stream (measured: a 300-frame 1080p clip at 31 instead of 53 frames/s,
    tools/clip_probe.py).  Skipped when it would take more than half of the
    free device memory."""
    dev = f0.data.device
    if dev.type != "cuda" or n < 3:
        return
    H, W = int(f0.data.shape[0]), int(f0.data.shape[1])
    nbytes = int(n * H * W * 4 * (K + 5) * 1.05)
    free, _ = torch.cuda.mem_get_info(dev)
    if nbytes > free // 2:
        return
    block = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    del block          # stays cached in the allocator; frame results are carved out of it


def decompose_frames(frames: list, weights: EnergyWeights, config: SolveConfig, seed: int = 0,
                     k_max: int = 10, clicks: list | None = None, streaming_outer: int = 2,
                     palette: BaseColorPalette | None = None,
                     cluster_map: ClusterMap | None = None,
                     on_frame=None, bands=0) -> PipelineResult:
    """Decompose an in-memory frame sequence (pipeline.py:87-167).

    Extra keyword arguments (not in the reference): `palette` /
    `cluster_map` skip first-frame estimation (SURVEY.md section 8d uses the
    generator palette); `on_frame(index, state)` is called after each frame
    (streams results out without keeping them); `bands` solves every frame
    as row bands (bands.py; 0 = whole frames)."""
    if not frames:
        raise ValueError("no frames")
    f0 = _as_frame(frames[0], bands)
    if palette is None:
        palette, cluster_map = estimate_palette(f0, k_max=k_max, seed=seed)
    elif cluster_map is None:
        cluster_map = segment(f0, palette)
    regions = []
    if clicks:                      # pipeline.py:100-106
        regions = _collect_regions(clicks, f0, cluster_map, palette, weights, config, seed)
    for region in regions:
        cluster_map = apply_region_correction(cluster_map, region, palette)
    result = PipelineResult(palette=palette, layer_stacks=[], cluster_maps=[], regions=regions,
                            records=[], statuses=[])
    _reserve_results(len(frames), f0, palette.K)
    dec = StreamingDecomposer(palette, weights, config, seed=seed, streaming_outer=streaming_outer,
                              bands=bands, regions=regions)
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


def decompose_bundle(bundle, weights: EnergyWeights, config: SolveConfig, seed: int = 0, k_max: int = 10,
                     clicks: list | None = None):
    """pipeline.py:170-177: decompose_frames over a ground-truth bundle's
    frames (any object with `.frames`, e.g. the reference's
    GroundTruthBundle or synth.Clip); returns (reflectances,
    illuminations, palette, result)."""
    result = decompose_frames(list(bundle.frames), weights, config, seed=seed, k_max=k_max, clicks=clicks)
    return result.reflectances(), result.illuminations(), result.palette, result


# disk-to-disk pipeline and per-frame outputs (pipeline.py:183-270)
from .frameio import (find_frames, run_pipeline, write_diagnostics,  # noqa: E402,F401
                      write_frame_outputs)

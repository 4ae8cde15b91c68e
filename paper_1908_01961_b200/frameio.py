"""Frame I/O and per-frame outputs: the reference's
disk-to-disk pipeline (pipeline.py:183-270), PNG previews (imaging.py:104-114)
and cluster-map files (palette.py:268-279), with the layer write-out
overlapped with the solve.

`AsyncFrameWriter` copies a solved frame's planar state and cluster ids into
pinned host buffers on a side stream (the device -> host copy runs beside the
next frame's kernels) and a writer thread turns them into the reference's
file set -- K+2 PFMs and K+3 PNGs per frame -- so disk I/O never stalls the
GPU.  File contents follow the reference byte for byte (same PFM header,
row order and PNG encoding).
"""
from __future__ import annotations

import json
import queue
import re
import threading
from pathlib import Path

import numpy as np
import torch

from .imaging import GAMMA, load_frame, load_pfm, save_pfm

FRAME_RE = re.compile(r"^frame_(\d+)\.(png|pfm)$")          # pipeline.py:180
PREVIEW_INDIRECT_SCALE = 2.0       # pipeline.py:30


def save_png_preview(path, data, scale: float = 1.0) -> None:
    """imaging.py:104-114: 8-bit PNG preview with the display gamma."""
    from PIL import Image
    arr = np.clip(np.asarray(data, dtype=np.float64) * scale, 0.0, 1.0)
    if arr.ndim == 2:
        arr = np.repeat(arr[:, :, None], 3, axis=2)
    encoded = np.round((arr ** (1.0 / GAMMA)) * 255.0).astype(np.uint8)
    Image.fromarray(encoded, mode="RGB").save(path)


def save_cluster_map(ids_path, rc_path, ids: np.ndarray, r_cluster: np.ndarray) -> None:
    """palette.py:268-273: ids as 16-bit PNG, clustered reflectance as PFM."""
    from PIL import Image
    Image.fromarray(np.asarray(ids).astype(np.uint16)).save(ids_path)
    save_pfm(rc_path, r_cluster)


def load_cluster_map(ids_path, rc_path):
    """palette.py:276-279 -> (ids (H, W) int32, r_cluster (H, W, 3))."""
    from PIL import Image
    return np.asarray(Image.open(ids_path), dtype=np.int32), load_pfm(rc_path)


def find_frames(input_dir) -> list[Path]:
    """pipeline.py:183-194: frame_<n>.png / .pfm, PFM wins on a tie."""
    chosen = {}
    for p in sorted(Path(input_dir).iterdir()):
        m = FRAME_RE.match(p.name)
        if m:
            idx = int(m.group(1))
            if idx not in chosen or p.suffix == ".pfm":
                chosen[idx] = p
    return [chosen[i] for i in sorted(chosen)]


def cluster_reflectance(cluster_map):
    """What the reference writes as r_cluster.pfm (pipeline.py:213-214): the
    map's own clustered reflectance -- for a segmented map the colors of the
    palette it was segmented with (palette.py:223), which for frame 1 is the
    palette BEFORE refinement.  Returns ("colors", (K, 3)) when the map is
    the lazy ids -> colors gather, else ("array", (H, W, 3) host array)."""
    if getattr(cluster_map, "_r_cluster", None) is None and getattr(cluster_map, "_colors", None) is not None:
        return "colors", np.array(cluster_map._colors, dtype=np.float64)
    rc = cluster_map.r_cluster
    if isinstance(rc, torch.Tensor):
        rc = rc.detach().cpu().numpy()
    return "array", np.asarray(rc)


def write_frame_files(out_dir, index: int, X: np.ndarray, colors: np.ndarray, ids: np.ndarray,
                      r_cluster=None) -> None:
    """pipeline.py:197-214 from host arrays: X (U, H, W) planar state,
    colors (K, 3) (the palette the layers were solved with), ids (H, W);
    r_cluster = cluster_reflectance(cluster_map) (default: colors[ids - 1])."""
    frame_dir = Path(out_dir) / f"frame_{index:06d}"
    frame_dir.mkdir(parents=True, exist_ok=True)
    r = np.transpose(X[:3], (1, 2, 0)).astype(np.float64)
    T = np.transpose(X[3:], (1, 2, 0)).astype(np.float64)
    R = np.exp(r)
    save_pfm(frame_dir / "reflectance.pfm", R)
    save_png_preview(frame_dir / "reflectance.png", R)
    save_pfm(frame_dir / "direct.pfm", T[:, :, 0])
    save_png_preview(frame_dir / "direct.png", T[:, :, 0])
    for k in range(1, T.shape[2]):
        tinted = T[:, :, k, None] * colors[k - 1]
        save_pfm(frame_dir / f"indirect_{k:02d}.pfm", T[:, :, k])
        save_png_preview(frame_dir / f"indirect_{k:02d}.png", tinted, scale=PREVIEW_INDIRECT_SCALE)
    B = np.vstack([np.ones((1, 3)), colors])
    recon = R * np.tensordot(T, B, axes=([2], [0]))
    save_png_preview(frame_dir / "reconstruction.png", recon)
    kind, src = r_cluster if r_cluster is not None else ("colors", colors)
    r_cluster = src[np.asarray(ids, dtype=np.int64) - 1] if kind == "colors" else src
    save_cluster_map(frame_dir / "cluster_ids.png", frame_dir / "r_cluster.pfm", ids, r_cluster)


def write_frame_outputs(out_dir, index: int, layers, palette, cluster_map) -> None:
    """pipeline.py:197-214 (synchronous)."""
    X = layers.X.detach().float().cpu().numpy()
    ids = cluster_map.ids.detach().cpu().numpy() if isinstance(cluster_map.ids, torch.Tensor) \
        else np.asarray(cluster_map.ids)
    write_frame_files(out_dir, index, X, np.asarray(palette.colors, dtype=np.float64), ids,
                      cluster_reflectance(cluster_map))


class AsyncFrameWriter:
    """Overlaps the layer write-out with the solve.

    submit() enqueues the device -> pinned-host copies on a side stream after
    the current stream's work (no host synchronisation) and hands the buffers
    to a writer thread; at most `depth` frames are in flight (pinned buffers
    are recycled).  close() drains the queue and re-raises a writer error."""

    def __init__(self, out_dir, depth: int = 3):
        self.out_dir = Path(out_dir)
        self.depth = depth
        self.free: queue.Queue = queue.Queue()
        self.todo: queue.Queue = queue.Queue()
        self.shape = None
        self.stream = None
        self.error = None
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _buffers(self, X: torch.Tensor, ids: torch.Tensor):
        if self.shape != (tuple(X.shape), tuple(ids.shape)):
            self.shape = (tuple(X.shape), tuple(ids.shape))
            while not self.free.empty():
                self.free.get_nowait()
            for _ in range(self.depth):
                self.free.put((torch.empty(X.shape, dtype=torch.float32).pin_memory(),
                               torch.empty(ids.shape, dtype=torch.int32).pin_memory()))
        return self.free.get()

    def submit(self, index: int, layers, palette, cluster_map) -> None:
        if self.error is not None:
            raise self.error
        X = layers.X
        ids = cluster_map.ids
        if not isinstance(ids, torch.Tensor):
            ids = torch.as_tensor(np.asarray(ids), dtype=torch.int32, device=X.device)
        ids = ids.to(device=X.device, dtype=torch.int32)
        hX, hids = self._buffers(X, ids)
        if self.stream is None:
            self.stream = torch.cuda.Stream(device=X.device)
        done = torch.cuda.Event()
        self.stream.wait_stream(torch.cuda.current_stream(X.device))
        with torch.cuda.stream(self.stream):
            X.record_stream(self.stream)
            ids.record_stream(self.stream)
            hX.copy_(X, non_blocking=True)
            hids.copy_(ids, non_blocking=True)
            done.record(self.stream)
        self.todo.put((index, hX, hids, np.array(palette.colors, dtype=np.float64),
                       cluster_reflectance(cluster_map), done))

    def _run(self):
        while True:
            item = self.todo.get()
            if item is None:
                return
            index, hX, hids, colors, rc, done = item
            try:
                done.synchronize()
                write_frame_files(self.out_dir, index, hX.numpy(), colors, hids.numpy(), rc)
            except Exception as e:      # surfaced by the next submit() / close()
                self.error = e
            finally:
                self.free.put((hX, hids))

    def close(self) -> None:
        self.todo.put(None)
        self.thread.join()
        if self.error is not None:
            raise self.error


def write_diagnostics(out_dir, result) -> None:
    """pipeline.py:217-234: diagnostics.jsonl + energy_terms.csv."""
    out_dir = Path(out_dir)
    with open(out_dir / "diagnostics.jsonl", "w") as fh:
        for frame_idx, records in enumerate(result.records):
            for it, rec in enumerate(records):
                row = {"frame": frame_idx + 1, "iteration": it, "phase": rec["phase"],
                       "accepted": rec["accepted"], "energy_before": rec["energy_before"],
                       "energy_after": rec["energy_after"]}
                if "pcg" in rec:
                    row["pcg_initial"] = rec["pcg"]["initial_residual"]
                    row["pcg_final"] = rec["pcg"]["final_residual"]
                fh.write(json.dumps(row) + "\n")
    with open(out_dir / "energy_terms.csv", "w") as fh:
        fh.write("frame,iteration,term,energy\n")
        for frame_idx, records in enumerate(result.records):
            for it, rec in enumerate(records):
                for term, value in rec.get("terms", {}).items():
                    fh.write(f"{frame_idx + 1},{it},{term},{value:.10g}\n")


def run_pipeline(input_dir, output_dir, weights=None, config=None, seed: int = 0, k_max: int = 10,
                 journal=None, streaming_outer: int = 2, bands=0):
    """pipeline.py:237-270 disk to disk: read numbered frames, decompose,
    write layer sets (while the next frames solve), palette, diagnostics and
    the manifest.  The energy-history figure (report.py, matplotlib) is not
    produced."""
    from .energy import EnergyWeights
    from .palette import save_palette
    from .pipeline import decompose_frames
    from .solver import SolveConfig
    weights = weights or EnergyWeights()
    config = config or SolveConfig()
    paths = find_frames(input_dir)
    if not paths:
        raise IOError(f"no frame_*.png or frame_*.pfm files in {input_dir}")
    frames = [load_frame(p) for p in paths]
    clicks = None
    if journal is not None:                 # pipeline.py:250-252
        from .pipeline import journal_clicks, read_journal
        clicks = journal_clicks(read_journal(journal))
    out = Path(output_dir)
    out.mkdir(parents=True, exist_ok=True)
    writer = AsyncFrameWriter(out)

    def on_frame(idx, state):
        writer.submit(idx + 1, state.layers, state.palette, state.cluster_map)

    try:
        result = decompose_frames(frames, weights, config, seed=seed, k_max=k_max, clicks=clicks,
                                  streaming_outer=streaming_outer, on_frame=on_frame, bands=bands)
    finally:
        writer.close()
    save_palette(out / "palette.json", result.palette)
    write_diagnostics(out, result)
    with open(out / "manifest.json", "w") as fh:
        json.dump({"n_frames": len(frames), "K": result.palette.K, "statuses": result.statuses,
                   "frame_seconds": result.frame_seconds}, fh, indent=2)
        fh.write("\n")
    return result

"""Independent-clip sharding across GPUs (BASELINE.json configs[4]: 64 1080p
clips over 8 B200).

Frames inside a clip are sequential (frame t warm-starts from t-1 and pairs
with its reflectance, pipeline.py:151-153); different clips share nothing.
So the multi-GPU path is replicas: one process per GPU, a static round-robin
clip assignment, no data-path collective.  The only communication is for
reporting: total frames (sum) over the max-over-ranks device time.
"""

from __future__ import annotations

from dataclasses import dataclass


def shard(n_clips: int, world: int, rank: int) -> list[int]:
    """Round-robin clip indices owned by `rank` (disjoint, covering 0..n-1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    return list(range(rank, n_clips, world))


@dataclass
class Throughput:
    frames: int          # frames decomposed by all ranks
    seconds: float       # max over ranks
    per_rank_seconds: list

    @property
    def fps(self) -> float:
        return self.frames / self.seconds if self.seconds > 0 else float("inf")


def aggregate(frames_local: int, seconds_local: float, group=None) -> Throughput:
    """Sum frames and take the max time over ranks (torch.distributed, any
    backend; single process when not initialised)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return Throughput(frames_local, seconds_local, [seconds_local])
    world = dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
        else torch.device("cpu")
    f = torch.tensor([float(frames_local)], dtype=torch.float64, device=dev)
    dist.all_reduce(f, op=dist.ReduceOp.SUM, group=group)
    ts = [torch.zeros(1, dtype=torch.float64, device=dev) for _ in range(world)]
    dist.all_gather(ts, torch.tensor([seconds_local], dtype=torch.float64, device=dev), group=group)
    per = [float(t.item()) for t in ts]
    return Throughput(int(round(f.item())), max(per), per)


def decompose_clips(clips, weights, config, rank: int = 0, world: int = 1, streaming_outer: int = 2,
                    on_frame=None):
    """Decompose this rank's share of `clips` (each a (frames, palette)
    pair); returns {clip index: PipelineResult}."""
    from .pipeline import decompose_frames
    out = {}
    for ci in shard(len(clips), world, rank):
        frames, palette = clips[ci]
        out[ci] = decompose_frames(frames, weights, config, seed=ci, palette=palette,
                                   streaming_outer=streaming_outer,
                                   on_frame=None if on_frame is None else
                                   (lambda i, st, ci=ci: on_frame(ci, i, st)))
    return out

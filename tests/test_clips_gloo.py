"""Multi-process (gloo, world size 2, CPU) coverage of the N>1 path:
clip sharding and the throughput reduction used by bench.py --gpus N."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1908_01961_b200 import clips


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_clips, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = clips.shard(n_clips, world, rank)
        frames = 10 * len(mine)                 # 10 frames per clip
        secs = 1.0 + rank                       # rank 1 is the slow one
        th = clips.aggregate(frames, secs)
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        q.put((rank, mine, th.frames, th.seconds, th.per_rank_seconds, gathered))
    finally:
        dist.destroy_process_group()


def test_shard_disjoint_cover():
    for n in (1, 7, 64):
        for w in (1, 2, 3, 8):
            parts = [clips.shard(n, w, r) for r in range(w)]
            flat = sorted(i for p in parts for i in p)
            assert flat == list(range(n))
    with pytest.raises(ValueError):
        clips.shard(4, 2, 2)


def test_aggregate_single_process():
    th = clips.aggregate(30, 2.0)
    assert th.frames == 30 and th.seconds == 2.0 and th.fps == 15.0


def test_gloo_world2_sharding_and_max_time():
    world, n_clips = 2, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_clips, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    owned = sorted(i for r in res for i in r[1])
    assert owned == list(range(n_clips))
    for rank, mine, frames, secs, per, gathered in res:
        assert frames == 10 * n_clips          # sum over ranks
        assert secs == 2.0                      # max over ranks
        assert per == [1.0, 2.0]
        assert sorted(i for g in gathered for i in g) == list(range(n_clips))

"""The multi-GPU row-band path (DistExchange over NCCL, one band per rank,
band-local frames) exercised on the one GPU available: a world-size-1 NCCL
group.  The all-gathers, the SPMD (non-whole) BandedSolver mode, the
band-aware segmentation hook and the eager device-resident band flip-flop
all run for real; the result must be bitwise the whole-frame solve (one band
in band-partial mode is the whole-frame arithmetic)."""
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_dist_exchange_world1_equals_whole_frame():
    import torch.distributed as dist
    from paper_1908_01961_b200 import bands as B
    from paper_1908_01961_b200 import synth
    from paper_1908_01961_b200.energy import EnergyWeights
    from paper_1908_01961_b200.palette import BaseColorPalette
    from paper_1908_01961_b200.pipeline import StreamingDecomposer
    from paper_1908_01961_b200.solver import SolveConfig
    H, W, K = 96, 128, 3
    clip = synth.make_clip(H, W, K, 3, seed=8, device="cuda")
    pal = BaseColorPalette(colors=clip.colors)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        specs = B.plan_bands(H, 1)
        solver = B.BandedSolver(torch.device("cuda", 0), H, W, K, exchange=B.DistExchange(specs))
        runs = []
        for bands in (0, solver):
            dec = StreamingDecomposer(pal, EnergyWeights(), SolveConfig(tol_rel=0.0, outer_iterations=3),
                                      seed=0, bands=bands)
            sts = [dec.first(clip.frames[0])] + [dec.step(f) for f in clip.frames[1:]]
            runs.append(sts)
        for a, b in zip(*runs):
            assert a.records == b.records and a.status == b.status
            assert torch.equal(a.layers.X, b.layers.X)
            assert np.array_equal(a.palette.colors, b.palette.colors)
    finally:
        dist.destroy_process_group()

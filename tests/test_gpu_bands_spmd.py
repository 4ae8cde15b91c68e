"""The one-band-per-rank (SPMD) row-band path with TWO ranks: two processes,
each owning one band of the frame through DistExchange, exchanging band
partials (all-gather) and halo rows (P2P, the cut r/T halos) -- here over
gloo with host staging, because this box has one GPU and both ranks share
it (no kernel waits on another rank's kernel; the exchange is host-side).
The clip (refined frame 1 + streaming frames) must equal, bit for bit, the
same two bands solved in one process with the LocalExchange."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

H, W, K, NF = 96, 128, 3, 3


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _clip():
    from paper_1908_01961_b200 import synth
    return synth.make_clip(H, W, K, NF, seed=13, device="cpu")


def _cfg():
    from paper_1908_01961_b200.solver import SolveConfig
    return SolveConfig(tol_rel=0.0, outer_iterations=4)


def _rank(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1908_01961_b200 import bands as B
        from paper_1908_01961_b200.energy import EnergyWeights
        from paper_1908_01961_b200.palette import BaseColorPalette
        from paper_1908_01961_b200.pipeline import StreamingDecomposer
        dev = torch.device("cuda", 0)
        clip = _clip()
        specs = B.plan_bands(H, world)
        me = specs[rank]
        solver = B.BandedSolver(dev, H, W, K, exchange=B.DistExchange(specs))
        dec = StreamingDecomposer(BaseColorPalette(colors=clip.colors), EnergyWeights(), _cfg(), seed=0,
                                  bands=solver)
        frames = [f[me.ya:me.yb].contiguous().to(dev) for f in clip.frames]
        sts = [dec.first(frames[0])] + [dec.step(f) for f in frames[1:]]
        torch.cuda.synchronize()
        out = [(st.records, st.status, st.palette.colors.copy(),
                st.layers.X[:, me.y_lo:me.y_hi].cpu().numpy()) for st in sts]
        q.put((rank, out, None))
    except Exception as e:
        import traceback
        q.put((rank, None, traceback.format_exc() + repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_rank_bands_equal_local_bands_bitwise():
    from paper_1908_01961_b200 import bands as B
    from paper_1908_01961_b200.energy import EnergyWeights
    from paper_1908_01961_b200.palette import BaseColorPalette
    from paper_1908_01961_b200.pipeline import StreamingDecomposer
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, out, err = q.get(timeout=600)
        assert err is None, err
        res[r] = out
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # the same two bands, one process
    clip = _clip()
    dec = StreamingDecomposer(BaseColorPalette(colors=clip.colors), EnergyWeights(), _cfg(), seed=0, bands=world)
    sts = [dec.first(clip.frames[0].cuda())] + [dec.step(f.cuda()) for f in clip.frames[1:]]
    specs = B.plan_bands(H, world)
    for i, st in enumerate(sts):
        X = st.layers.X.cpu().numpy()
        for r in range(world):
            recs, status, colors, Xr = res[r][i]
            assert recs == st.records and status == st.status, (i, r)
            assert np.array_equal(colors, st.palette.colors)
            assert np.array_equal(Xr, X[:, specs[r].y0:specs[r].y1]), (i, r)

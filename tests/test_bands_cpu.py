"""CPU tests of the row-band host logic (bands.py): band geometry, halo
plans, the LocalExchange and -- with the gloo backend at world sizes 2 and
3 -- the DistExchange a multi-GPU run uses (all-gather order, P2P halo
refresh), and the cross-band carry of the dark-pixel inheritance against the
oracle's whole-frame segmentation."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lumisplit_oracle as O
from paper_1908_01961_b200 import bands as B


@pytest.mark.parametrize("H,n", [(2160, 2), (2160, 4), (2160, 8), (200, 5), (123, 3), (64, 1)])
def test_plan_bands_cover_rows_with_halos(H, n):
    specs = B.plan_bands(H, n)
    assert specs[0].y0 == 0 and specs[-1].y1 == H
    for a, b in zip(specs, specs[1:]):
        assert a.y1 == b.y0
    for s in specs:
        assert s.y1 - s.y0 >= min(H, B.HALO)
        assert s.ya == max(0, s.y0 - B.HALO) and s.yb == min(H, s.y1 + B.HALO)
        assert 0 <= s.y_lo < s.y_hi <= s.height
    if H % (8 * n) == 0:
        assert all((s.y0 % 8) == 0 for s in specs)


def _full(H, W, C=5, seed=0):
    g = torch.Generator().manual_seed(seed)
    return torch.rand(C, H, W, generator=g, dtype=torch.float64)


def _needed(s, H):
    """Mask of the halo cells the kernels read: R_HALO rows of the r planes
    and T_HALO rows of the T planes next to each band boundary."""
    m = torch.zeros(5, s.height, dtype=torch.bool)
    m[:, s.y_lo:s.y_hi] = True
    for planes, rows in ((slice(0, 3), B.R_HALO), (slice(3, None), B.T_HALO)):
        m[planes, max(0, s.y_lo - rows):s.y_lo] = True
        m[planes, s.y_hi:min(s.height, s.y_hi + rows)] = True
    return m


@pytest.mark.parametrize("full", [False, True])
def test_local_exchange_refreshes_every_halo(full):
    H, W = 70, 12
    specs = B.plan_bands(H, 4)
    ref = _full(H, W)
    locs = []
    for s in specs:
        t = ref[:, s.ya:s.yb].clone()
        t[:, :s.y_lo] = -1.0          # stale halos
        t[:, s.y_hi:] = -2.0
        locs.append(t)
    B.LocalExchange(specs).halo(locs, full=full)
    for s, t in zip(specs, locs):
        want = ref[:, s.ya:s.yb]
        if full:
            assert torch.equal(t, want)
        else:
            m = _needed(s, H)[:, :, None].expand_as(t)
            assert torch.equal(t[m], want[m])
            far = torch.zeros_like(m)           # the 8th halo row (nobody reads it) is not moved
            far[:, :max(0, s.y_lo - B.R_HALO)] = True
            far[:, s.y_hi + B.R_HALO:] = True
            assert (t[far] < 0).all()


def test_halo_pieces_cut_bytes():
    """r planes: 7 rows, T planes: 1 row per boundary instead of 8 rows of
    all U planes (U = 12 at K = 8: 30 / 96 of the rows)."""
    specs = B.plan_bands(2160, 4)
    for mv in B.halo_moves(specs):
        (a0, a1, r0, r1), (b0, b1, t0, t1) = B.halo_pieces(mv)
        assert (a0, a1, b0, b1) == (0, 3, 3, None)
        assert r1 - r0 == B.R_HALO and t1 - t0 == B.T_HALO
        assert (r0 <= t0 < t1 <= r1) and (t1 == r1 if mv[0] < mv[1] else t0 == r0)


def test_local_exchange_gather_is_band_ordered():
    specs = B.plan_bands(64, 3)
    parts = [torch.full((4,), float(i), dtype=torch.float64) for i in range(3)]
    g = B.LocalExchange(specs).gather(parts)
    assert all(torch.equal(x, g[0]) for x in g)
    assert torch.equal(g[0][:, 0], torch.tensor([0.0, 1.0, 2.0], dtype=torch.float64))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, H, W, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        specs = B.plan_bands(H, world)
        ex = B.DistExchange(specs)
        me = specs[rank]
        full = _full(H, W, seed=3)
        t = full[:, me.ya:me.yb].clone()
        t[:, :me.y_lo] = float("nan")
        t[:, me.y_hi:] = float("nan")
        ex.halo([t])
        m = _needed(me, H)[:, :, None].expand_as(t)
        ok_halo = torch.equal(t[m], full[:, me.ya:me.yb][m]) and bool(torch.isnan(t[~m]).all())
        t2 = t.clone()
        ex.halo([t2], full=True)
        ok_halo = ok_halo and torch.equal(t2, full[:, me.ya:me.yb])
        part = torch.tensor([rank * 10.0 + j for j in range(3)], dtype=torch.float64)
        (g,) = ex.gather([part])
        ok_gather = torch.equal(g, torch.tensor([[r * 10.0 + j for j in range(3)] for r in range(world)],
                                                dtype=torch.float64))
        # identical band-ordered sums on every rank (what k_band_finalize computes)
        s = 0.0
        for r in range(world):
            s += float(g[r, 1])
        q.put((rank, ok_halo, ok_gather, s))
    except Exception as e:      # report instead of leaving the parent waiting
        q.put((rank, False, False, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_dist_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 48, 8, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=90) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[1] and r[2] for r in res), res
    assert len({r[3] for r in res}) == 1


@pytest.mark.parametrize("n", [2, 3, 4])
def test_segment_carry_matches_whole_frame_segmentation(n):
    """Per-band raw ids + the gathered summaries reproduce O.segment."""
    rng = np.random.default_rng(n)
    H, W, K = 40, 9, 3
    colors = rng.uniform(0.1, 0.9, size=(K, 3))
    img = rng.uniform(0.0, 1.0, size=(H, W, 3))
    dark = np.zeros((H, W), bool)
    dark[:7] = True                     # dark frame start
    dark[15:29] = True                  # a dark run across band boundaries
    dark[33, 2:] = True
    img[dark] = 0.001
    ref = O.segment(img, colors)
    specs = B.plan_bands(H, n, halo=4, align=4)
    chroma, _, dk = O.chromaticity(img)
    raw = np.argmin(np.linalg.norm(chroma.reshape(-1, 1, 2) - O.chroma_of_colors(colors)[None], axis=2),
                    axis=1).reshape(H, W) + 1
    summ = np.zeros((n, 3), np.int64)
    for s in specs:
        own = ~dk[s.y0:s.y1].ravel()
        if own.any():
            r = raw[s.y0:s.y1].ravel()
            summ[s.index] = (1, r[np.argmax(own)], r[len(own) - 1 - np.argmax(own[::-1])])
    out = np.zeros((H, W), np.int64)
    for s in specs:
        carry = B.segment_carry(summ, s.index)
        r, d = raw[s.y0:s.y1].ravel(), dk[s.y0:s.y1].ravel()
        last, ids = carry, np.empty_like(r)
        for i in range(r.size):
            if not d[i]:
                last = r[i]
            ids[i] = last
        out[s.y0:s.y1] = ids.reshape(-1, W)
    assert np.array_equal(out, ref)


def test_zero_scan_ranges_partition_the_stream():
    GH, W = 2160, 3840
    for n in (1, 2, 3, 8):
        rs = [B.zero_scan_range(GH, W, n, b) for b in range(n)]
        assert rs[0][0] == 0 and rs[-1][1] == 12 * GH * W + 64
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))

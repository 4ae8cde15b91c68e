"""Row bands: one frame solved as horizontal bands of rows, one C-ABI context
per band (BASELINE configs[3], >= 4K frames split spatially
across GPUs).

The reference solves every frame as one problem (solver.py:143-192).  A band
context owns its rows [y0, y1) plus up to HALO = 8 halo rows on each side
(the consistency window reaches 7 rows, energy.py:23, 161-173; the gradient
stencils 1).  Each GN step is the same sequence of kernels as the
whole-frame path, issued per band:

    EG  -> gather partials -> finalise -> halo(z)
    16 x [ apply  -> gather -> finalise -> halo(p_i)
           update -> gather -> finalise -> halo(z) ]
    x = sum alpha_i p_i; halo(x); trials (gather, finalise, accept / halve); halo(X_out)

(every search direction p_i kept in its own buffer, ls_band_dirs, as in the
whole-frame loop).

Every reduction is a band partial (fp64, fixed order inside the band) and the
finalisation sums the gathered partials in band order on every band, so all
bands take bitwise identical scalar decisions, and a run with the bands on
one GPU gives the same bits as the same bands on separate GPUs.  Against the
whole-frame solve the only difference is the grouping of the fp64 sums.

Exchanges are pluggable:
  * LocalExchange -- every band in this process (one GPU, or several GPUs
    driven from one process): on one device a phase's gather + finalisation
    is one launch reading every band's partials in place
    (ls_band_finalize_group) and a halo exchange one launch (ls_copy_slabs).
  * DistExchange  -- one band per rank of a torch.distributed group (NCCL
    over NVLink on B200s; gloo in the CPU tests): all_gather_into_tensor of
    the partials, batched P2P send / recv of the halo rows.

The partner sampler stays bit-exact with the reference's single PCG64
stream: each band scans a slice of the stream for Lemire rejections
(ls_band_zero_scan), the lists are gathered, and every band draws its local
pixels with global pixel indices (ls_band_set_zeros + ls_sample_consistency).
Cluster ids follow the reference's raster-order dark-pixel inheritance across
band boundaries through a gathered 3-int summary per band (ls_band_segment).
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass
from types import SimpleNamespace

import numpy as np
import torch

from . import _device
from . import _lib as L

HALO = 8        # rows of halo each band keeps (consistency 7 + stencil 1)
R_HALO = 7      # rows of the 3 r planes a kernel reads across a boundary (energy.py:23)
T_HALO = 1      # rows of the T planes (gradient stencils, energy.py:272-291)


# ---------------------------------------------------------------------------
# band geometry
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class BandSpec:
    index: int
    y0: int          # own global rows [y0, y1)
    y1: int
    ya: int          # local region: global rows [ya, yb)
    yb: int

    @property
    def y_lo(self) -> int:
        return self.y0 - self.ya

    @property
    def y_hi(self) -> int:
        return self.y1 - self.ya

    @property
    def height(self) -> int:
        return self.yb - self.ya


def plan_bands(H: int, n: int, halo: int = HALO, align: int = 8) -> list[BandSpec]:
    """n bands of (nearly) equal height, boundaries on multiples of `align`
    rows (the kernels' tile height) where possible; every band at least
    `halo` rows tall so a halo comes from one neighbour."""
    if n < 1:
        raise ValueError("need at least one band")
    if n > 1 and H < n * halo:
        raise ValueError(f"{H} rows cannot hold {n} bands of >= {halo} rows")
    cuts = [0]
    for b in range(1, n):
        c = int(round(H * b / n / align)) * align
        c = min(max(c, cuts[-1] + halo), H - (n - b) * halo)
        cuts.append(c)
    cuts.append(H)
    out = []
    for b in range(n):
        y0, y1 = cuts[b], cuts[b + 1]
        out.append(BandSpec(b, y0, y1, max(0, y0 - halo), min(H, y1 + halo)))
    return out


def halo_moves(bands: list[BandSpec]):
    """Copies that refresh every halo: (src band, dst band, global rows
    [g0, g1)).  The rows are owned by src and lie in dst's halo."""
    moves = []
    for b in range(len(bands) - 1):
        up, dn = bands[b], bands[b + 1]
        # dn's top halo = up's last own rows; up's bottom halo = dn's first own rows
        moves.append((up.index, dn.index, dn.ya, dn.y0))
        moves.append((dn.index, up.index, up.y1, up.yb))
    return moves


def halo_pieces(move, r_planes: int = 3):
    """The parts of a halo move the kernels read: the R_HALO rows of the r
    planes and the T_HALO rows of the T planes nearest the boundary (the
    r planes' partner window reaches 7 rows, every stencil 1).  Returns
    [(plane0, plane1, g0, g1)] (plane1 None = to the last plane)."""
    s, d, g0, g1 = move
    if s < d:   # the upper band's last own rows -> the lower band's top halo
        return [(0, r_planes, max(g0, g1 - R_HALO), g1), (r_planes, None, max(g0, g1 - T_HALO), g1)]
    return [(0, r_planes, g0, min(g1, g0 + R_HALO)), (r_planes, None, g0, min(g1, g0 + T_HALO))]


def zero_scan_range(GH: int, W: int, n: int, b: int) -> tuple[int, int]:
    """Stream positions band b scans for rejections: the bands split
    [0, 12 N + 64) (dx, dy, temporal sections of energy.py:162-171 plus the
    shift the rejections themselves cause)."""
    total = 12 * GH * W + 64
    return total * b // n, total * (b + 1) // n


def segment_carry(summaries: np.ndarray, band: int) -> int:
    """palette.py:209-219 across bands: the id a dark pixel takes when no
    non-dark pixel precedes it inside its band (mirrors k_segment_band_final;
    used by the CPU tests)."""
    for b in range(band - 1, -1, -1):
        if summaries[b, 0]:
            return int(summaries[b, 2])
    for b in range(len(summaries)):
        if summaries[b, 0]:
            return int(summaries[b, 1])
    return 1


# ---------------------------------------------------------------------------
# exchanges
# ---------------------------------------------------------------------------
class LocalExchange:
    """All bands live in this process."""

    def __init__(self, bands: list[BandSpec]):
        self.bands = bands
        self.local = list(range(len(bands)))
        self.nbands = len(bands)

    def gather(self, parts: list[torch.Tensor]) -> list[torch.Tensor]:
        g = torch.stack([p.to(parts[0].device) for p in parts]).contiguous()
        return [g if p.device == g.device else g.to(p.device) for p in parts]

    def halo(self, tensors: list[torch.Tensor], full: bool = False):
        """tensors[i]: (U, H_loc, W) local tensor of band i.  Refreshes the
        halo rows the kernels read: on one device a copy costs a launch more
        than its bytes, so each move is ONE copy of the R_HALO rows next to
        the boundary in every plane (covering halo_pieces); full=True copies
        the whole HALO rows."""
        moves = []
        for mv in halo_moves(self.bands):
            src, dst = self.bands[mv[0]], self.bands[mv[1]]
            g0, g1 = (mv[2], mv[3]) if full else halo_pieces(mv)[0][2:4]
            moves.append((mv[0], mv[1], g0 - src.ya, g0 - dst.ya, g1 - g0))
        t0 = tensors[0]
        fused = (len(moves) <= 32 and t0.is_cuda and
                 all(t.dtype == torch.float32 and t.is_contiguous() and t.dim() == 3 and t.device == t0.device
                     for t in tensors))
        if not fused:
            for s_i, d_i, ys, yd, n in moves:
                tensors[d_i][:, yd:yd + n].copy_(tensors[s_i][:, ys:ys + n], non_blocking=True)
            return
        # one launch for every move (ls_copy_slabs): on one device each copy
        # costs a launch more than its bytes
        k = len(moves)
        srcs, dsts = (C.c_void_p * k)(), (C.c_void_p * k)()
        sst, dst_, cnt = (C.c_int64 * k)(), (C.c_int64 * k)(), (C.c_int64 * k)()
        pls = (C.c_int * k)()
        for i, (s_i, d_i, ys, yd, n) in enumerate(moves):
            ts, td = tensors[s_i], tensors[d_i]
            W = ts.shape[2]
            srcs[i] = ts.data_ptr() + 4 * ys * W
            dsts[i] = td.data_ptr() + 4 * yd * W
            sst[i], dst_[i] = ts.shape[1] * W, td.shape[1] * W
            cnt[i], pls[i] = n * W, ts.shape[0]
        lib = L.load()
        st = torch.cuda.current_stream(t0.device).cuda_stream
        rc = lib.ls_copy_slabs(k, srcs, dsts, sst, dst_, cnt, pls, C.c_void_p(st))
        if rc != L.LS_OK:
            raise L.NativeError(L.last_error())


class DistExchange:
    """One band per rank of a torch.distributed process group (rank r owns
    band r).  With NCCL the buffers stay on the device (NVLink P2P, all-
    gather); with gloo (CPU tests, or several ranks sharing one GPU) they are
    staged through host memory."""

    def __init__(self, bands: list[BandSpec], group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        if dist.get_world_size(group) != len(bands):
            raise ValueError("one band per rank")
        self.bands = bands
        self.local = [self.rank]
        self.nbands = len(bands)
        self.host = dist.get_backend(group) == "gloo"

    def _stage(self, t: torch.Tensor) -> torch.Tensor:
        return t.cpu() if self.host and t.is_cuda else t

    def gather(self, parts: list[torch.Tensor]) -> list[torch.Tensor]:
        (p,) = parts
        flat = self._stage(p.contiguous().view(-1))
        out = torch.empty(self.nbands * flat.numel(), dtype=p.dtype, device=flat.device)
        self.dist.all_gather_into_tensor(out, flat, group=self.group)
        return [out.to(p.device).view((self.nbands,) + tuple(p.shape))]

    def halo(self, tensors: list[torch.Tensor], full: bool = False):
        """Each move is one message: the r-plane rows and the T-plane rows the
        kernels read (halo_pieces), packed; full=True sends whole halos."""
        (t,) = tensors
        me = self.bands[self.rank]
        ops, recvs = [], []
        peer = lambda b: self.dist.get_global_rank(self.group, b) if self.group is not None else b
        for mv in halo_moves(self.bands):
            s, d = mv[0], mv[1]
            if self.rank not in (s, d):
                continue
            pieces = [(0, None, mv[2], mv[3])] if full else halo_pieces(mv)
            views = [t[p0:p1, g0 - me.ya:g1 - me.ya] for p0, p1, g0, g1 in pieces]
            if s == self.rank:
                buf = self._stage(torch.cat([v.reshape(-1) for v in views]))
                ops.append(self.dist.P2POp(self.dist.isend, buf, peer(d), self.group))
            else:
                buf = torch.empty(sum(v.numel() for v in views), dtype=t.dtype,
                                  device="cpu" if self.host else t.device)
                ops.append(self.dist.P2POp(self.dist.irecv, buf, peer(s), self.group))
                recvs.append((buf, views))
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()
        for buf, views in recvs:
            off = 0
            for v in views:
                v.copy_(buf[off:off + v.numel()].view(v.shape))
                off += v.numel()


# ---------------------------------------------------------------------------
# device views of a context's internal buffers
# ---------------------------------------------------------------------------
class _Cai:
    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 2}


def _view(ptr: int, shape, dtype, device) -> torch.Tensor:
    ts = {torch.float32: "<f4", torch.float64: "<f8"}[dtype]
    return torch.as_tensor(_Cai(ptr, shape, ts), device=device)


class _Band:
    def __init__(self, spec: BandSpec, device, GH: int, W: int, K: int):
        self.spec = spec
        self.solver = _device.DeviceSolver(device, spec.height, W, K)
        lib = self.solver.lib
        self.lib, self.ctx = lib, self.solver.ctx
        self.solver._chk(lib.ls_band_set(self.ctx, spec.ya, GH, spec.y_lo, spec.y_hi))
        ptrs = (C.c_void_p * 6)()
        self.solver._chk(lib.ls_band_buffers(self.ctx, ptrs))
        U, Hl = K + 4, spec.height
        self.bsum = _view(ptrs[0], (512,), torch.float64, device)
        self.z = _view(ptrs[1], (U, Hl, W), torch.float32, device)
        self.p = [_view(ptrs[2], (U, Hl, W), torch.float32, device),
                  _view(ptrs[3], (U, Hl, W), torch.float32, device)]
        self.x = _view(ptrs[4], (U, Hl, W), torch.float32, device)
        self.zlist = torch.zeros(L.ZERO_LIST, dtype=torch.int64, device=device)
        self.ring = None        # state buffers of the device-resident flip-flop
        self.dirs = None        # the kept PCG search directions (ls_band_dirs), U x Hl x W each
        self._shape = (U, Hl, W)
        self.summary = torch.zeros(3, dtype=torch.int32, device=device)

    def chk(self, rc):
        self.solver._chk(rc)

    def ensure_dirs(self, n: int):
        """Keep this band's PCG search directions (the whole-frame loop's
        layout: no x-update in the operator, x = sum alpha_i p_i once per GN
        step).  Left off (p ping-pong, deferred x) where the context keeps
        none (LS_X_DEFERRED=1, LS_PCG=cg1) or n is out of range."""
        if self.dirs is not None and len(self.dirs) >= n:
            return
        if not 1 <= n <= 64:
            return
        ptrs = (C.c_void_p * n)()
        if self.lib.ls_band_dirs(self.ctx, int(n), ptrs) != L.LS_OK:
            self.dirs = None
            return
        dev = self.solver.device
        self.dirs = [_view(ptrs[i], self._shape, torch.float32, dev) for i in range(n)]

    def pdir(self, it: int):
        """The buffer p_it lands in (its halo rows are exchanged)."""
        return self.dirs[it] if self.dirs is not None and it < len(self.dirs) else self.p[it & 1]


def _rec(**kw):
    return SimpleNamespace(**kw)


def _esum(terms) -> float:
    """Left-to-right fp64 sum of the block energies, as the whole-frame
    kernels / C host do (Python 3.12's sum() would compensate)."""
    e = 0.0
    for t in terms:
        e += float(t)
    return e


# ---------------------------------------------------------------------------
# the banded solver (duck-types the DeviceSolver calls solver.py makes)
# ---------------------------------------------------------------------------
class BandedSolver:
    """Solves full-frame problems as row bands.

    With a LocalExchange the state tensors passed in are whole frames
    (U, H, W): they are cut into band-local copies (own rows + halos), solved,
    and the own rows written back.  With a DistExchange they are this rank's
    band-local tensors (U, H_loc, W)."""

    def __init__(self, device, H: int, W: int, K: int, n: int | None = None, exchange=None,
                 halo: int = HALO):
        if exchange is None:
            exchange = LocalExchange(plan_bands(H, n, halo))
        self.exchange = exchange
        self.specs = exchange.bands
        self.device, self.H, self.W, self.K = device, H, W, K
        self.U = K + 4
        self.whole = isinstance(exchange, LocalExchange)
        self.bands = [_Band(self.specs[i], device, H, W, K) for i in exchange.local]
        self.installed = None
        self.cfg = None
        self._graph, self._graph_key, self._graph_steps = None, None, 0

    # -- plumbing ---------------------------------------------------------------
    def configure(self, weights, config):
        self.cfg = config
        for b in self.bands:
            b.solver.configure(weights, config)

    def _enter(self):
        for b in self.bands:
            b.solver._enter()

    def _local(self, X: torch.Tensor) -> list[torch.Tensor]:
        """Band-local copies of a state (whole-frame mode) or the state itself."""
        if not self.whole:
            return [X]
        return [X[:, b.spec.ya:b.spec.yb].contiguous() for b in self.bands]

    def _store(self, Xs: list[torch.Tensor], X_out: torch.Tensor):
        if not self.whole:
            if Xs[0].data_ptr() != X_out.data_ptr():
                X_out.copy_(Xs[0])
            return
        for b, Xb in zip(self.bands, Xs):
            X_out[:, b.spec.y0:b.spec.y1].copy_(Xb[:, b.spec.y_lo:b.spec.y_hi])

    def _gather_finalize(self, phase: int, nv: int, it: int = 0, alpha: float = 0.0):
        gs = self.exchange.gather([b.bsum[:nv].clone() for b in self.bands])
        for b, g in zip(self.bands, gs):
            b.chk(b.lib.ls_band_finalize(b.ctx, phase, L.dptr(g), len(self.specs), it, float(alpha)))
        self._keep = gs   # keep the gathered buffers alive until the kernels ran

    # -- per-frame state (energy.install for bands) -----------------------------
    def install(self, frame, aux):
        inst = self.installed
        if inst is not None and inst[0] is frame and inst[1] is aux:
            return
        if aux._recipe is None or aux._recipe[0] is not frame:
            raise NotImplementedError("row bands draw their own partners: build the aux with build_aux")
        _, seed, prev = aux._recipe
        img = frame.data
        self._enter()
        for b in self.bands:
            sl = slice(b.spec.ya, b.spec.yb) if self.whole else slice(None)
            b.solver.set_image(img[sl].contiguous())
        # partner draws: rejection positions of the global stream, then local draws
        st = np.random.PCG64(int(seed)).state["state"]
        s, inc = int(st["state"]), int(st["inc"])
        m64 = (1 << 64) - 1
        for b in self.bands:
            lo, hi = zero_scan_range(self.H, self.W, len(self.specs), b.spec.index)
            b.chk(b.lib.ls_band_zero_scan(b.ctx, s >> 64, s & m64, inc >> 64, inc & m64, lo, hi,
                                          L.dptr(b.zlist)))
        lists = self.exchange.gather([b.zlist for b in self.bands])
        for b, g in zip(self.bands, lists):
            b.chk(b.lib.ls_band_set_zeros(b.ctx, L.dptr(g), len(self.specs)))
            pc = None
            if prev is not None:
                pp = prev.planes
                pc = (pp[:, b.spec.ya:b.spec.yb] if self.whole else pp).contiguous()
            b.solver.sample(seed, None, pc)
        self._keep = lists
        ids = aux.cluster_ids
        for b in self.bands:
            sl = slice(b.spec.ya, b.spec.yb) if self.whole else slice(None)
            if ids is not None:
                t = torch.as_tensor(ids).to(device=self.device, dtype=torch.int32)
                b.solver.set_anchor(ids=t[sl].contiguous())
            elif aux.r_cluster_log is not None:
                rcl = torch.as_tensor(aux.r_cluster_log).to(device=self.device, dtype=torch.float32)
                b.solver.set_anchor(anchor_planes=rcl[sl].permute(2, 0, 1).contiguous())
            else:
                raise ValueError("EnergyAux needs cluster_ids or r_cluster_log")
            if aux.prev_r is not None:
                pr = torch.as_tensor(aux.prev_r).to(device=self.device, dtype=torch.float32)
                b.solver.set_prev_r(pr[sl].permute(2, 0, 1).contiguous())
            else:
                b.solver.set_prev_r(None)
        self.installed = (frame, aux)

    def segment(self, image: torch.Tensor, colors) -> torch.Tensor:
        """palette.segment (palette.py:195-224) band by band.  Whole-frame
        mode returns the (H, W) ids; otherwise this band's (H_loc, W) ids
        (own rows exact, halo rows unused)."""
        a, pa = L.dbl_array(colors)
        self._enter()
        for b in self.bands:
            sl = slice(b.spec.ya, b.spec.yb) if self.whole else slice(None)
            b.solver.set_image(image[sl].contiguous())
            b.chk(b.lib.ls_band_segment(b.ctx, pa, L.dptr(b.summary)))
        sums = self.exchange.gather([b.summary for b in self.bands])
        outs = []
        for b, g in zip(self.bands, sums):
            ids = torch.empty(b.spec.height, self.W, dtype=torch.int32, device=self.device)
            b.chk(b.lib.ls_band_segment_final(b.ctx, L.dptr(g), len(self.specs), b.spec.index, L.dptr(ids)))
            outs.append(ids)
        self.installed = None
        if not self.whole:
            return outs[0]
        full = torch.empty(self.H, self.W, dtype=torch.int32, device=self.device)
        for b, ids in zip(self.bands, outs):
            full[b.spec.y0:b.spec.y1] = ids[b.spec.y_lo:b.spec.y_hi]
        return full

    # -- one GN step (solver.py:143-192) ----------------------------------------
    def _gn_step_local(self, pa, Xs, Xouts, iters: int, max_halvings: int):
        bands, ex = self.bands, self.exchange
        for b, Xb in zip(bands, Xs):
            b.chk(b.lib.ls_band_eg(b.ctx, pa, L.dptr(Xb)))
        self._gather_finalize(L.BAND_EG, L.NUM_TERMS + 2)
        ex.halo([b.z for b in bands])
        for it in range(iters):
            for b, Xb in zip(bands, Xs):
                b.chk(b.lib.ls_band_pcg_apply(b.ctx, pa, L.dptr(Xb), it))
            self._gather_finalize(L.BAND_APPLY, 1, it)
            ex.halo([b.pdir(it) for b in bands])
            for b in bands:
                b.chk(b.lib.ls_band_pcg_update(b.ctx, it))
            self._gather_finalize(L.BAND_UPDATE, 2, it)
            ex.halo([b.z for b in bands])
        for b in bands:
            b.chk(b.lib.ls_band_pcg_finish(b.ctx))
        ex.halo([b.x for b in bands])
        info = np.zeros(21)
        alpha, e0, e1, accepted = 1.0, 0.0, 0.0, False
        rec = _rec(energy_before=0.0, energy_after=0.0, alpha=0.0, accepted=0, pcg_iterations=0,
                   initial_residual=0.0, final_residual=0.0, terms_before=[0.0] * 8, terms=[0.0] * 8)
        for h in range(max_halvings + 1):
            for b, Xb, Xo in zip(bands, Xs, Xouts):
                b.chk(b.lib.ls_band_trial(b.ctx, pa, L.dptr(Xb), float(alpha), L.dptr(Xo)))
            self._gather_finalize(L.BAND_TRIAL, L.NUM_TERMS, 0, alpha)
            b0 = bands[0]
            b0.chk(b0.lib.ls_band_read(b0.ctx, info.ctypes.data_as(L.DBL_P)))
            if h == 0:
                rec.terms_before = list(info[:8])
                e0 = _esum(info[:8])                     # block order (solver.py:139-140)
                rec.energy_before = e0
                rec.pcg_iterations = int(info[18])
                rec.initial_residual = float(np.sqrt(info[16]))
                rec.final_residual = float(np.sqrt(info[17]))
                if not np.isfinite(e0):
                    rec.terms = list(info[:8])
                    return L.LS_ERR_NONFINITE, rec
            e1 = _esum(info[8:16])
            if np.isfinite(e1) and e1 <= e0:
                accepted = True
                rec.terms = list(info[8:16])
                break
            alpha *= 0.5
        rec.accepted = 1 if accepted else 0
        rec.alpha = alpha if accepted else 0.0
        rec.energy_after = e1 if accepted else e0
        if not accepted:
            rec.terms = list(rec.terms_before)
        else:
            ex.halo(Xouts)
        return L.LS_OK, rec

    def _ensure_dirs(self):
        for b in self.bands:
            b.ensure_dirs(int(self.cfg.pcg_iterations))

    def gn_step(self, colors, X, X_out):
        a, pa = L.dbl_array(colors)
        self._enter()
        self._ensure_dirs()
        Xs = self._local(X)
        Xouts = [torch.empty_like(x) for x in Xs]
        rc, rec = self._gn_step_local(pa, Xs, Xouts, self.cfg.pcg_iterations, self.cfg.max_halvings)
        if rc == L.LS_OK and rec.accepted:
            self._store(Xouts, X_out)
        return rc, rec

    # -- energies / dense step (solver.py:207-255) ------------------------------
    def _energy_local(self, colors, Xs) -> np.ndarray:
        a, pa = L.dbl_array(colors)
        for b, Xb in zip(self.bands, Xs):
            b.chk(b.lib.ls_band_trial(b.ctx, pa, L.dptr(Xb), 0.0, None))
        self._gather_finalize(L.BAND_TRIAL, L.NUM_TERMS)
        info = np.zeros(21)
        b0 = self.bands[0]
        b0.chk(b0.lib.ls_band_read(b0.ctx, info.ctypes.data_as(L.DBL_P)))
        return info[8:16].copy()

    def energy_terms(self, colors, X) -> np.ndarray:
        self._enter()
        return self._energy_local(colors, self._local(X))

    def dense_step(self, colors, X):
        K = self.K
        cols = np.ascontiguousarray(np.asarray(colors, dtype=np.float64).ravel().copy())
        applied = np.zeros_like(cols)
        rec = _rec(energy_before=0.0, energy_after=0.0, alpha=0.0, delta_b_norm=0.0, accepted=0,
                   solved_nonzero=0)
        self._enter()
        Xs = self._local(X)
        use_ids = 1 if self.installed is not None and self.installed[1].cluster_ids is not None else 0
        a, pa = L.dbl_array(cols)
        ns = self.bands[0].lib.ls_band_dense_nsums(self.bands[0].ctx)
        for b, Xb in zip(self.bands, Xs):
            b.chk(b.lib.ls_band_dense_accum(b.ctx, pa, L.dptr(Xb), use_ids))
        gs = self.exchange.gather([b.bsum[:ns].clone() for b in self.bands])
        db = np.zeros(3 * K)
        b0, g0 = self.bands[0], gs[0]
        b0.chk(b0.lib.ls_band_dense_solve(b0.ctx, pa, L.dptr(g0), len(self.specs), use_ids,
                                          db.ctypes.data_as(L.DBL_P)))
        if not np.any(db != 0.0):
            return cols.reshape(K, 3), applied.reshape(K, 3), rec     # solver.py:218-219
        rec.solved_nonzero = 1
        big = float(np.max(np.abs(db)))
        if big > self.cfg.max_delta_b:                                # solver.py:221-224
            db = db * (self.cfg.max_delta_b / big)
        e0 = _esum(self._energy_local(cols, Xs))
        alpha, e1, accepted = 1.0, e0, False
        for _ in range(self.cfg.max_halvings + 1):                    # solver.py:226-243
            cand = np.minimum(1.0, np.maximum(0.0, cols + alpha * db))
            et = _esum(self._energy_local(cand, Xs))
            if np.isfinite(et) and et <= e0:
                applied = cand - cols
                nrm = 0.0                 # left-to-right, as ls_dense_step does
                for v in applied.tolist():
                    nrm += v * v
                rec.delta_b_norm = float(np.sqrt(nrm))
                cols = cand
                e1, accepted = et, True
                break
            alpha *= 0.5
        rec.energy_before = e0
        rec.energy_after = e1 if accepted else e0
        rec.accepted = 1 if accepted else 0
        rec.alpha = alpha if accepted else 0.0
        return cols.reshape(K, 3), applied.reshape(K, 3), rec

    # -- streaming flip-flop (solver.py:311-338, refine = False) ----------------
    def flip_flop_stream_host(self, colors, X0, outer: int, gn_steps: int, tol_rel: float):
        """Host-driven reference loop (one host decision per line-search
        trial); the device-resident flip_flop_stream must match it."""
        a, pa = L.dbl_array(colors)
        self._enter()
        self._ensure_dirs()
        Xs = self._local(X0)
        recs, e_prev, stalled = [], None, False
        status = 0
        for _ in range(outer):
            for _ in range(gn_steps):
                Xouts = [torch.empty_like(x) for x in Xs]
                rc, rec = self._gn_step_local(pa, Xs, Xouts, self.cfg.pcg_iterations, self.cfg.max_halvings)
                recs.append(rec)
                if rc == L.LS_ERR_NONFINITE:
                    out = torch.empty_like(X0)
                    self._store(Xs, out)
                    return rc, recs, 0, out, len(recs) - 1
                if rec.accepted:
                    Xs = Xouts
                else:
                    stalled = True
            hist = [r.energy_after for r in recs if r.accepted]
            if hist:
                e_now = hist[-1]
                if e_prev is not None and e_prev > 0.0:
                    rel = (e_prev - e_now) / e_prev
                    if 0.0 <= rel < tol_rel:
                        status = 2
                        break
                e_prev = e_now
        else:
            status = 1 if stalled else 0
        out = torch.empty_like(X0)
        if self.whole:
            out.copy_(X0)
        self._store(Xs, out)
        return L.LS_OK, recs, status, out, -1

    @staticmethod
    def _state_key(b) -> bytes:
        n = C.c_int64()
        buf = (C.c_char * 1024)()
        b.chk(b.lib.ls_state_key(b.ctx, buf, 1024, C.byref(n)))
        return bytes(buf[:min(1024, n.value)])

    @staticmethod
    def _launches(b) -> int:
        n = C.c_int64()
        b.chk(b.lib.ls_launch_count(b.ctx, C.byref(n)))
        return int(n.value)

    def _gfd(self, phase: int, nv: int, it: int = 0, alpha: float = 0.0, last: int = 0):
        """gather + device-side finalisation (ls_band_finalize_dev); every band
        in this process on one device: one ls_band_finalize_group launch
        reading all bands' partials in place."""
        if isinstance(self.exchange, LocalExchange) and len({b.solver.device for b in self.bands}) == 1:
            if getattr(self, "_group", None) is None or len(self._group) != len(self.bands):
                self._group = (C.c_void_p * len(self.bands))(*[b.ctx.value for b in self.bands])
            b0 = self.bands[0]
            b0.chk(b0.lib.ls_band_finalize_group(self._group, len(self.bands), phase, it, float(alpha), last))
            return
        gs = self.exchange.gather([b.bsum[:nv].clone() for b in self.bands])
        for b, g in zip(self.bands, gs):
            b.chk(b.lib.ls_band_finalize_dev(b.ctx, phase, L.dptr(g), len(self.specs), it, float(alpha), last))
        self._keep = gs

    def _enqueue_frame(self, pa, outer: int, gn_steps: int, tol_rel: float) -> int:
        """The whole device-resident frame (no host decision): enqueue only."""
        bands, ex = self.bands, self.exchange
        iters, mh = self.cfg.pcg_iterations, self.cfg.max_halvings
        self._enter()
        for b in bands:
            b.chk(b.lib.ls_band_frame_begin(b.ctx))
        k = 0
        for _ in range(outer):
            for _ in range(gn_steps):
                in_id, out_id = (0 if k == 0 else 1 + ((k - 1) & 1)), 1 + (k & 1)
                Xs = [b.ring[in_id] for b in bands]
                Xo = [b.ring[out_id] for b in bands]
                for b, Xb in zip(bands, Xs):
                    b.chk(b.lib.ls_band_eg(b.ctx, pa, L.dptr(Xb)))
                self._gfd(L.BAND_EG, L.NUM_TERMS + 2)
                ex.halo([b.z for b in bands])
                for it in range(iters):
                    for b, Xb in zip(bands, Xs):
                        b.chk(b.lib.ls_band_pcg_apply(b.ctx, pa, L.dptr(Xb), it))
                    self._gfd(L.BAND_APPLY, 1, it)
                    ex.halo([b.pdir(it) for b in bands])
                    for b in bands:
                        b.chk(b.lib.ls_band_pcg_update(b.ctx, it))
                    self._gfd(L.BAND_UPDATE, 2, it)
                    ex.halo([b.z for b in bands])
                for b in bands:
                    b.chk(b.lib.ls_band_pcg_finish(b.ctx))
                ex.halo([b.x for b in bands])
                alpha = 1.0
                for h in range(mh + 1):    # speculative trials, decided on the device
                    last = int(h == mh)
                    for b, Xb, Xob in zip(bands, Xs, Xo):
                        b.chk(b.lib.ls_band_trial_dev(b.ctx, pa, L.dptr(Xb), alpha, L.dptr(Xob), last))
                    self._gfd(L.BAND_TRIAL, L.NUM_TERMS, 0, alpha, last)
                    alpha *= 0.5
                for b, Xb, Xob in zip(bands, Xs, Xo):
                    b.chk(b.lib.ls_band_step_end(b.ctx, L.dptr(Xb), L.dptr(Xob), out_id))
                ex.halo(Xo)
                k += 1
            for b in bands:
                b.chk(b.lib.ls_band_outer_end(b.ctx, float(tol_rel)))
        return k

    def flip_flop_stream(self, colors, X0, outer: int, gn_steps: int, tol_rel: float, graph=None):
        """Device-resident streaming flip-flop over the bands, same contract
        as DeviceSolver.flip_flop_stream.  With every band in this process
        the frame is captured once as a CUDA graph (torch.cuda.graph) and
        replayed while palette and configuration are unchanged."""
        a, pa = L.dbl_array(colors)
        if outer * gn_steps > 256:
            raise ValueError("too many GN steps")
        self._enter()
        self._ensure_dirs()          # (allocations: before any capture)
        for b in self.bands:
            if b.ring is None:
                b.ring = [torch.empty((self.U, b.spec.height, self.W), dtype=torch.float32, device=self.device)
                          for _ in range(3)]
        for b, Xb in zip(self.bands, self._local(X0)):
            b.ring[0].copy_(Xb)
        if graph is None:
            import os
            graph = (self.whole and not os.environ.get("LS_NO_GRAPH")
                     and not any(b.solver.prof_on for b in self.bands))
        # everything the band kernels bake into their launch arguments: the
        # palette, the loop shape, and each band context's weights / config /
        # per-frame pointers and flags (prev_r present, ids vs anchor, ...)
        key = (np.asarray(colors, dtype=np.float64).tobytes(), outer, gn_steps, float(tol_rel),
               self.cfg.pcg_iterations, self.cfg.max_halvings,
               tuple(self._state_key(b) for b in self.bands))
        if graph:
            if self._graph is None or self._graph_key != key:
                g = torch.cuda.CUDAGraph()
                side = torch.cuda.Stream(device=self.device)
                side.wait_stream(torch.cuda.current_stream(self.device))
                before = [self._launches(b) for b in self.bands]
                with torch.cuda.stream(side):
                    with torch.cuda.graph(g, stream=side):
                        nsteps = self._enqueue_frame(pa, outer, gn_steps, tol_rel)
                torch.cuda.current_stream(self.device).wait_stream(side)
                self._graph_launches = [self._launches(b) - n0 for b, n0 in zip(self.bands, before)]
                for b, n in zip(self.bands, self._graph_launches):   # capture ran nothing
                    b.chk(b.lib.ls_add_launches(b.ctx, -n))
                self._graph, self._graph_key, self._graph_steps = g, key, nsteps
                self._enter()
            self._graph.replay()
            for b, n in zip(self.bands, self._graph_launches):
                b.chk(b.lib.ls_add_launches(b.ctx, n))
            nsteps = self._graph_steps
        else:
            nsteps = self._enqueue_frame(pa, outer, gn_steps, tol_rel)
        self._enter()
        results = []
        for b in self.bands:
            n = max(1, nsteps)
            recs = (L.GNRecord * n)()
            nrec, status, final, fault = C.c_int(), C.c_int(), C.c_int(), C.c_int()
            rc = b.lib.ls_band_frame_end(b.ctx, nsteps, recs, C.byref(nrec), C.byref(status), C.byref(final),
                                         C.byref(fault))
            if rc not in (L.LS_OK, L.LS_ERR_NONFINITE):
                b.chk(rc)
            results.append((rc, [recs[i] for i in range(nrec.value)], status.value, final.value, fault.value))
        rc, recs, status, final, fault = results[0]
        out = torch.empty_like(X0)
        if self.whole:
            out.copy_(X0)
        self._store([b.ring[final] for b in self.bands], out)
        return rc, recs, status, out, fault


_cache: dict = {}
_lock = threading.Lock()


def banded_solver(device, H: int, W: int, K: int, n: int) -> BandedSolver:
    """Cached whole-frame-mode solver with n bands on `device` (per thread)."""
    key = (device.index or 0, H, W, K, n, threading.get_ident())
    with _lock:
        s = _cache.get(key)
        if s is None:
            s = BandedSolver(device, H, W, K, n=n)
            _cache[key] = s
        return s

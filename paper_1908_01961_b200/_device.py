"""Device-side solver context: one C-ABI `ls_ctx` per (device, H, W, K,
host thread), caching the per-frame auxiliary state it has installed.

Everything here calls the sm_100a kernels through `_lib`; a missing library
or CUDA device raises (no CPU path).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np
import torch

from . import _lib as L

from collections import OrderedDict

# (device, H, W, K, thread, slot) -> DeviceSolver, least recently used first; the
# streaming loop reuses one entry, varying sizes (correction bounding boxes,
# segmentation of other frame sizes) are evicted beyond MAX_CONTEXTS
_cache: "OrderedDict" = OrderedDict()
_cache_lock = threading.Lock()
MAX_CONTEXTS = 32


def _device_of(t) -> torch.device:
    if isinstance(t, torch.Tensor) and t.is_cuda:
        return t.device
    if not torch.cuda.is_available():
        raise L.NativeError("lumisplit_b200 needs a CUDA device (B200); none is visible")
    return torch.device("cuda", torch.cuda.current_device())


def weights_struct(w) -> L.Weights:
    s = L.Weights()
    for name, _ in L.Weights._fields_:
        if name == "chroma_reg":
            s.chroma_reg = 1 if w.chroma_reg == "identity" else 0
        else:
            setattr(s, name, float(getattr(w, name)))
    return s


def config_struct(cfg) -> L.SolveCfg:
    s = L.SolveCfg()
    s.pcg_iterations = int(cfg.pcg_iterations)
    s.max_halvings = int(cfg.max_halvings)
    s.svd_truncation = float(cfg.svd_truncation)
    s.max_delta_b = float(cfg.max_delta_b)
    return s


class DeviceSolver:
    """Owns one ls_ctx; all tensors passed in are CUDA tensors on `device`."""

    def __init__(self, device: torch.device, H: int, W: int, K: int):
        self.lib = L.load()
        self.device = device
        self.H, self.W, self.K = H, W, K
        self.N = H * W
        self.U = K + 4
        self.ctx = C.c_void_p()
        from .energy import EnergyWeights
        from .solver import SolveConfig
        with torch.cuda.device(device):
            self._chk(self.lib.ls_ctx_create(device.index or 0, H, W, K,
                                             C.byref(weights_struct(EnergyWeights())),
                                             C.byref(config_struct(SolveConfig())),
                                             C.byref(self.ctx)))
        self.installed = None       # (frame_key, aux_key) of the installed frame context
        self._image_key = None      # ((ptr, shape, version), tensor) of the image in the context
        self.prof_on = False        # per-kernel CUDA events (no graph capture while on)
        self.sample_gen = 0         # bumps whenever the adjacency is rebuilt
        self.csr_owner = None       # device-backed ConsistencySamples using the adjacency

    def __del__(self):
        try:
            if self.ctx:
                self.lib.ls_ctx_destroy(self.ctx)
        except Exception:
            pass

    # -- plumbing -------------------------------------------------------------
    def _chk(self, rc: int):
        if rc == L.LS_OK:
            return
        msg = L.last_error()
        if rc == L.LS_ERR_ARG:
            raise ValueError(msg)
        if rc == L.LS_ERR_NONFINITE:
            raise FloatingPointError(msg)
        raise L.NativeError(msg)

    def _enter(self):
        stream = torch.cuda.current_stream(self.device)
        self.lib.ls_set_stream(self.ctx, C.c_void_p(stream.cuda_stream))

    def configure(self, weights, config):
        self._chk(self.lib.ls_set_weights(self.ctx, C.byref(weights_struct(weights)),
                                          C.byref(config_struct(config))))

    def profile(self, enable: bool):
        self.prof_on = bool(enable)
        self._enter()
        self._chk(self.lib.ls_profile(self.ctx, int(bool(enable))))

    def profile_read(self) -> dict:
        out = np.zeros(13)
        self._enter()
        self._chk(self.lib.ls_profile_read(self.ctx, out.ctypes.data_as(L.DBL_P)))
        names = ("energy_grad", "apply", "update", "trial", "dense")
        d = {n: {"count": int(out[2 * i]), "ms": float(out[2 * i + 1])} for i, n in enumerate(names)}
        d["launches"] = int(out[10])
        d["adjacency_entries"] = int(out[11])
        d["pairs"] = int(out[12])
        return d

    # -- per-frame context --------------------------------------------------------
    def set_image(self, image_hwc: torch.Tensor):
        """ls_set_image (image planes, chroma and edge gate), skipped when this
        context already holds exactly this tensor, unmodified: a streaming
        step installs its frame twice (segmentation, then the solve).  The
        key holds a reference to the tensor (so its memory cannot be reused
        under the same address) and torch's in-place version counter."""
        try:
            version = image_hwc._version
        except RuntimeError:        # inference tensors keep no version counter: never skip
            version = None
        key = (image_hwc.data_ptr(), tuple(image_hwc.shape), version)
        if (version is not None and self._image_key is not None and self._image_key[0] == key
                and self._image_key[1] is image_hwc):
            return
        self._enter()
        self._chk(self.lib.ls_set_image(self.ctx, L.dptr(image_hwc)))
        self._image_key = (key, image_hwc)

    def get_edge(self) -> torch.Tensor:
        self._enter()
        out = torch.empty(self.H, self.W, dtype=torch.float32, device=self.device)
        self._chk(self.lib.ls_get_edge(self.ctx, L.dptr(out)))
        return out

    def get_chroma(self) -> torch.Tensor:
        self._enter()
        out = torch.empty(2, self.H, self.W, dtype=torch.float64, device=self.device)
        self._chk(self.lib.ls_get_chroma(self.ctx, L.dptr(out)))
        return out

    def pair_count(self) -> int:
        n, t, e = C.c_int64(), C.c_int64(), C.c_int64()
        self._enter()
        self._chk(self.lib.ls_pair_count(self.ctx, C.byref(n), C.byref(t), C.byref(e)))
        return int(n.value)

    def sample(self, seed: int, chroma_planes=None, prev_chroma_planes=None) -> int:
        st = np.random.PCG64(int(seed)).state["state"]
        s, inc = int(st["state"]), int(st["inc"])
        m64 = (1 << 64) - 1
        n = C.c_int64(0)
        self._enter()
        self._chk(self.lib.ls_sample_consistency(
            self.ctx, L.dptr(chroma_planes), L.dptr(prev_chroma_planes),
            C.c_uint64(s >> 64), C.c_uint64(s & m64), C.c_uint64(inc >> 64),
            C.c_uint64(inc & m64), C.byref(n)))
        self.sample_gen += 1
        return int(n.value)

    def get_pairs(self, n: int | None = None):
        if n is None or n < 0:
            n = self.pair_count()
        src = torch.empty(n, dtype=torch.int64, device=self.device)
        dst = torch.empty(n, dtype=torch.int64, device=self.device)
        tmp = torch.empty(n, dtype=torch.uint8, device=self.device)
        self._enter()
        if n:
            self._chk(self.lib.ls_get_pairs(self.ctx, L.dptr(src), L.dptr(dst), L.dptr(tmp)))
        return src, dst, tmp.bool()

    def set_pairs(self, src, dst, temporal, weight=None):
        n = int(src.numel())
        t8 = temporal.to(device=self.device, dtype=torch.uint8).contiguous()
        s = src.to(device=self.device, dtype=torch.int64).contiguous()
        d = dst.to(device=self.device, dtype=torch.int64).contiguous()
        w = None
        if weight is not None:
            w = weight.to(device=self.device, dtype=torch.float64).contiguous()
            if bool(torch.all(w == 1.0)):
                w = None
        self._enter()
        self._chk(self.lib.ls_set_pairs(self.ctx, C.c_int64(n), L.dptr(s), L.dptr(d),
                                        L.dptr(t8), L.dptr(w)))
        self.sample_gen += 1

    def set_edge(self, edge: torch.Tensor):
        self._image_key = None      # the context's edge gate is no longer the image's
        self._enter()
        self._chk(self.lib.ls_set_edge(self.ctx, L.dptr(edge)))

    def set_prev_r(self, prev_planes):
        self._enter()
        self._chk(self.lib.ls_set_prev_r(self.ctx, L.dptr(prev_planes)))

    def set_anchor(self, ids=None, anchor_planes=None):
        self._enter()
        self._chk(self.lib.ls_set_anchor(self.ctx, L.dptr(ids), L.dptr(anchor_planes)))

    def segment(self, colors: np.ndarray) -> torch.Tensor:
        a, pa = L.dbl_array(colors)
        ids = torch.empty(self.H, self.W, dtype=torch.int32, device=self.device)
        self._enter()
        self._chk(self.lib.ls_segment(self.ctx, pa, L.dptr(ids)))
        return ids

    def initialize(self, colors: np.ndarray, ids: torch.Tensor) -> torch.Tensor:
        a, pa = L.dbl_array(colors)
        X = torch.empty(self.U, self.H, self.W, dtype=torch.float32, device=self.device)
        self._enter()
        self._chk(self.lib.ls_initialize(self.ctx, pa, L.dptr(ids), L.dptr(X)))
        return X

    # -- operators ---------------------------------------------------------------
    def energy_terms(self, colors, X, Y=None) -> np.ndarray:
        a, pa = L.dbl_array(colors)
        out = np.zeros(L.NUM_TERMS)
        self._enter()
        self._chk(self.lib.ls_energy_terms(self.ctx, pa, L.dptr(X), L.dptr(X if Y is None else Y),
                                           out.ctypes.data_as(L.DBL_P)))
        return out

    def unpack_hwc(self, planes: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        """(C, H, W) planes -> (H, W, C) interleaved (ls_unpack_hwc), on the
        current stream."""
        self._enter()
        self._chk(self.lib.ls_unpack_hwc(self.ctx, L.dptr(planes), int(planes.shape[0]), L.dptr(out)))
        return out

    # -- per-block residual protocol (ls_block_*, energy.py:194-452) ------------
    def block_rows(self, block: int, n_pairs: int) -> int:
        n = C.c_int64()
        self._chk(self.lib.ls_block_rows(self.ctx, int(block), int(n_pairs), C.byref(n)))
        return int(n.value)

    def block_call(self, op: str, colors, X0, block: int, pairs, vec=None, out=None):
        """op: residual / apply_j (vec = U planes, returns the rows) or
        apply_jt (vec = rows) / add_diag (accumulate into the U planes `out`)."""
        a, pa = L.dbl_array(colors)
        pr = pairs if pairs is not None else L.Pairs(0, None, None, None, None)
        self._enter()
        if op in ("residual", "apply_j"):
            rows = torch.empty(self.block_rows(block, pr.n), dtype=torch.float32, device=self.device)
            fn = self.lib.ls_block_residual if op == "residual" else self.lib.ls_block_apply_j
            self._chk(fn(self.ctx, pa, L.dptr(X0), int(block), C.byref(pr), L.dptr(vec), L.dptr(rows)))
            return rows
        if op == "apply_jt":
            self._chk(self.lib.ls_block_apply_jt(self.ctx, pa, L.dptr(X0), int(block), C.byref(pr), L.dptr(vec),
                                                 L.dptr(out)))
        else:
            self._chk(self.lib.ls_block_add_diag(self.ctx, pa, L.dptr(X0), int(block), C.byref(pr), L.dptr(out)))
        return out

    def grad_diag(self, colors, X):
        a, pa = L.dbl_array(colors)
        b = torch.empty_like(X)
        d = torch.empty_like(X)
        self._enter()
        self._chk(self.lib.ls_grad_diag(self.ctx, pa, L.dptr(X), L.dptr(b), L.dptr(d)))
        return b, d

    def apply(self, colors, X, p):
        a, pa = L.dbl_array(colors)
        out = torch.empty_like(X)
        self._enter()
        self._chk(self.lib.ls_apply_normal(self.ctx, pa, L.dptr(X), L.dptr(p), L.dptr(out)))
        return out

    def pcg(self, colors, X, iterations: int):
        a, pa = L.dbl_array(colors)
        x = torch.empty_like(X)
        info = np.zeros(3)
        self._enter()
        self._chk(self.lib.ls_pcg(self.ctx, pa, L.dptr(X), int(iterations), L.dptr(x),
                                  info.ctypes.data_as(L.DBL_P)))
        return x, {"iterations": int(info[0]), "initial_residual": float(info[1]),
                   "final_residual": float(info[2])}

    def gn_step(self, colors, X, X_out):
        a, pa = L.dbl_array(colors)
        rec = L.GNRecord()
        self._enter()
        rc = self.lib.ls_gn_step(self.ctx, pa, L.dptr(X), L.dptr(X_out), C.byref(rec))
        if rc not in (L.LS_OK, L.LS_ERR_NONFINITE):
            self._chk(rc)
        return rc, rec

    def flip_flop_stream(self, colors, X0, outer: int, gn_steps: int, tol_rel: float,
                         graph: bool | None = None):
        """Device-resident streaming flip-flop; returns (rc, records, status,
        final state tensor, fault step).  By default one CUDA-graph launch
        (ls_flip_flop_graph); LS_NO_GRAPH=1 or graph=False enqueues the
        kernels one by one (ls_flip_flop_stream) -- same results, bit for bit."""
        a, pa = L.dbl_array(colors)
        if graph is None:
            graph = not os.environ.get("LS_NO_GRAPH")
        if graph:
            Xo = torch.empty_like(X0)
            n = max(1, outer * gn_steps)
            recs = (L.GNRecord * n)()
            nrec, status, fault = C.c_int(), C.c_int(), C.c_int()
            self._enter()
            rc = self.lib.ls_flip_flop_graph(self.ctx, pa, L.dptr(X0), L.dptr(Xo), int(outer), int(gn_steps),
                                             float(tol_rel), recs, C.byref(nrec), C.byref(status), C.byref(fault))
            if rc not in (L.LS_OK, L.LS_ERR_NONFINITE):
                self._chk(rc)
            return rc, [recs[i] for i in range(nrec.value)], status.value, Xo, fault.value
        X1 = torch.empty_like(X0)
        X2 = torch.empty_like(X0)
        n = max(1, outer * gn_steps)
        recs = (L.GNRecord * n)()
        nrec, status, final, fault = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        self._enter()
        rc = self.lib.ls_flip_flop_stream(self.ctx, pa, L.dptr(X0), L.dptr(X1), L.dptr(X2), int(outer),
                                          int(gn_steps), float(tol_rel), recs, C.byref(nrec), C.byref(status),
                                          C.byref(final), C.byref(fault))
        if rc not in (L.LS_OK, L.LS_ERR_NONFINITE):
            self._chk(rc)
        return rc, [recs[i] for i in range(nrec.value)], status.value, (X0, X1, X2)[final.value], fault.value

    def dense_normal(self, colors, X, use_ids: bool):
        a, pa = L.dbl_array(colors)
        n = 3 * self.K
        A = np.zeros((n, n))
        rhs = np.zeros(n)
        self._enter()
        self._chk(self.lib.ls_dense_normal(self.ctx, pa, L.dptr(X), int(bool(use_ids)),
                                           A.ctypes.data_as(L.DBL_P), rhs.ctypes.data_as(L.DBL_P)))
        return A, rhs

    def svd_solve(self, A: np.ndarray, rhs: np.ndarray, truncation: float) -> np.ndarray:
        A = np.ascontiguousarray(A, dtype=np.float64)
        rhs = np.ascontiguousarray(rhs, dtype=np.float64).ravel()
        n = rhs.size
        x = np.zeros(n)
        self._enter()
        self._chk(self.lib.ls_svd_solve(self.ctx, n, A.ctypes.data_as(L.DBL_P),
                                        rhs.ctypes.data_as(L.DBL_P), float(truncation),
                                        x.ctypes.data_as(L.DBL_P)))
        return x

    def dense_step(self, colors, X):
        cols = np.ascontiguousarray(np.asarray(colors, dtype=np.float64).copy())
        applied = np.zeros_like(cols)
        rec = L.DenseRecord()
        self._enter()
        self._chk(self.lib.ls_dense_step(self.ctx, cols.ctypes.data_as(L.DBL_P), L.dptr(X),
                                         applied.ctypes.data_as(L.DBL_P), C.byref(rec)))
        return cols, applied, rec


def device_copy(dst: torch.Tensor, src: torch.Tensor) -> torch.Tensor:
    """dst <- src (same-size contiguous CUDA tensors) with an SM copy kernel on
    the current stream: a D2D cudaMemcpyAsync (torch's clone / copy_) runs on
    a copy engine and would queue behind a large host transfer."""
    if dst.numel() != src.numel() or dst.dtype != src.dtype or not (dst.is_contiguous() and src.is_contiguous()):
        raise ValueError("device_copy needs same-size contiguous tensors of one dtype")
    lib = L.load()
    st = torch.cuda.current_stream(src.device).cuda_stream
    rc = lib.ls_device_copy(L.dptr(dst), L.dptr(src), C.c_int64(src.numel() * src.element_size()), C.c_void_p(st))
    if rc != L.LS_OK:
        raise L.NativeError(L.last_error())
    return dst


def all_finite(t: torch.Tensor) -> bool:
    """No NaN / inf in a contiguous float32 CUDA tensor (synchronises the
    current stream; no copy-engine read-back)."""
    lib = L.load()
    flag = C.c_int(0)
    st = torch.cuda.current_stream(t.device).cuda_stream
    rc = lib.ls_all_finite(L.dptr(t), C.c_int64(t.numel()), C.c_void_p(st), C.byref(flag))
    if rc != L.LS_OK:
        raise L.NativeError(L.last_error())
    return bool(flag.value)


def chromaticity_planes(image_hwc: torch.Tensor) -> torch.Tensor:
    """(2, H, W) fp64 chroma planes of a CUDA (H, W, 3) float32 image."""
    lib = L.load()
    H, W = int(image_hwc.shape[0]), int(image_hwc.shape[1])
    out = torch.empty(2, H, W, dtype=torch.float64, device=image_hwc.device)
    st = torch.cuda.current_stream(image_hwc.device).cuda_stream
    rc = lib.ls_chromaticity(L.dptr(image_hwc), H, W, L.dptr(out), C.c_void_p(st))
    if rc != L.LS_OK:
        raise L.NativeError(L.last_error())
    return out


def edge_from_chroma(chroma_planes: torch.Tensor) -> torch.Tensor:
    lib = L.load()
    H, W = int(chroma_planes.shape[1]), int(chroma_planes.shape[2])
    out = torch.empty(H, W, dtype=torch.float32, device=chroma_planes.device)
    st = torch.cuda.current_stream(chroma_planes.device).cuda_stream
    rc = lib.ls_edge_from_chroma(L.dptr(chroma_planes), H, W, L.dptr(out), C.c_void_p(st))
    if rc != L.LS_OK:
        raise L.NativeError(L.last_error())
    return out


_slot = threading.local()


class solver_slot:
    """Context manager: inside it, get_solver hands out the contexts of slot
    `name` (distinct from the thread's default ones), so that several solves
    of the same size can be prepared and then run side by side, each on its
    own context and stream (correction.correct_reflectance)."""

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        self.prev = getattr(_slot, "name", None)
        _slot.name = self.name
        return self

    def __exit__(self, *exc):
        _slot.name = self.prev
        return False


def get_solver(device: torch.device, H: int, W: int, K: int) -> DeviceSolver:
    key = (device.index or 0, H, W, K, threading.get_ident(), getattr(_slot, "name", None))
    with _cache_lock:
        s = _cache.get(key)
        if s is None:
            s = DeviceSolver(device, H, W, K)
            _cache[key] = s
            while len(_cache) > MAX_CONTEXTS:     # the context is freed with its last reference
                _cache.popitem(last=False)
        else:
            _cache.move_to_end(key)
        return s


def flip_flop_batch(solvers, streams, colors, X0s, outer: int, gn_steps: int, tol_rel: float):
    """ls_flip_flop_batch: the device-resident flip-flop of every solver (one
    context each, its state X0s[i]) enqueued on streams[i] before any is
    waited for.  Returns per solver (rc, records, status, final state, fault
    step) as DeviceSolver.flip_flop_stream does; rc is the solver's own code."""
    n = len(solvers)
    if n == 0:
        return []
    lib = solvers[0].lib
    a, pa = L.dbl_array(colors)
    X1s, X2s = [], []
    for s, st, X0 in zip(solvers, streams, X0s):
        with torch.cuda.stream(st):
            X1s.append(torch.empty_like(X0))
            X2s.append(torch.empty_like(X0))
        lib.ls_set_stream(s.ctx, C.c_void_p(st.cuda_stream))
    per = max(1, outer * gn_steps)
    recs = (L.GNRecord * (n * per))()
    ptrs = lambda ts: (C.c_void_p * n)(*[t.data_ptr() for t in ts])     # noqa: E731
    ints = lambda: (C.c_int * n)()                                      # noqa: E731
    nrec, status, final, fault, rcs = ints(), ints(), ints(), ints(), ints()
    ctxs = (C.c_void_p * n)(*[s.ctx.value for s in solvers])
    solvers[0]._chk(lib.ls_flip_flop_batch(ctxs, n, pa, ptrs(X0s), ptrs(X1s), ptrs(X2s), int(outer),
                                           int(gn_steps), float(tol_rel), recs, nrec, status, final,
                                           fault, rcs))
    out = []
    for i in range(n):
        X = (X0s[i], X1s[i], X2s[i])[final[i]]
        out.append((rcs[i], [recs[i * per + j] for j in range(nrec[i])], status[i], X, fault[i]))
    return out


def utility_solver(device=None) -> DeviceSolver:
    """A 1x1 context for size-independent device work (the SVD solve)."""
    dev = device if device is not None else _device_of(None)
    return get_solver(dev, 1, 1, 0)


def clear_cache():
    with _cache_lock:
        _cache.clear()

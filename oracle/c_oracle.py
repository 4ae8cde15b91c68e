"""ctypes front end of the compiled CPU restatement (oracle/ls_oracle.c).

TEST / MEASUREMENT INFRASTRUCTURE ONLY: imported by tests/ and by bench.py's
cpu_baseline leg and `--impl reference` arm, never by the product package.

Mirrors the NumPy oracle's API (`lumisplit_oracle.py`: Weights, Config, Aux,
Pairs, State, FrozenSystem-like operators, gn_step_sparse, flip_flop,
solve_frame, decompose_clip) so a test can run either; the C one is what
makes the 1920x1080 K=8 headline configuration checkable in seconds and the
CPU baseline measurable at full size.  Arrays are fp64 in the reference's
(H, W, C) layout.
"""

from __future__ import annotations

import ctypes as C
import subprocess
from dataclasses import replace
from pathlib import Path

import numpy as np

from . import lumisplit_oracle as O

HERE = Path(__file__).resolve().parent
LIB = HERE / "libls_oracle.so"

_lib = None


class _W(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("lam_d", "lam_cl", "lam_rs", "p", "lam_rc", "lam_m", "lam_is",
                                          "lam_sm", "lam_nn", "lam_ir", "lam_cr", "eps_nn", "eps_irls")] + \
               [("chroma_reg", C.c_int)]


class _Cfg(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("outer_iterations", "gn_steps", "pcg_iterations", "max_halvings",
                                       "refine", "refine_warmup")] + \
               [(n, C.c_double) for n in ("tol_rel", "svd_truncation", "max_delta_b", "refine_gate_rel")]


class Rec(C.Structure):
    _fields_ = [("phase", C.c_int), ("accepted", C.c_int), ("pcg_iterations", C.c_int), ("pad", C.c_int)] + \
               [(n, C.c_double) for n in ("energy_before", "energy_after", "alpha", "initial_residual",
                                          "final_residual", "delta_b_norm")] + \
               [("terms", C.c_double * 8)]


P = C.c_void_p
D = C.POINTER(C.c_double)
_SIG = {
    "or_set_threads": ([C.c_int], None),
    "or_max_threads": ([], C.c_int),
    "or_chromaticity": ([C.c_int, C.c_int, P, P, P], None),
    "or_edge_gate": ([C.c_int, C.c_int, P, P], None),
    "or_sample_consistency": ([C.c_int, C.c_int, P, P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                               P, P, P], C.c_int64),
    "or_segment": ([C.c_int, C.c_int, P, C.c_int, P, P], None),
    "or_initialize": ([C.c_int, C.c_int, C.c_int, P, P, P, P, P], None),
    "or_sys_create": ([C.c_int, C.c_int, C.c_int, C.POINTER(_W), P, P, P, C.c_int64, P, P, P, P, P, P, P], P),
    "or_sys_free": ([P], None),
    "or_sys_set_colors": ([P, P], None),
    "or_linearize": ([P, P, P], None),
    "or_terms": ([P, P, P, P], C.c_int),
    "or_grad_diag": ([P, P, P], None),
    "or_apply": ([P, P, P], None),
    "or_pcg": ([P, P, P, C.c_int, P, P], None),
    "or_gn_step": ([P, P, P, C.c_int, C.c_int, C.POINTER(Rec)], C.c_int),
    "or_dense_normal": ([P, P, P, C.c_int, P, P], None),
    "or_svd_solve": ([C.c_int, P, P, C.c_double, P], None),
    "or_dense_step": ([P, P, P, C.POINTER(_Cfg), C.POINTER(Rec), P], C.c_int),
    "or_flip_flop": ([P, P, P, P, C.POINTER(_Cfg), C.POINTER(Rec), C.c_int, C.POINTER(C.c_int),
                      C.POINTER(C.c_int)], C.c_int),
}


def build() -> Path:
    """Compile the library if it is missing or older than its source."""
    src = HERE / "ls_oracle.c"
    if not LIB.exists() or LIB.stat().st_mtime < max(src.stat().st_mtime, (HERE / "Makefile").stat().st_mtime):
        subprocess.check_call(["make", "-s", "-C", str(HERE)])
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        l = C.CDLL(str(LIB))
        for n, (a, r) in _SIG.items():
            f = getattr(l, n)
            f.argtypes = a
            f.restype = r
        _lib = l
    return _lib


def set_threads(n: int) -> None:
    lib().or_set_threads(int(n))


def max_threads() -> int:
    return int(lib().or_max_threads())


def _p(a):
    return None if a is None else a.ctypes.data_as(P)


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _wts(w: O.Weights) -> _W:
    return _W(w.lambda_data, w.lambda_clustering, w.lambda_r_sparsity, w.p, w.lambda_r_consistency,
              w.lambda_monochrome, w.lambda_i_sparsity, w.lambda_smoothness, w.lambda_non_neg, w.lambda_ir,
              w.lambda_cr, w.eps_nonneg, w.eps_irls, 0 if w.chroma_reg == "projection" else 1)


def _cfg(c: O.Config) -> _Cfg:
    return _Cfg(c.outer_iterations, c.gn_steps, c.pcg_iterations, c.max_halvings, int(c.refine),
                c.refine_warmup, c.tol_rel, c.svd_truncation, c.max_delta_b, c.refine_gate_rel)


# -- per-frame auxiliary context ------------------------------------------------

def chromaticity(image):
    """imaging.py:160-171 -> (chroma (H,W,2), dark (H,W))."""
    img = _f64(image)
    H, W = img.shape[:2]
    ch = np.empty((H, W, 2))
    dark = np.empty((H, W), dtype=np.uint8)
    lib().or_chromaticity(H, W, _p(img), _p(ch), _p(dark))
    return ch, dark.astype(bool)


def edge_gate(chroma):
    ch = _f64(chroma)
    H, W = ch.shape[:2]
    out = np.empty((H, W))
    lib().or_edge_gate(H, W, _p(ch), _p(out))
    return out


def sample_pairs(chroma, prev_chroma, seed) -> O.Pairs:
    """energy.py:154-187, bit-exact with numpy's Generator stream."""
    ch = _f64(chroma)
    H, W = ch.shape[:2]
    st = np.random.PCG64(seed).state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    M = 4 * H * W
    src = np.empty(M, dtype=np.int64)
    dst = np.empty(M, dtype=np.int64)
    tmp = np.empty(M, dtype=np.uint8)
    pc = None if prev_chroma is None else _f64(prev_chroma)
    m = 0xFFFFFFFFFFFFFFFF
    n = lib().or_sample_consistency(H, W, _p(ch), _p(pc), s >> 64, s & m, inc >> 64, inc & m, _p(src),
                                    _p(dst), _p(tmp))
    return O.Pairs(src=src[:n].copy(), dst=dst[:n].copy(), temporal=tmp[:n].astype(bool),
                   weight=np.ones(n), shape=(H, W))


def segment(image, colors):
    img = _f64(image)
    cols = _f64(colors)
    H, W = img.shape[:2]
    ids = np.empty((H, W), dtype=np.int32)
    lib().or_segment(H, W, _p(img), cols.shape[0], _p(cols), _p(ids))
    return ids


def initialize(image, cluster_ids, colors, previous=None):
    if previous is not None:
        return previous[0].copy(), previous[1].copy()
    if cluster_ids is None:
        raise ValueError("first frame needs a cluster map")
    img, cols = _f64(image), _f64(colors)
    ids = np.ascontiguousarray(cluster_ids, dtype=np.int32)
    H, W = img.shape[:2]
    K = cols.shape[0]
    r = np.empty((H, W, 3))
    T = np.empty((H, W, K + 1))
    lib().or_initialize(H, W, K, _p(img), _p(ids), _p(cols), _p(r), _p(T))
    return r, T


def build_aux(image, cluster_ids, seed, prev_chroma=None, prev_r=None) -> O.Aux:
    """solver.py:341-351."""
    ch, _ = chromaticity(image)
    return O.Aux(edge=edge_gate(ch), pairs=sample_pairs(ch, prev_chroma, seed), prev_r=prev_r,
                 cluster_ids=cluster_ids)


# -- the frozen system and the solver ----------------------------------------------

class System:
    """The eight terms over one frame (energy.py:478-511) in the C oracle;
    `linearize(r, T)` freezes weights / linearisation like assemble_blocks."""

    def __init__(self, image, colors, aux: O.Aux, wts: O.Weights):
        self.img = _f64(image)
        self.H, self.W = self.img.shape[:2]
        self.colors = _f64(colors).copy()
        self.K = self.colors.shape[0]
        self.N = self.H * self.W
        self.M = self.N * (self.K + 4)
        self.edge = _f64(aux.edge)
        pr = aux.pairs
        self.src = np.ascontiguousarray(pr.src, dtype=np.int64)
        self.dst = np.ascontiguousarray(pr.dst, dtype=np.int64)
        self.tmp = np.ascontiguousarray(pr.temporal, dtype=np.uint8)
        self.pw = _f64(pr.weight)
        self.prev_r = None if aux.prev_r is None else _f64(aux.prev_r)
        self.ids = None if aux.cluster_ids is None else np.ascontiguousarray(aux.cluster_ids, dtype=np.int32)
        self.anchor = None
        if self.ids is None:
            if aux.r_cluster_log is None:
                raise ValueError("aux needs cluster_ids or r_cluster_log")
            self.anchor = _f64(aux.r_cluster_log)
        if np.any(pr.temporal) and aux.prev_r is None:
            raise ValueError("temporal partners need the previous frame's reflectance")
        self._w = _wts(wts)
        self.h = lib().or_sys_create(self.H, self.W, self.K, C.byref(self._w), _p(self.img), _p(self.colors),
                                     _p(self.edge), len(self.src), _p(self.src), _p(self.dst), _p(self.tmp),
                                     _p(self.pw), _p(self.prev_r), _p(self.ids), _p(self.anchor))
        if not self.h:
            raise ValueError("or_sys_create failed")

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_sys_free(self.h)
            self.h = None

    def set_colors(self, colors):
        self.colors = _f64(colors).copy()
        lib().or_sys_set_colors(self.h, _p(self.colors))

    def linearize(self, r, T):
        self.r0, self.T0 = _f64(r), _f64(T)
        lib().or_linearize(self.h, _p(self.r0), _p(self.T0))

    def terms(self, r, T) -> dict:
        out = np.zeros(8)
        r, T = _f64(r), _f64(T)
        if lib().or_terms(self.h, _p(r), _p(T), _p(out)):
            raise ValueError("temporal partners need the previous frame's reflectance")
        return dict(zip(O.TERM_NAMES, out.tolist()))

    def energy(self, r, T) -> float:
        return float(sum(self.terms(r, T).values()))

    def grad_diag(self):
        b = np.empty(self.M)
        d = np.empty(self.M)
        lib().or_grad_diag(self.h, _p(b), _p(d))
        return b, d

    def apply(self, p):
        p = _f64(p)
        out = np.empty(self.M)
        lib().or_apply(self.h, _p(p), _p(out))
        return out

    def pcg(self, b, diag, iterations):
        x = np.empty(self.M)
        info = np.zeros(3)
        lib().or_pcg(self.h, _p(_f64(b)), _p(_f64(diag)), int(iterations), _p(x), _p(info))
        return x, {"iterations": int(info[0]), "initial_residual": float(info[1]),
                   "final_residual": float(info[2])}

    def dense_normal(self, r, T, use_ids=True):
        n = 3 * self.K
        A = np.empty((n, n))
        rhs = np.empty(n)
        lib().or_dense_normal(self.h, _p(_f64(r)), _p(_f64(T)), int(use_ids), _p(A), _p(rhs))
        return A, rhs


def svd_solve(A, rhs, truncation):
    A, rhs = _f64(A), _f64(rhs)
    x = np.empty(rhs.shape[0])
    lib().or_svd_solve(rhs.shape[0], _p(A), _p(rhs), float(truncation), _p(x))
    return x


def record_dict(rec: Rec) -> dict:
    if rec.phase == 1:
        return {"phase": "dense", "energy_before": rec.energy_before, "energy_after": rec.energy_after,
                "accepted": bool(rec.accepted), "alpha": rec.alpha, "delta_b_norm": rec.delta_b_norm}
    return {"phase": "sparse", "energy_before": rec.energy_before, "energy_after": rec.energy_after,
            "accepted": bool(rec.accepted), "alpha": rec.alpha,
            "pcg": {"iterations": rec.pcg_iterations, "initial_residual": rec.initial_residual,
                    "final_residual": rec.final_residual},
            "terms": dict(zip(O.TERM_NAMES, list(rec.terms)))}


def gn_step_sparse(st: O.State, system: System | None = None) -> dict:
    """solver.py:143-192 on an O.State (r, T replaced by the stepped arrays)."""
    sysm = system or System(st.image, st.colors, st.aux, st.weights)
    sysm.set_colors(st.colors)
    r, T = _f64(st.r).copy(), _f64(st.T).copy()
    rec = Rec()
    rc = lib().or_gn_step(sysm.h, _p(r), _p(T), st.config.pcg_iterations, st.config.max_halvings,
                          C.byref(rec))
    if rc == 1:
        raise O.NumericalFault("non-finite residuals in sparse phase",
                               {"iteration": len(st.records), "terms": dict(zip(O.TERM_NAMES, rec.terms))})
    if rc:
        raise ValueError("temporal partners need the previous frame's reflectance")
    st.r, st.T = r, T
    d = record_dict(rec)
    st.records.append(d)
    if d["accepted"]:
        st.energy_history.append(d["energy_after"])
    return d


def flip_flop(st: O.State, system: System | None = None) -> O.State:
    """solver.py:311-338 (with the refine race when config.refine)."""
    sysm = system or System(st.image, st.colors, st.aux, st.weights)
    r, T = _f64(st.r).copy(), _f64(st.T).copy()
    cols = _f64(st.colors).copy()
    cfg = _cfg(st.config)
    cap = st.config.outer_iterations * (st.config.gn_steps + 3) + 8
    recs = (Rec * cap)()
    n, status = C.c_int(), C.c_int()
    rc = lib().or_flip_flop(sysm.h, _p(r), _p(T), _p(cols), C.byref(cfg), recs, cap, C.byref(n),
                            C.byref(status))
    if rc == 1:
        raise O.NumericalFault("non-finite residuals in sparse phase", {"iteration": n.value, "terms": {}})
    if rc:
        raise ValueError("temporal partners need the previous frame's reflectance")
    st.r, st.T, st.colors = r, T, cols
    for i in range(min(n.value, cap)):
        d = record_dict(recs[i])
        st.records.append(d)
        if d["accepted"]:
            st.energy_history.append(d["energy_after"])
    st.status = ("max_outer", "stalled", "converged")[status.value]
    return st


def refine_palette(st: O.State):
    """refine.py:20-40."""
    before = _f64(st.colors).copy()
    st.config = replace(st.config, refine=True)
    flip_flop(st)
    if st.status == "stalled" and not st.energy_history:
        st.colors = before
        return before, np.zeros(before.shape[0])
    return st.colors, np.linalg.norm(st.colors - before, axis=1)


def solve_frame(image, colors, cluster_ids, wts, cfg, seed, previous=None, prev_chroma=None,
                prev_r=None) -> O.State:
    """solver.py:354-363."""
    aux = build_aux(image, cluster_ids, seed, prev_chroma, prev_r)
    r, T = initialize(image, cluster_ids, colors, previous)
    return flip_flop(O.State(image=_f64(image), colors=_f64(colors), r=r, T=T, aux=aux, weights=wts,
                             config=cfg))


def stream_frame(image, colors, prev, prev_image, wts, cfg, seed) -> O.State:
    """One streaming frame of pipeline.py:136-166: segment with the frozen
    palette, aux with temporal partners, warm start, flip_flop (no refine)."""
    ids = segment(image, colors)
    pch, _ = chromaticity(prev_image)
    return solve_frame(image, colors, ids, wts, replace(cfg, refine=False), seed, previous=(prev.r, prev.T),
                       prev_chroma=pch, prev_r=prev.r)


def decompose_clip(frames, colors, ids0, wts, cfg, seed=0, streaming_outer=2):
    """pipeline.py:87-167 with an explicit palette and first-frame ids
    (same contract as lumisplit_oracle.decompose_clip)."""
    colors = _f64(colors)
    aux = build_aux(frames[0], ids0, seed)
    r, T = initialize(frames[0], ids0, colors)
    st = O.State(image=_f64(frames[0]), colors=colors, r=r, T=T, aux=aux, weights=wts, config=cfg)
    if cfg.refine:
        refine_palette(st)
    else:
        st.config = replace(cfg, refine=False)
        flip_flop(st)
    out = [st]
    colors = st.colors
    scfg = replace(cfg, refine=False, outer_iterations=streaming_outer)
    prev = st
    for i in range(1, len(frames)):
        st = stream_frame(frames[i], colors, prev, frames[i - 1], wts, scfg, seed + i)
        out.append(st)
        prev = st
    return out

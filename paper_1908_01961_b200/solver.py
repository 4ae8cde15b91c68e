"""Gauss-Newton solver with sparse-dense splitting (reference solver.py).

Same entry points, dataclasses, record dicts and error behaviour as the
reference; each step runs on the device through the C ABI:

  gn_step_sparse     -> ls_gn_step   (fused energy/gradient kernel,
                        16 x (J^T J apply, PCG update) with device-resident
                        scalars, line-search trial kernels)
  solve_dense_block  -> ls_dense_step (pixel reduction of the 3K x 3K system,
                        on-device Jacobi-SVD solve, clipped line search)

The outer control flow (flip_flop, refine_round) mirrors solver.py:258-338
line for line; it branches on the step records the device returns.
"""

from __future__ import annotations

from dataclasses import dataclass, field, fields, replace
from typing import Callable

import numpy as np
import torch

from . import _device
from . import _lib as L
from .energy import (EnergyAux, EnergyWeights, LayerStack, TERM_NAMES, install,
                     sample_consistency, chroma_edge_weights)
from .imaging import Frame, chromaticity
from .palette import BaseColorPalette, ClusterMap


class NumericalFaultError(RuntimeError):
    """solver.py:24-29: non-finite values; carries an iteration dump."""

    def __init__(self, message: str, dump: dict):
        super().__init__(message)
        self.dump = dump


@dataclass(frozen=True)
class SolveConfig:
    """solver.py:32-63 (same fields and defaults)."""

    outer_iterations: int = 8
    gn_steps: int = 2
    pcg_iterations: int = 16
    tol_rel: float = 1e-4
    max_halvings: int = 4
    refine: bool = True
    svd_truncation: float = 1e-8
    max_delta_b: float = 0.1
    refine_warmup: int = 2
    refine_gate_rel: float = 2e-2

    def with_overrides(self, overrides: dict) -> "SolveConfig":
        known = {f.name for f in fields(self)}
        picked = {}
        for key, value in overrides.items():
            if key not in known:
                continue
            if key in ("tol_rel", "svd_truncation", "max_delta_b", "refine_gate_rel"):
                picked[key] = float(value)
            elif key == "refine":
                picked[key] = str(value).lower() in ("1", "true", "yes")
            else:
                picked[key] = int(value)
        return replace(self, **picked)


@dataclass
class SolverState:
    """solver.py:66-76."""

    frame: Frame
    palette: BaseColorPalette
    layers: LayerStack
    aux: EnergyAux
    weights: EnergyWeights
    config: SolveConfig
    energy_history: list = field(default_factory=list)
    records: list = field(default_factory=list)
    status: str = "running"


def _solver_for(state: SolverState):
    bands = getattr(state.frame, "bands", 0)
    if bands:     # row bands (bands.py): same calls, band-partitioned
        from .bands import BandedSolver, banded_solver
        H, W = state.frame.height, state.frame.width
        s = bands if isinstance(bands, BandedSolver) else banded_solver(
            state.layers.X.device, H, W, state.palette.K, int(bands))
        s.configure(state.weights, state.config)
        s.install(state.frame, state.aux)
        return s
    H, W = state.layers.shape
    s = _device.get_solver(state.layers.X.device, H, W, state.palette.K)
    s.configure(state.weights, state.config)
    install(s, state.frame, state.aux)
    return s


def pcg(apply_A: Callable, b, diag, iterations: int):
    """solver.py:79-107 for an arbitrary operator (numpy or torch vectors).
    The solver's own PCG is the fused device loop inside gn_step_sparse."""
    is_np = not isinstance(b, torch.Tensor)
    bt = torch.as_tensor(np.array(b, dtype=np.float64)) if is_np else b
    dt = torch.as_tensor(np.array(diag, dtype=np.float64)) if is_np else diag
    op = (lambda v: torch.as_tensor(np.asarray(apply_A(v.numpy())))) if is_np else apply_A
    x = torch.zeros_like(bt)
    bn = float(torch.linalg.norm(bt))
    info = {"iterations": 0, "initial_residual": bn, "final_residual": bn}
    if bn == 0.0:
        return (x.numpy() if is_np else x), info
    d = torch.where(dt > 0.0, dt, torch.ones_like(dt))
    r = bt.clone()
    z = r / d
    p = z.clone()
    rz = float(r @ z)
    for it in range(iterations):
        Ap = op(p)
        pAp = float(p @ Ap)
        if pAp <= 0.0 or not np.isfinite(pAp):
            break
        alpha = rz / pAp
        x += alpha * p
        r -= alpha * Ap
        info["iterations"] = it + 1
        rz_new = float(r @ (r / d))
        if rz_new <= 0.0:
            break
        p = r / d + (rz_new / rz) * p
        rz = rz_new
    info["final_residual"] = float(torch.linalg.norm(r))
    return (x.numpy() if is_np else x), info


# streaming flip-flops (refine = False) run device-resident (ls_flip_flop_stream)
DEVICE_FLIP_FLOP = True


def _record_from(rec) -> dict:
    accepted = bool(rec.accepted)
    return {
        "phase": "sparse",
        "energy_before": float(rec.energy_before),
        "energy_after": float(rec.energy_after),
        "accepted": accepted,
        "alpha": float(rec.alpha) if accepted else 0.0,
        "pcg": {"iterations": int(rec.pcg_iterations),
                "initial_residual": float(rec.initial_residual),
                "final_residual": float(rec.final_residual)},
        "terms": {k: float(v) for k, v in zip(TERM_NAMES, rec.terms)},
    }


def gn_step_sparse(state: SolverState) -> dict:
    """solver.py:143-192: one device Gauss-Newton step on the per-pixel unknowns."""
    solver = _solver_for(state)
    X = state.layers.X
    X_out = torch.empty_like(X)
    rc, rec = solver.gn_step(state.palette.colors, X, X_out)
    if rc == L.LS_ERR_NONFINITE:
        terms = {k: float(v) for k, v in zip(TERM_NAMES, rec.terms_before)}
        raise NumericalFaultError("non-finite residuals in sparse phase",
                                  dump={"iteration": len(state.records), "terms": terms})
    accepted = bool(rec.accepted)
    if accepted:
        state.layers = LayerStack(planes=X_out)
    record = _record_from(rec)
    state.records.append(record)
    if accepted:
        state.energy_history.append(record["energy_after"])
    return record


def svd_solve(A, rhs, truncation: float) -> np.ndarray:
    """solver.py:195-204: truncated-SVD minimum-norm solve, one-sided Jacobi
    SVD in fp64 on the device."""
    A = A.detach().cpu().numpy() if isinstance(A, torch.Tensor) else np.asarray(A, dtype=np.float64)
    rhs = rhs.detach().cpu().numpy() if isinstance(rhs, torch.Tensor) else np.asarray(rhs, dtype=np.float64)
    if A.shape[0] > 3 * L.MAX_K:
        raise ValueError(f"svd_solve supports n <= {3 * L.MAX_K}")
    return _device.utility_solver().svd_solve(A, rhs, truncation)


def solve_dense_block(state: SolverState) -> np.ndarray:
    """solver.py:207-255; returns the applied (K, 3) update."""
    K = state.palette.K
    solver = _solver_for(state)
    cols, applied, rec = solver.dense_step(state.palette.colors, state.layers.X)
    if not rec.solved_nonzero:
        return np.zeros((K, 3))
    accepted = bool(rec.accepted)
    if accepted:
        state.palette = replace(state.palette, colors=cols.reshape(K, 3))
    state.records.append({
        "phase": "dense",
        "energy_before": float(rec.energy_before),
        "energy_after": float(rec.energy_after),
        "accepted": accepted,
        "alpha": float(rec.alpha) if accepted else 0.0,
        "delta_b_norm": float(rec.delta_b_norm),
    })
    if accepted:
        state.energy_history.append(float(rec.energy_after))
    return applied.reshape(K, 3)


def _clone_state(state: SolverState) -> SolverState:
    """solver.py:258-263."""
    return SolverState(frame=state.frame, palette=state.palette, layers=state.layers.copy(),
                       aux=state.aux, weights=state.weights, config=state.config,
                       energy_history=list(state.energy_history), records=list(state.records),
                       status=state.status)


def _adopt(state: SolverState, winner: SolverState) -> None:
    """solver.py:266-271."""
    state.palette = winner.palette
    state.layers = winner.layers
    state.energy_history = winner.energy_history
    state.records = winner.records
    state.status = winner.status


def refine_round(state: SolverState) -> bool:
    """solver.py:274-292: plain sparse step vs dense + sparse; lower wins."""
    plain = _clone_state(state)
    gn_step_sparse(plain)
    refined = _clone_state(state)
    solve_dense_block(refined)
    gn_step_sparse(refined)
    e_plain = plain.energy_history[-1] if plain.energy_history else np.inf
    e_refined = refined.energy_history[-1] if refined.energy_history else np.inf
    if e_refined < e_plain:
        _adopt(state, refined)
        return True
    _adopt(state, plain)
    return False


def initialize(frame: Frame, cluster_map: ClusterMap | None, palette: BaseColorPalette,
               previous: LayerStack | None = None) -> LayerStack:
    """solver.py:295-308."""
    if previous is not None:
        return previous.copy()
    if cluster_map is None:
        raise ValueError("first frame needs a cluster map")
    img = frame.data
    H, W = int(img.shape[0]), int(img.shape[1])
    rc = cluster_map.r_cluster.to(device=img.device, dtype=torch.float32)
    cols = torch.as_tensor(palette.colors, dtype=torch.float32, device=img.device)
    ids = cluster_map.ids.to(device=img.device, dtype=torch.int32).contiguous()
    if palette.K >= 1 and torch.equal(rc, cols[(ids - 1).long()]):
        solver = _device.get_solver(img.device, H, W, palette.K)
        solver.set_image(img)
        solver.installed = None
        return LayerStack(planes=solver.initialize(palette.colors, ids))
    # hand-made cluster maps (r_cluster not read off the palette)
    rcd = rc.double()
    X = torch.zeros(palette.K + 4, H, W, dtype=torch.float32, device=img.device)
    X[:3] = torch.log(rcd.clamp_min(1e-4)).permute(2, 0, 1).float()
    ratio = img.double() / rcd.clamp_min(1e-4)
    X[3] = ratio.mean(dim=2).clamp(0.0, 2.0).float()
    return LayerStack(planes=X)


def _flip_flop_device(state: SolverState) -> SolverState:
    """solver.py:311-338 with refine = False, decided on the device (the
    same accept / halve / convergence rules, one host synchronisation)."""
    cfg = state.config
    solver = _solver_for(state)
    rc, recs, status, X_final, fault = solver.flip_flop_stream(
        state.palette.colors, state.layers.X, cfg.outer_iterations, cfg.gn_steps, cfg.tol_rel)
    for i, rec in enumerate(recs):
        if rc == L.LS_ERR_NONFINITE and i == fault:
            state.layers = LayerStack(planes=X_final)
            terms = {k: float(v) for k, v in zip(TERM_NAMES, rec.terms_before)}
            raise NumericalFaultError("non-finite residuals in sparse phase",
                                      dump={"iteration": len(state.records), "terms": terms})
        d = _record_from(rec)
        state.records.append(d)
        if d["accepted"]:
            state.energy_history.append(d["energy_after"])
    state.layers = LayerStack(planes=X_final)
    state.status = ("max_outer", "stalled", "converged")[status]
    return state


def flip_flop(state: SolverState) -> SolverState:
    """solver.py:311-338."""
    cfg = state.config
    if not cfg.refine and DEVICE_FLIP_FLOP:
        return _flip_flop_device(state)
    e_prev = None
    stalled = False
    for outer in range(cfg.outer_iterations):
        sparse_rel = None
        for _ in range(cfg.gn_steps):
            rec = gn_step_sparse(state)
            if not rec["accepted"]:
                stalled = True
            elif rec["energy_before"] > 0.0:
                sparse_rel = (rec["energy_before"] - rec["energy_after"]) / rec["energy_before"]
        settled = sparse_rel is not None and sparse_rel < cfg.refine_gate_rel
        if cfg.refine and outer >= cfg.refine_warmup and (settled or stalled):
            refine_round(state)
        if not state.energy_history:
            continue
        e_now = state.energy_history[-1]
        if e_prev is not None and e_prev > 0.0:
            rel = (e_prev - e_now) / e_prev
            if 0.0 <= rel < cfg.tol_rel:
                state.status = "converged"
                return state
        e_prev = e_now
    state.status = "stalled" if stalled else "max_outer"
    return state


def build_aux(frame: Frame, cluster_map: ClusterMap, seed: int, prev_chroma=None,
              prev_r=None) -> EnergyAux:
    """solver.py:341-351.  The chroma gate and partner draws run on the
    device when the context is first installed (see energy.EnergyAux)."""
    return EnergyAux(prev_r=prev_r, cluster_ids=cluster_map.ids,
                     _recipe=(frame, int(seed), prev_chroma))


def solve_frame(frame: Frame, palette: BaseColorPalette, cluster_map: ClusterMap,
                weights: EnergyWeights, config: SolveConfig, seed: int,
                previous: LayerStack | None = None, prev_chroma=None,
                prev_r=None) -> SolverState:
    """solver.py:354-363."""
    aux = build_aux(frame, cluster_map, seed, prev_chroma, prev_r)
    layers = initialize(frame, cluster_map, palette, previous)
    state = SolverState(frame=frame, palette=palette, layers=layers, aux=aux,
                        weights=weights, config=config)
    return flip_flop(state)

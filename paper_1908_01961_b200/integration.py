"""Drop-in B200 backend for the reference package itself.

`install(lumisplit)` is the maintainer's patch: it swaps the solver seam of
the UNMODIFIED reference -- `flip_flop` (solver.py:311-338), through which
`solve_frame` (solver.py:354-363), `decompose_frames` (pipeline.py:117-156)
and `refine_palette` (refine.py:31) run every Gauss-Newton, PCG, dense and
refine step -- for an adapter that converts the reference's NumPy state to
the device at the seam, runs this package's flip_flop (sm_100a kernels
through the C ABI) and writes the results back into the reference's own
objects (LayerStack arrays, BaseColorPalette, records, energy history,
status).  Everything around the seam (palette estimation, per-frame aux,
corrections, I/O) stays the reference's code.

    import lumisplit
    from paper_1908_01961_b200 import integration
    undo = integration.install(lumisplit)
    res = lumisplit.pipeline.decompose_frames(frames, EnergyWeights(), SolveConfig())
    undo()
"""

from __future__ import annotations

import dataclasses

import numpy as np
import torch

from . import energy as E
from . import solver as S
from .imaging import Frame
from .palette import BaseColorPalette

# the reference modules that bound `flip_flop` by name at import time
_SEAMS = ("solver", "pipeline", "refine")


def _cuda(a, dtype=torch.float32):
    if a is None:
        return None
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).cuda()


def to_device_state(ref_state) -> S.SolverState:
    """The reference's SolverState (NumPy, solver.py:66-76) as this package's
    device state: frame / layers / aux tensors on cuda:0, same weights,
    configuration, records and energy history."""
    aux = ref_state.aux
    smp = aux.samples
    samples = E.ConsistencySamples(src=_cuda(smp.src, torch.int64), dst=_cuda(smp.dst, torch.int64),
                                   temporal=_cuda(smp.temporal, torch.bool),
                                   weight=_cuda(smp.weight, torch.float64), shape=smp.shape)
    dev_aux = E.EnergyAux(edge_weights=_cuda(aux.edge_weights), samples=samples, prev_r=_cuda(aux.prev_r),
                          cluster_ids=_cuda(aux.cluster_ids, torch.int32),
                          r_cluster_log=_cuda(aux.r_cluster_log))
    weights = E.EnergyWeights(**{f.name: getattr(ref_state.weights, f.name)
                                 for f in dataclasses.fields(E.EnergyWeights)})
    config = S.SolveConfig(**{f.name: getattr(ref_state.config, f.name)
                              for f in dataclasses.fields(S.SolveConfig)})
    return S.SolverState(frame=Frame(_cuda(ref_state.frame.data)),
                         palette=BaseColorPalette(colors=np.array(ref_state.palette.colors, dtype=np.float64)),
                         layers=E.LayerStack(_cuda(ref_state.layers.r), _cuda(ref_state.layers.T)),
                         aux=dev_aux, weights=weights, config=config,
                         energy_history=list(ref_state.energy_history), records=list(ref_state.records),
                         status=ref_state.status)


def make_flip_flop(lumisplit):
    """flip_flop with the reference's signature and side effects
    (solver.py:311-338): mutates state.layers / palette / records /
    energy_history / status and returns the state."""
    ref_layer_stack = lumisplit.energy.LayerStack
    ref_palette = lumisplit.palette.BaseColorPalette

    def flip_flop(state):
        dev = to_device_state(state)
        before = np.array(state.palette.colors, dtype=np.float64)
        S.flip_flop(dev)
        torch.cuda.synchronize()
        state.layers = ref_layer_stack(r=dev.layers.r.double().cpu().numpy(),
                                       T=dev.layers.T.double().cpu().numpy())
        cols = np.array(dev.palette.colors, dtype=np.float64)
        if not np.array_equal(cols, before):      # dense steps replace the palette (solver.py:237-243)
            state.palette = ref_palette(colors=cols)
        state.records[:] = dev.records
        state.energy_history[:] = dev.energy_history
        state.status = dev.status
        return state

    flip_flop.__doc__ = "B200 backend of lumisplit.solver.flip_flop (paper_1908_01961_b200.integration)"
    return flip_flop


def install(lumisplit):
    """Point the reference's flip_flop seam at the device solver; returns a
    function that restores the original bindings."""
    import importlib
    mods = [importlib.import_module(f"{lumisplit.__name__}.{m}") for m in _SEAMS]
    saved = [(m, m.flip_flop) for m in mods]
    ff = make_flip_flop(lumisplit)
    for m in mods:
        m.flip_flop = ff

    def uninstall():
        for m, f in saved:
            m.flip_flop = f

    return uninstall

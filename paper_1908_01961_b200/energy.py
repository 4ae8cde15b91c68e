"""Decomposition energy (reference energy.py) on the device.

The reference stacks eight residual-block objects and evaluates them with
NumPy.  `assemble_blocks` returns the same eight blocks (`ResidualBlock`:
residual / apply_j / apply_jt / add_diag per block, device kernels of
csrc/ls_blocks.cu) -- and, on the returned list, the fused operator the
solver actually runs (`FusedEnergy`), whose gradient, Jacobi diagonal and
J^T J products are computed by the sm_100a kernels without ever
materialising the stacked residual F (~61 rows per pixel at K=8): per-term
energies, b = -J^T F, diag(J^T J) and J^T J p are what the solver consumes
(solver.py:110-140), exposed with the reference's names and term keys.
"""

from __future__ import annotations

from dataclasses import dataclass, fields, replace

import numpy as np
import torch

from . import _device
from . import _lib as L
from .imaging import ChromaticityImage, Frame, as_cuda, log_reflectance
from .palette import BaseColorPalette

CONSISTENCY_WINDOW = 15      # energy.py:23-25
CONSISTENCY_SAMPLES = 4
CONSISTENCY_CHROMA_GATE = 0.05
TERM_NAMES = L.TERM_NAMES


@dataclass(frozen=True)
class EnergyWeights:
    """energy.py:28-56 (same fields and defaults)."""

    lambda_data: float = 5000.0
    lambda_clustering: float = 200.0
    lambda_r_sparsity: float = 20.0
    p: float = 1.0
    lambda_r_consistency: float = 10.0
    lambda_monochrome: float = 10.0
    lambda_i_sparsity: float = 3.0
    lambda_smoothness: float = 3.0
    lambda_non_neg: float = 1000.0
    lambda_ir: float = 10.0
    lambda_cr: float = 100.0
    eps_nonneg: float = 0.002
    eps_irls: float = 0.02
    chroma_reg: str = "projection"

    def with_overrides(self, overrides: dict) -> "EnergyWeights":
        known = {f.name for f in fields(self)}
        picked = {k: (v if k == "chroma_reg" else float(v))
                  for k, v in overrides.items() if k in known}
        return replace(self, **picked)


def parse_keyvalue_file(path) -> dict:
    """energy.py:59-71."""
    out = {}
    with open(path) as fh:
        for line in fh:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            if "=" not in line:
                raise ValueError(f"bad config line: {line!r}")
            key, value = line.split("=", 1)
            out[key.strip()] = value.strip()
    return out


class LayerStack:
    """Log-reflectance r plus K+1 transport layers (energy.py:74-94).

    Stored as ONE planar float32 CUDA tensor `X` of shape (K+4, H, W): the
    device layout of include/lumisplit_b200.h.  `r` (H, W, 3) and `T`
    (H, W, K+1) are views with the reference's indexing.
    """

    def __init__(self, r=None, T=None, *, planes: torch.Tensor | None = None):
        if planes is not None:
            self.X = planes
            return
        r_t = as_cuda(r)
        T_t = as_cuda(T, device=r_t.device)
        if r_t.ndim != 3 or r_t.shape[2] != 3 or T_t.ndim != 3 or T_t.shape[:2] != r_t.shape[:2]:
            raise ValueError("expected r (H, W, 3) and T (H, W, K+1)")
        self.X = torch.cat([r_t.permute(2, 0, 1), T_t.permute(2, 0, 1)], 0).contiguous()

    @property
    def r(self) -> torch.Tensor:
        return self.X[:3].permute(1, 2, 0)

    @r.setter
    def r(self, value):
        self.X[:3] = as_cuda(value, device=self.X.device).permute(2, 0, 1)

    @property
    def T(self) -> torch.Tensor:
        return self.X[3:].permute(1, 2, 0)

    @T.setter
    def T(self, value):
        self.X[3:] = as_cuda(value, device=self.X.device).permute(2, 0, 1)

    @property
    def K(self) -> int:
        return int(self.X.shape[0]) - 4

    @property
    def shape(self):
        return int(self.X.shape[1]), int(self.X.shape[2])

    @property
    def reflectance(self) -> torch.Tensor:
        return torch.exp(self.r)

    def illumination(self, palette: BaseColorPalette) -> torch.Tensor:
        B = torch.as_tensor(palette.matrix(), dtype=self.X.dtype, device=self.X.device)
        return torch.einsum("khw,kc->hwc", self.X[3:], B)

    def copy(self) -> "LayerStack":
        if self.X.is_cuda and self.X.is_contiguous():
            return LayerStack(planes=_device.device_copy(torch.empty_like(self.X), self.X))
        return LayerStack(planes=self.X.clone())


def export_reference_layout(layers: LayerStack, out_r: torch.Tensor | None = None,
                            out_T: torch.Tensor | None = None):
    """The reference's arrays of a layer stack -- r (H, W, 3) and T (H, W, K+1),
    interleaved as NumPy C order (energy.py:74-94) -- written on the device by
    one unpack kernel per array (contiguous, ready for a host copy)."""
    X = layers.X
    H, W = layers.shape
    out_r = out_r if out_r is not None else torch.empty((H, W, 3), dtype=torch.float32, device=X.device)
    out_T = out_T if out_T is not None else torch.empty((H, W, layers.K + 1), dtype=torch.float32, device=X.device)
    s = _device.get_solver(X.device, H, W, layers.K)
    s.unpack_hwc(X[:3], out_r)
    s.unpack_hwc(X[3:], out_T)
    return out_r, out_T


def reconstruct(layers: LayerStack, palette: BaseColorPalette) -> torch.Tensor:
    """energy.py:97-99."""
    return layers.reflectance * layers.illumination(palette)


def irls_weight(magnitude, p: float, eps_irls: float):
    """energy.py:102-112 (elementwise helper; the kernels inline it)."""
    tt = isinstance(magnitude, torch.Tensor)
    mag = magnitude.abs().double() if tt else np.abs(np.asarray(magnitude, dtype=np.float64))
    if p >= 2.0:
        return torch.ones_like(mag) if tt else np.ones_like(mag)
    floor = eps_irls ** (1.0 / (2.0 - p))
    big = mag >= floor
    if tt:
        return torch.where(big, mag.clamp_min(floor) ** (p - 2.0), torch.full_like(mag, 1.0 / eps_irls))
    out = np.full_like(mag, 1.0 / eps_irls)
    out[big] = mag[big] ** (p - 2.0)
    return out


def nonneg_weight(T_old, eps_nonneg: float):
    """energy.py:115-118."""
    if isinstance(T_old, torch.Tensor):
        t = T_old.double()
        return torch.where(t > 0.0, torch.zeros_like(t), 1.0 / (t.abs() + eps_nonneg))
    t = np.asarray(T_old, dtype=np.float64)
    return np.where(t > 0.0, 0.0, 1.0 / (np.abs(t) + eps_nonneg))


def chroma_edge_weights(chroma: ChromaticityImage) -> torch.Tensor:
    """energy.py:121-136 on the device."""
    return _device.edge_from_chroma(chroma.planes)


class ConsistencySamples:
    """Gate-surviving partner rows (energy.py:139-151).

    Samples drawn on the device stay in the solver context's adjacency and
    are copied out to (src, dst, temporal, weight) tensors only when those
    attributes are read.
    """

    def __init__(self, src=None, dst=None, temporal=None, weight=None, shape=None):
        self._src, self._dst, self._temporal, self._weight = src, dst, temporal, weight
        self.shape = tuple(shape) if shape is not None else None
        self._solver = None
        self._gen = -1
        self._n = 0
        self._recipe = None     # (frame, seed, prev_chroma): the draws are deterministic

    @classmethod
    def _device_backed(cls, solver, n: int, shape, recipe=None):
        s = cls(shape=shape)
        s._solver, s._gen, s._n, s._recipe = solver, solver.sample_gen, n, recipe
        solver.csr_owner = s
        return s

    def backed_by(self, solver) -> bool:
        return self._solver is solver and self._gen == solver.sample_gen

    def _materialize(self):
        if self._src is not None:
            return
        if self._solver is not None and self._gen == self._solver.sample_gen:
            self._src, self._dst, self._temporal = self._solver.get_pairs(self._n)
        elif self._recipe is not None:
            # the adjacency was rebuilt since: redraw (bit-identical) in a scratch context
            from .imaging import chromaticity
            frame, seed, prev = self._recipe
            again = sample_consistency(chromaticity(frame), prev, seed)
            self._src, self._dst, self._temporal = again.src, again.dst, again.temporal
        else:
            raise RuntimeError("consistency samples were overwritten before being read")
        self._solver = None
        self._n = int(self._src.numel())
        self._weight = torch.ones(self._n, dtype=torch.float64, device=self._src.device)

    def __len__(self):
        if self._src is None and self._n < 0:
            if self._solver is not None and self._gen == self._solver.sample_gen:
                self._n = self._solver.pair_count()
            else:
                self._materialize()
        return self._n if self._src is None else int(self._src.numel())

    @property
    def src(self):
        self._materialize()
        return self._src

    @property
    def dst(self):
        self._materialize()
        return self._dst

    @property
    def temporal(self):
        self._materialize()
        return self._temporal

    @property
    def weight(self):
        self._materialize()
        return self._weight


def _guard_csr(solver):
    """Before the adjacency is rebuilt: device-backed samples that can be
    redrawn (a recipe) are just detached; others are copied out."""
    owner = getattr(solver, "csr_owner", None)
    if owner is not None and owner._src is None and owner.backed_by(solver):
        if owner._recipe is not None:
            owner._solver = None
        else:
            owner._materialize()
    solver.csr_owner = None


def sample_consistency(chroma_t: ChromaticityImage, chroma_prev: ChromaticityImage | None,
                       seed: int) -> ConsistencySamples:
    """energy.py:154-187 on the device, bit-exact (PCG64 + Lemire)."""
    H, W = int(chroma_t.planes.shape[1]), int(chroma_t.planes.shape[2])
    solver = _device.get_solver(chroma_t.planes.device, H, W, 0)
    _guard_csr(solver)
    solver.installed = None
    n = solver.sample(seed, chroma_t.planes,
                      None if chroma_prev is None else chroma_prev.planes)
    s = ConsistencySamples._device_backed(solver, n, (H, W))
    s._materialize()
    return s


class EnergyAux:
    """Per-frame immutable context (energy.py:455-475).

    `build_aux` defers the device work (chroma, edge gate, partner draws)
    until the context is installed into the solver for the frame's palette
    size, so the pipeline draws the partners straight into the adjacency
    the kernels read.
    """

    def __init__(self, edge_weights=None, samples=None, prev_r=None, cluster_ids=None,
                 r_cluster_log=None, *, _recipe=None):
        self._edge = edge_weights
        self._samples = samples
        self.prev_r = prev_r
        self.cluster_ids = cluster_ids
        self.r_cluster_log = r_cluster_log
        self._recipe = _recipe          # (frame, seed, prev_chroma) for deferred draws

    def _realize(self):
        if self._edge is not None and self._samples is not None:
            return
        frame, seed, prev = self._recipe
        from .imaging import chromaticity
        ch = chromaticity(frame)
        if self._edge is None:
            self._edge = chroma_edge_weights(ch)
        if self._samples is None:
            self._samples = sample_consistency(ch, prev, seed)

    @property
    def edge_weights(self):
        self._realize()
        return self._edge

    @property
    def samples(self):
        self._realize()
        return self._samples

    def anchor_log(self, palette: BaseColorPalette):
        if self.cluster_ids is not None:
            cols = torch.as_tensor(palette.colors, dtype=torch.float64,
                                   device=self.cluster_ids.device)
            return log_reflectance(cols[(self.cluster_ids - 1).long()])
        if self.r_cluster_log is None:
            raise ValueError("EnergyAux needs cluster_ids or r_cluster_log")
        return self.r_cluster_log


def install(solver, frame: Frame, aux: EnergyAux):
    """Make (frame, aux) the solver context's per-frame state (no-op if it is)."""
    inst = solver.installed
    if inst is not None and inst[0] is frame and inst[1] is aux:
        return
    img = frame.data
    solver.set_image(img)
    if aux._samples is None and aux._recipe is not None and aux._recipe[0] is frame:
        # deferred draws straight into this context's adjacency
        _guard_csr(solver)
        _, seed, prev = aux._recipe
        n = solver.sample(seed, None, None if prev is None else prev.planes)
        aux._samples = ConsistencySamples._device_backed(solver, n, (solver.H, solver.W),
                                                         recipe=(frame, seed, prev))
        if aux._edge is None:
            aux._edge = solver.get_edge()
    else:
        smp = aux.samples
        if not smp.backed_by(solver):
            _guard_csr(solver)
            solver.set_pairs(smp.src, smp.dst, smp.temporal, smp.weight)
        solver.set_edge(as_cuda(aux.edge_weights, device=img.device))
    if aux.cluster_ids is not None:
        solver.set_anchor(ids=as_cuda(aux.cluster_ids, dtype=torch.int32, device=img.device))
    elif aux.r_cluster_log is not None:
        rcl = as_cuda(aux.r_cluster_log, device=img.device)
        solver.set_anchor(anchor_planes=rcl.permute(2, 0, 1).contiguous())
    else:
        raise ValueError("EnergyAux needs cluster_ids or r_cluster_log")
    if aux.prev_r is not None:
        pr = aux.prev_r
        planes = pr.permute(2, 0, 1) if isinstance(pr, torch.Tensor) else None
        if not (planes is not None and planes.is_cuda and planes.dtype == torch.float32
                and planes.device == img.device and planes.is_contiguous()):
            # (the streaming case passes the previous state's r, a view of its
            # planes: used as it is, no (H, W, 3) round trip)
            planes = as_cuda(pr, device=img.device).permute(2, 0, 1).contiguous()
        solver.set_prev_r(planes)
    else:
        solver.set_prev_r(None)
    solver.installed = (frame, aux)


def to_reference_vector(planes: torch.Tensor) -> torch.Tensor:
    """(U, H, W) planes -> the reference's flat [r.ravel(), T.ravel()]."""
    return torch.cat([planes[:3].permute(1, 2, 0).reshape(-1),
                      planes[3:].permute(1, 2, 0).reshape(-1)])


def from_reference_vector(v, H: int, W: int, K: int, device=None) -> torch.Tensor:
    """Inverse of to_reference_vector."""
    t = as_cuda(v, device=device)
    nr = H * W * 3
    r = t[:nr].reshape(H, W, 3).permute(2, 0, 1)
    T = t[nr:].reshape(H, W, K + 1).permute(2, 0, 1)
    return torch.cat([r, T], 0).contiguous()


class FusedEnergy:
    """All eight terms frozen at `layers` (assemble_blocks, energy.py:478-496)."""

    names = TERM_NAMES

    def __init__(self, frame: Frame, palette: BaseColorPalette, layers: LayerStack,
                 aux: EnergyAux, weights: EnergyWeights):
        self.frame, self.palette, self.aux, self.weights = frame, palette, aux, weights
        self.X = layers.X
        H, W = layers.shape
        self.solver = _device.get_solver(self.X.device, H, W, palette.K)

    def _ready(self):
        from .solver import SolveConfig
        self.solver.configure(self.weights, SolveConfig())
        install(self.solver, self.frame, self.aux)

    def energies(self, r=None, T=None, *, planes: torch.Tensor | None = None) -> dict:
        """block_energies at (r, T) (energy.py:503-504)."""
        self._ready()
        Y = planes if planes is not None else (
            self.X if r is None else LayerStack(r, T).X)
        vals = self.solver.energy_terms(self.palette.colors, self.X, Y)
        return {k: float(v) for k, v in zip(TERM_NAMES, vals)}

    def gradient_and_diag(self):
        """(b = -J^T F, diag(J^T J)) at the linearisation point, planar."""
        self._ready()
        return self.solver.grad_diag(self.palette.colors, self.X)

    def apply_normal(self, p_planes: torch.Tensor) -> torch.Tensor:
        """J^T J p (solver.py:110-122), planar in and out."""
        self._ready()
        return self.solver.apply(self.palette.colors, self.X, as_cuda(p_planes, device=self.X.device))

    def pcg(self, iterations: int):
        self._ready()
        return self.solver.pcg(self.palette.colors, self.X, iterations)


class ResidualBlock:
    """One residual block of the reference's protocol (energy.py:194-452):
    `name`, residual(r, T) -> 1-D rows, apply_j(dr, dT) -> 1-D rows,
    apply_jt(w, out_dr, out_dT) and add_diag(out_dr, out_dT) accumulating in
    place.  The IRLS weights and the linearisation are those of the layers
    the blocks were assembled at.  r / dr / out_dr are (H, W, 3) and T / dT
    / out_dT (H, W, K+1), CUDA tensors or NumPy arrays (the reference's
    tests pass arrays; results come back as the same kind).  Rows are the
    reference's row order (ls_block_* in include/lumisplit_b200.h)."""

    def __init__(self, owner: "FusedEnergy", block_id: int, name: str):
        self._e = owner
        self.block_id = block_id
        self.name = name

    def _pairs(self):
        if self.block_id != L.TERM_NAMES.index("r_consistency"):
            return None
        return self._e._pair_struct()

    def _planes(self, r, T):
        dev = self._e.X.device
        return LayerStack(as_cuda(r, device=dev), as_cuda(T, device=dev)).X

    def residual(self, r, T):
        self._e._ready()
        rows = self._e.solver.block_call("residual", self._e.palette.colors, self._e.X, self.block_id,
                                         self._pairs(), vec=self._planes(r, T))
        return _like(rows, r)

    def apply_j(self, dr, dT):
        self._e._ready()
        rows = self._e.solver.block_call("apply_j", self._e.palette.colors, self._e.X, self.block_id,
                                         self._pairs(), vec=self._planes(dr, dT))
        return _like(rows, dr)

    def _accumulate(self, planes, out_dr, out_dT):
        for out, part in ((out_dr, planes[:3]), (out_dT, planes[3:])):
            upd = part.permute(1, 2, 0)
            if isinstance(out, torch.Tensor):
                out += upd.to(device=out.device, dtype=out.dtype)
            else:
                out += upd.double().cpu().numpy()

    def apply_jt(self, w, out_dr, out_dT):
        self._e._ready()
        acc = torch.zeros_like(self._e.X)
        wv = as_cuda(w, device=self._e.X.device).reshape(-1).float().contiguous()
        self._e.solver.block_call("apply_jt", self._e.palette.colors, self._e.X, self.block_id, self._pairs(),
                                  vec=wv, out=acc)
        self._accumulate(acc, out_dr, out_dT)

    def add_diag(self, out_dr, out_dT):
        self._e._ready()
        acc = torch.zeros_like(self._e.X)
        self._e.solver.block_call("add_diag", self._e.palette.colors, self._e.X, self.block_id, self._pairs(),
                                  out=acc)
        self._accumulate(acc, out_dr, out_dT)

    def __repr__(self):
        return f"ResidualBlock({self.name!r})"


def _like(rows: torch.Tensor, ref):
    return rows if isinstance(ref, torch.Tensor) else rows.double().cpu().numpy()


class EnergyBlocks(list):
    """What assemble_blocks returns: the eight blocks in the reference's
    order (energy.py:478-496, names as `block.name`), and -- as attributes
    -- the fused operator the solver runs (energies, gradient_and_diag,
    apply_normal, pcg of FusedEnergy): the blocks are the reference's
    per-block protocol, the fused kernels the hot path."""

    def __init__(self, fused: "FusedEnergy"):
        super().__init__(ResidualBlock(fused, i, n) for i, n in enumerate(TERM_NAMES))
        self.fused = fused

    def __getattr__(self, name):
        if name == "fused":
            raise AttributeError(name)
        return getattr(self.fused, name)


def _fused_pair_struct(self):
    """ls_pairs of the installed partner rows (device arrays kept alive)."""
    smp = self.aux.samples
    dev = self.X.device
    src = as_cuda(smp.src, dtype=torch.int64, device=dev).contiguous()
    dst = as_cuda(smp.dst, dtype=torch.int64, device=dev).contiguous()
    tmp = as_cuda(smp.temporal, dtype=torch.uint8, device=dev).contiguous()
    wgt = as_cuda(smp.weight, dtype=torch.float64, device=dev).contiguous() if smp.weight is not None else None
    has_t = bool(tmp.any()) if tmp.numel() else False
    if has_t and self.aux.prev_r is None:
        raise ValueError("temporal partners need the previous frame's reflectance")
    self._pair_keep = (src, dst, tmp, wgt)
    return L.Pairs(int(src.numel()), src.data_ptr(), dst.data_ptr(), tmp.data_ptr() if has_t else None,
                   wgt.data_ptr() if wgt is not None else None)


FusedEnergy._pair_struct = _fused_pair_struct


def assemble_blocks(image, palette: BaseColorPalette, layers: LayerStack, aux: EnergyAux,
                    weights: EnergyWeights) -> EnergyBlocks:
    """energy.py:478-496: the eight residual blocks frozen at `layers`."""
    frame = image if isinstance(image, Frame) else _RawFrame(as_cuda(image))
    return EnergyBlocks(FusedEnergy(frame, palette, layers, aux, weights))


def stack_residuals(blocks, r, T):
    """energy.py:499-500: all residual rows, block after block."""
    res = [b.residual(r, T) for b in blocks]
    if res and not isinstance(res[0], torch.Tensor):
        return np.concatenate(res)
    return torch.cat(res)


class _RawFrame:
    """Unvalidated image holder (the reference's tests pass raw 2x2 arrays)."""

    def __init__(self, data):
        self.data = data


def block_energies(blocks, r, T) -> dict:
    """energy.py:503-504 (the fused energy kernel: same per-term values as
    summing each block's squared residual)."""
    return blocks.energies(r, T)


def total_energy(frame: Frame, layers: LayerStack, palette: BaseColorPalette,
                 weights: EnergyWeights, aux: EnergyAux) -> float:
    """energy.py:507-511."""
    e = assemble_blocks(frame, palette, layers, aux, weights).energies()
    return float(sum(e.values()))


def chroma_projections(palette: BaseColorPalette, mode: str) -> np.ndarray:
    """energy.py:518-539."""
    K = palette.K
    mats = np.zeros((K, 3, 3))
    for k in range(K):
        b = palette.colors[k]
        nrm = np.linalg.norm(b)
        if mode == "identity" or nrm < 1e-9:
            mats[k] = np.eye(3)
        else:
            u = b / nrm
            mats[k] = np.eye(3) - np.outer(u, u)
    return mats


def refine_normal_system(image, layers: LayerStack, palette: BaseColorPalette,
                         weights: EnergyWeights, cluster_ids=None):
    """energy.py:563-610: device reduction of the 3K x 3K system at delta_b = 0."""
    img = image.data if hasattr(image, "data") and not isinstance(image, torch.Tensor) else image
    img = as_cuda(img, device=layers.X.device)
    H, W = layers.shape
    solver = _device.get_solver(layers.X.device, H, W, palette.K)
    from .solver import SolveConfig
    solver.configure(weights, SolveConfig())
    solver.installed = None
    solver.set_image(img)
    if cluster_ids is not None:
        solver.set_anchor(ids=as_cuda(cluster_ids, dtype=torch.int32, device=img.device))
    return solver.dense_normal(palette.colors, layers.X, cluster_ids is not None)

"""Layer-aware appearance edits (reference editing.py:24-74) on the device.

All edits are pure: they recombine the converged layers with a modified
palette matrix and return a new (H, W, 3) frame; the per-pixel
recomposition is the `ls_recompose` kernel (fp64 per pixel, like the
reference's float64 numpy).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib as L
from .energy import LayerStack
from .imaging import Frame, as_cuda
from .palette import BaseColorPalette, ClusterMap

_DIV_GUARD = 1e-4      # editing.py:15


def _check_k(k: int, palette: BaseColorPalette) -> None:
    if not 1 <= k <= palette.K:
        raise ValueError(f"cluster id {k} outside 1..{palette.K}")


def _recompose(layers: LayerStack, B: np.ndarray, k: int = 0, ratio=None, ids=None, matte=None,
               background=None) -> torch.Tensor:
    X = layers.X
    if not X.is_cuda:
        raise L.NativeError("layer edits run on the device (CUDA tensors)")
    U, H, W = (int(v) for v in X.shape)
    K = U - 4
    out = torch.empty(H, W, 3, dtype=torch.float32, device=X.device)
    Bh = np.ascontiguousarray(np.asarray(B, dtype=np.float64).reshape(-1))
    rh = None if ratio is None else np.ascontiguousarray(np.asarray(ratio, dtype=np.float64).reshape(3))
    ids_t = None if ids is None else as_cuda(ids, dtype=torch.int32, device=X.device)
    matte_t = None if matte is None else as_cuda(matte, dtype=torch.uint8, device=X.device)
    bg_t = None if background is None else as_cuda(background, device=X.device)
    st = torch.cuda.current_stream(X.device).cuda_stream
    rc = L.load().ls_recompose(L.dptr(X.contiguous()), K, H, W, Bh.ctypes.data_as(L.DBL_P), int(k),
                               None if rh is None else rh.ctypes.data_as(L.DBL_P), L.dptr(ids_t),
                               L.dptr(matte_t), L.dptr(bg_t), L.dptr(out), C.c_void_p(st))
    if rc != L.LS_OK:
        raise (ValueError if rc == L.LS_ERR_ARG else L.NativeError)(L.last_error())
    return out


def recolor(layers: LayerStack, palette: BaseColorPalette, k: int, new_color,
            cluster_map: ClusterMap) -> torch.Tensor:
    """editing.py:24-45: cluster k's reflectance rescaled by new_color / b_k
    and its indirect bounce re-tinted with new_color."""
    _check_k(k, palette)
    new_color = np.asarray(new_color, dtype=np.float64)
    ratio = new_color / np.maximum(palette.colors[k - 1], _DIV_GUARD)
    B = palette.matrix().copy()
    B[k] = new_color
    return _recompose(layers, B, k=k, ratio=ratio, ids=cluster_map.ids)


def suppress_spill(layers: LayerStack, palette: BaseColorPalette, k: int) -> torch.Tensor:
    """editing.py:48-55: reconstruction with cluster k's indirect layer removed."""
    _check_k(k, palette)
    B = palette.matrix().copy()
    B[k] = 0.0
    return _recompose(layers, B)


def rekey_background(layers: LayerStack, palette: BaseColorPalette, k: int, new_background: Frame,
                     matte) -> torch.Tensor:
    """editing.py:58-74: matte pixels take the new background; cluster k's base
    color becomes the background's mean color so its spill re-tints."""
    _check_k(k, palette)
    U, H, W = (int(v) for v in layers.X.shape)
    bg = new_background.data
    if tuple(bg.shape) != (H, W, 3):
        raise ValueError("background dimensions do not match the layers")
    m = torch.as_tensor(np.asarray(matte)) if not isinstance(matte, torch.Tensor) else matte
    if tuple(m.shape) != (H, W):
        raise ValueError("matte dimensions do not match the layers")
    B = palette.matrix().copy()
    B[k] = bg.double().reshape(-1, 3).mean(dim=0).cpu().numpy()
    return _recompose(layers, B, matte=m.bool(), background=bg)

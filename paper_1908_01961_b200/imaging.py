"""Frames, chromaticity and discrete gradients (reference imaging.py).

Frames live on the GPU as (H, W, 3) float32 tensors; chromaticity is
computed by the sm_100a kernel in fp64 (imaging.py:160-171), so its gates
and argmins match the reference bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch

from . import _device

GAMMA = 2.2
DARK_INTENSITY = 0.02      # imaging.py:18-20
LOG_FLOOR = 1e-4           # imaging.py:21-22
MIN_SIZE = 8


class FrameError(ValueError):
    """Bad frame contents (too small, wrong shape) -- imaging.py:26-27."""


class FormatError(ValueError):
    """Unsupported or malformed image file -- imaging.py:30-31."""


def as_cuda(a, dtype=torch.float32, device=None) -> torch.Tensor:
    """numpy / torch -> contiguous CUDA tensor of `dtype` (no copy if already so)."""
    dev = device if device is not None else _device._device_of(a)
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=dev).contiguous()


@dataclass(frozen=True)
class Frame:
    """A linear-light RGB image in [0, 1] (imaging.py:36-57), held on the GPU
    as float32 (inputs are expected to be float32-representable)."""

    data: torch.Tensor  # (H, W, 3) float32, CUDA
    # solve as row bands (bands.py): a band count (all bands in this process)
    # or a bands.BandedSolver (e.g. one band per rank); 0 = whole frame
    bands: object = field(default=0, compare=False, repr=False)

    def __post_init__(self):
        d = self.data
        if d.ndim != 3 or d.shape[2] != 3:
            raise FrameError(f"expected (H, W, 3) array, got {tuple(d.shape)}")
        if d.shape[0] < MIN_SIZE or d.shape[1] < MIN_SIZE:
            raise FrameError(f"frame too small: {d.shape[1]}x{d.shape[0]} (min {MIN_SIZE})")
        t = as_cuda(d)
        if not _device.all_finite(t):
            raise FrameError("frame contains non-finite values")
        object.__setattr__(self, "data", t)

    @property
    def height(self) -> int:
        return int(self.data.shape[0])

    @property
    def width(self) -> int:
        return int(self.data.shape[1])


class ChromaticityImage:
    """(r, g) chroma, channel-sum intensity and dark flag (imaging.py:60-66).
    `planes` is the (2, H, W) fp64 layout the kernels consume; `chroma` is
    the reference's (H, W, 2) view of it.  `intensity` / `dark` are computed
    from the image on first access (the kernels need only the planes)."""

    def __init__(self, planes, intensity=None, dark=None, *, image=None):
        self.planes = planes
        self._intensity, self._dark, self._image = intensity, dark, image

    @property
    def intensity(self) -> torch.Tensor:
        if self._intensity is None:
            self._intensity = self._image.double().sum(dim=2)
        return self._intensity

    @property
    def dark(self) -> torch.Tensor:
        if self._dark is None:
            self._dark = self.intensity < DARK_INTENSITY
        return self._dark

    @property
    def chroma(self) -> torch.Tensor:
        return self.planes.permute(1, 2, 0)


@dataclass(frozen=True)
class GradientField:
    gx: torch.Tensor
    gy: torch.Tensor


def frame_from_array(data) -> Frame:
    """imaging.py:76-78: clamp into [0, 1]."""
    return Frame(as_cuda(data).clamp(0.0, 1.0))


def chromaticity(frame: Frame) -> ChromaticityImage:
    """imaging.py:160-171 on the device (fp64)."""
    img = frame.data if isinstance(frame, Frame) else as_cuda(frame)
    return ChromaticityImage(planes=_device.chromaticity_planes(img), image=img)


def chroma_of_color(color) -> np.ndarray:
    """imaging.py:174-180 (host; palettes are tiny)."""
    color = np.asarray(color, dtype=np.float64)
    total = color.sum(axis=-1, keepdims=True)
    return np.divide(color[..., :2], total, out=np.full_like(color[..., :2], 1.0 / 3.0),
                     where=total > 1e-12)


def log_reflectance(values):
    """imaging.py:183-185."""
    if isinstance(values, torch.Tensor):
        return torch.log(values.clamp_min(LOG_FLOOR))
    return np.log(np.maximum(np.asarray(values, dtype=np.float64), LOG_FLOOR))


def gradient(image: torch.Tensor) -> GradientField:
    """imaging.py:188-195: forward differences, zero on the far edge."""
    gx = torch.zeros_like(image)
    gy = torch.zeros_like(image)
    gx[:, :-1] = image[:, 1:] - image[:, :-1]
    gy[:-1] = image[1:] - image[:-1]
    return GradientField(gx=gx, gy=gy)


# ---- frame I/O (imaging.py:82-157); host-side, outside the solver path ------

def load_pfm(path) -> np.ndarray:
    with open(path, "rb") as fh:
        header = fh.readline().rstrip()
        if header not in (b"PF", b"Pf"):
            raise FormatError(f"not a PFM file: {path}")
        channels = 3 if header == b"PF" else 1
        parts = fh.readline().decode("ascii").split()
        if len(parts) != 2 or not all(p.isdigit() for p in parts):
            raise FormatError(f"malformed PFM dimensions in {path}")
        width, height = int(parts[0]), int(parts[1])
        scale = float(fh.readline().decode("ascii").strip())
        count = width * height * channels
        raw = np.frombuffer(fh.read(count * 4), dtype=("<" if scale < 0 else ">") + "f4")
        if raw.size != count:
            raise FormatError(f"truncated PFM data in {path}")
    shape = (height, width, 3) if channels == 3 else (height, width)
    return np.flipud(raw.reshape(shape)).astype(np.float64)


def save_pfm(path, data) -> None:
    arr = data.detach().cpu().numpy() if isinstance(data, torch.Tensor) else np.asarray(data)
    arr = arr.astype(np.float32)
    if arr.ndim == 3 and arr.shape[2] == 3:
        header = b"PF"
    elif arr.ndim == 2:
        header = b"Pf"
    else:
        raise FormatError(f"cannot write PFM for shape {arr.shape}")
    with open(path, "wb") as fh:
        fh.write(header + b"\n" + f"{arr.shape[1]} {arr.shape[0]}\n".encode() + b"-1.0\n")
        fh.write(np.flipud(arr).astype("<f4").tobytes())


def load_frame(path) -> Frame:
    path = Path(path)
    if not path.exists():
        raise IOError(f"no such file: {path}")
    suffix = path.suffix.lower()
    if suffix == ".png":
        from PIL import Image
        arr = np.asarray(Image.open(path).convert("RGB"), dtype=np.float64) / 255.0
        return frame_from_array((arr ** GAMMA).astype(np.float32))
    if suffix == ".pfm":
        arr = load_pfm(path)
        if arr.ndim == 2:
            arr = np.repeat(arr[:, :, None], 3, axis=2)
        return frame_from_array(arr.astype(np.float32))
    raise FormatError(f"unsupported frame format: {path.suffix!r}")

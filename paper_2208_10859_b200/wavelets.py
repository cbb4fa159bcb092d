"""Public wavelet API of the reference (pkg/src/wavevid/wavelets.py,
exported by wavevid/__init__.py:70): WaveletKind, DimensionError,
CoefficientPyramid, analyze_2d and synthesize_2d.

``synthesize_2d`` of a CDF 9/7 pyramid runs on the B200 through the C ABI
(``wv_synthesize_2d``: the decode's K3 kernels in float32 for every level,
bit-exact with the reference's numpy lifting, wavelets.py:167-182); there is
no CPU path for it.  ``analyze_2d`` (the encoder side) is the package
encoder's torch restatement (encoding.analyze_2d, bit-exact with
wavelets.py:128-149) on the tensor's device.  The Haar kind (used by the
reference only for the temporal transform) is a few elementwise torch ops.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _native as N


class WaveletKind(Enum):
    CDF97 = "cdf97"
    HAAR = "haar"

    @property
    def half_width(self) -> int:
        """Synthesis support half-width in coefficient samples (wavelets.py:30-32)."""
        return 4 if self is WaveletKind.CDF97 else 0


class DimensionError(ValueError):
    """Signal or grid dimensions incompatible with the requested transform."""


@dataclass
class CoefficientPyramid:
    """Multilevel 2-D coefficients of one frame in the in-place Mallat layout
    (wavelets.py:104-125): ``data`` (M, N) or (M, N, C), ``levels`` = l_max."""

    data: np.ndarray
    levels: int

    def __post_init__(self):
        m, n = self.data.shape[:2]
        if self.levels < 1 or (1 << self.levels) > min(m, n):
            raise DimensionError(f"invalid level count {self.levels} for {n}x{m}")
        if m % (1 << self.levels) or n % (1 << self.levels):
            raise DimensionError(f"dimensions {n}x{m} not divisible by 2^{self.levels}")

    @property
    def shape(self):
        return self.data.shape


def _planar(x: np.ndarray) -> torch.Tensor:
    a = np.asarray(x, dtype=np.float32)
    t = torch.from_numpy(np.ascontiguousarray(a if a.ndim == 2 else np.moveaxis(a, -1, 0)))
    return t[None] if a.ndim == 2 else t


def _hwc(t: torch.Tensor, ndim: int) -> np.ndarray:
    a = t.cpu().numpy()
    return a[0] if ndim == 2 else np.ascontiguousarray(np.moveaxis(a, 0, -1))


def _haar_1d(x: torch.Tensor, dim: int, inverse: bool) -> torch.Tensor:
    """Haar along ``dim`` (wavelets.py:55-56 analysis, :77-81 synthesis)."""
    y = x.movedim(dim, -1)
    n = y.shape[-1]
    if inverse:
        s, d = y[..., : n // 2], y[..., n // 2:]
        out = torch.empty_like(y)
        out[..., 0::2] = s + d
        out[..., 1::2] = s - d
    else:
        half = torch.tensor(0.5, dtype=y.dtype, device=y.device)
        e, o = y[..., 0::2], y[..., 1::2]
        out = torch.cat([(e + o) * half, (e - o) * half], -1)
    return out.movedim(-1, dim)


def analyze_2d(frame, levels: int, wavelet: WaveletKind) -> CoefficientPyramid:
    """Recursive separable analysis into a Mallat pyramid, rows then columns
    per level (wavelets.py:128-149); channels transform independently."""
    data = np.array(frame, dtype=np.float32, copy=True)
    CoefficientPyramid(data, levels)   # validates divisibility
    dev = torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")
    x = _planar(data).to(dev)
    if wavelet is WaveletKind.CDF97:
        from .encoding import analyze_2d as _an
        y = _an(x, levels)
    else:
        y = x.clone()
        h, w = y.shape[-2:]
        for _ in range(levels):
            y[..., :h, :w] = _haar_1d(y[..., :h, :w], -1, False)
            y[..., :h, :w] = _haar_1d(y[..., :h, :w], -2, False)
            h, w = h // 2, w // 2
    return CoefficientPyramid(_hwc(y, data.ndim), levels)


def synthesize_2d(pyramid: CoefficientPyramid, wavelet: WaveletKind) -> np.ndarray:
    """Full inverse of analyze_2d (wavelets.py:167-182): float32 (M, N[, C])."""
    data = np.asarray(pyramid.data, dtype=np.float32)
    m, n = data.shape[:2]
    L = pyramid.levels
    if wavelet is WaveletKind.HAAR:
        if not torch.cuda.is_available():
            raise RuntimeError("synthesize_2d runs on the GPU (no CPU fallback)")
        y = _planar(data).cuda()
        for k in range(L, 0, -1):
            h, w = m >> (k - 1), n >> (k - 1)
            y[..., :h, :w] = _haar_1d(y[..., :h, :w], -2, True)
            y[..., :h, :w] = _haar_1d(y[..., :h, :w], -1, True)
        return _hwc(y, data.ndim)
    if not torch.cuda.is_available():
        raise RuntimeError("synthesize_2d runs on the GPU (no CPU fallback)")
    lib = N.load()
    ch = 1 if data.ndim == 2 else data.shape[2]
    # geometry: only width/height/channels/levels matter; 32-px blocks and a
    # 1x1 mask keep the workspace small (m, n are multiples of 2^L)
    bs = 1
    while bs < 32 and m % (bs * 2) == 0 and n % (bs * 2) == 0:
        bs *= 2
    g = N.Geometry(n, m, ch, L, 1, bs, 0, 1, 1)
    nbytes = C.c_uint64()
    N.check(lib.wv_workspace_bytes(C.byref(g), C.byref(nbytes)), "wv_workspace_bytes")
    stream = torch.cuda.current_stream()
    ws = torch.zeros(int(nbytes.value), dtype=torch.uint8, device="cuda")
    pyr = _planar(data).cuda()
    out = torch.empty_like(pyr)
    res = torch.zeros(64, dtype=torch.uint8, device="cuda")
    N.check(lib.wv_synthesize_2d(C.byref(g), C.c_void_p(pyr.data_ptr()),
                                 C.c_void_p(out.data_ptr()), C.c_void_p(ws.data_ptr()),
                                 C.c_void_p(res.data_ptr()), C.c_void_p(stream.cuda_stream)),
            "wv_synthesize_2d")
    return _hwc(out, data.ndim)

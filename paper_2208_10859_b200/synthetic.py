"""Synthetic content, head trajectories and PSNR for benchmarks and tests.

``make_synthetic_clip`` restates the reference generator
(pkg/src/wavevid/bench.py:204-238) for an H x W frame (disc
radii use min(H, W)); for H == W it is byte-identical to the reference
(tests/test_encoder.py checks the digests).  ``make_synthetic_clip_torch``
computes the same content on a device for 8K inputs (float64 on the GPU;
a libm/CUDA ulp difference can move a rare pixel by one level, which only
changes the synthetic input, never a parity comparison).
"""
from __future__ import annotations

import math

import numpy as np
import torch

PSNR_CAP = 99.0


def _params(channels: int, seed: int):
    rng = np.random.default_rng(seed)
    phases = rng.uniform(0, 2 * np.pi, size=(channels, 2))
    pos = rng.uniform(0.2, 0.8, size=(3, 2))
    vel = rng.uniform(-0.01, 0.01, size=(3, 2))
    col = rng.integers(60, 255, size=(3, channels))
    return phases, pos, vel, col


def make_synthetic_clip(frames: int = 16, size: int = 512, channels: int = 3,
                        seed: int = 7, height: int | None = None,
                        width: int | None = None) -> np.ndarray:
    """(F, H, W, C) uint8 drifting gradients plus three moving discs."""
    h = size if height is None else height
    w = size if width is None else width
    phases, pos, vel, col = _params(channels, seed)
    yy = np.linspace(0, 2 * np.pi, h, endpoint=False)[:, None]
    xx = np.linspace(0, 2 * np.pi, w, endpoint=False)[None, :]
    ry = np.arange(h)[:, None]
    rx = np.arange(w)[None, :]
    scale = min(h, w)
    out = np.empty((frames, h, w, channels), np.uint8)
    for f in range(frames):
        drift = 2 * np.pi * f / max(frames, 1) * 0.1
        img = np.empty((h, w, channels), np.float64)
        for c in range(channels):
            img[..., c] = (0.5 + 0.25 * np.sin(yy + phases[c, 0] + drift)
                           + 0.25 * np.cos(xx + phases[c, 1] - drift))
        img = np.clip(img, 0, 1) * 255.0
        for i in range(3):
            cy, cx = (pos[i] + f * vel[i]) % 1.0
            r = scale * (0.05 + 0.02 * i)
            dy = ry - cy * h
            dx = rx - cx * w
            img[dy * dy + dx * dx < r * r] = col[i]
        out[f] = np.clip(np.rint(img), 0, 255).astype(np.uint8)
    return out


def make_synthetic_clip_torch(frames: int, height: int, width: int,
                              channels: int = 3, seed: int = 7,
                              device="cuda", first_frame: int = 0,
                              total_frames: int | None = None) -> torch.Tensor:
    """Device version: frames [first_frame, first_frame+frames) of a clip of
    ``total_frames`` (drift depends on the clip length), (F, H, W, C) u8."""
    tot = frames if total_frames is None else total_frames
    phases, pos, vel, col = _params(channels, seed)
    d = torch.device(device)
    f64 = torch.float64
    yy = (torch.arange(height, device=d, dtype=f64) * (2 * math.pi / height))[:, None]
    xx = (torch.arange(width, device=d, dtype=f64) * (2 * math.pi / width))[None, :]
    ry = torch.arange(height, device=d, dtype=f64)[:, None]
    rx = torch.arange(width, device=d, dtype=f64)[None, :]
    scale = min(height, width)
    out = torch.empty((frames, height, width, channels), dtype=torch.uint8, device=d)
    for j in range(frames):
        f = first_frame + j
        drift = 2 * math.pi * f / max(tot, 1) * 0.1
        for c in range(channels):
            img = (0.5 + 0.25 * torch.sin(yy + (phases[c, 0] + drift))
                   + 0.25 * torch.cos(xx + (phases[c, 1] - drift)))
            img = img.clamp(0, 1) * 255.0
            for i in range(3):
                cy, cx = (pos[i] + f * vel[i]) % 1.0
                r = scale * (0.05 + 0.02 * i)
                inside = (ry - cy * height) ** 2 + (rx - cx * width) ** 2 < r * r
                img = torch.where(inside, torch.tensor(float(col[i, c]), dtype=f64, device=d), img)
            out[j, :, :, c] = torch.round(img).clamp(0, 255).to(torch.uint8)
    return out


def psnr(a, b) -> float:
    """PSNR over 8-bit data, capped at 99 dB (bench.py:22-30)."""
    if isinstance(a, torch.Tensor):
        mse = ((a.to(torch.float64) - b.to(torch.float64)) ** 2).mean().item()
    else:
        if a.shape != b.shape:
            raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
        mse = float(np.mean((a.astype(np.float64) - b.astype(np.float64)) ** 2))
    if mse == 0:
        return PSNR_CAP
    return min(PSNR_CAP, 10.0 * math.log10(255.0 ** 2 / mse))

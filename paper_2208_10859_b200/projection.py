"""Sphere geometry (host) and the perspective writeout (K4, device).

Host side (pose -> low-res viewport mask) stays on the CPU exactly as in the
reference (<10 ms, input to the tile-selection kernel):
pkg/src/wavevid/projection.py:24-108, :175-179.  ``render_perspective`` keeps
the reference signature (projection.py:111) but runs the K4 kernel.
"""
from __future__ import annotations

import ctypes as C
import functools
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N


class ProjectionError(ValueError):
    pass


class CoverageError(ProjectionError):
    """Perspective sampling hit a pixel outside the decoded footprint."""


@dataclass
class CameraPose:
    """Yaw about y, then pitch about x, then roll about z (degrees)."""

    yaw: float = 0.0
    pitch: float = 0.0
    roll: float = 0.0
    fov_h: float = 90.0
    fov_v: float = 90.0

    def __post_init__(self):
        if not 0 < self.fov_h <= 360:
            raise ProjectionError(f"fov_h {self.fov_h} outside (0, 360]")
        if not 0 < self.fov_v <= 180:
            raise ProjectionError(f"fov_v {self.fov_v} outside (0, 180]")
        if not -90 <= self.pitch <= 90:
            raise ProjectionError(f"pitch {self.pitch} outside [-90, 90]")

    def rotation(self) -> np.ndarray:
        """World-from-camera rotation Ry @ Rx @ Rz (projection.py:39-52)."""
        y, p, r = (math.radians(v) for v in (self.yaw, self.pitch, self.roll))
        cy, sy, cp, sp, cr, sr = (math.cos(y), math.sin(y), math.cos(p), math.sin(p),
                                  math.cos(r), math.sin(r))
        ry = np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]])
        rx = np.array([[1, 0, 0], [0, cp, sp], [0, -sp, cp]])
        rz = np.array([[cr, -sr, 0], [sr, cr, 0], [0, 0, 1]])
        return ry @ rx @ rz


def mapping_factor(y: int, s_y: int) -> float:
    return 1.0 - math.sin(y * math.pi / s_y)


def lonlat_to_dir(lon, lat) -> np.ndarray:
    lon, lat = np.broadcast_arrays(lon, lat)
    cl = np.cos(lat)
    return np.stack([np.sin(lon) * cl, np.sin(lat), np.cos(lon) * cl], axis=-1)


def direction_of_pixel(x, y, dims) -> np.ndarray:
    n, m = dims
    lon = np.radians((np.asarray(x, dtype=np.float64) + 0.5) / n * 360.0 - 180.0)
    lat = np.radians(90.0 - (np.asarray(y, dtype=np.float64) + 0.5) / m * 180.0)
    return lonlat_to_dir(lon, lat)


def _dilate2_wrapped(a: np.ndarray) -> np.ndarray:
    """2-cell square dilation; columns wrap (longitude), rows clamp."""
    h, w = a.shape
    ext = np.concatenate([a[:, -2:], a, a[:, :2]], axis=1)
    out = ext.copy()
    for axis in (0, 1):
        src = out.copy()
        n = src.shape[axis]
        for r in (1, 2):
            if axis == 0:
                out[r:] |= src[:n - r]
                out[:n - r] |= src[r:]
            else:
                out[:, r:] |= src[:, :n - r]
                out[:, :n - r] |= src[:, r:]
    return out[:, 2:2 + w]


def viewport_to_mask(pose: CameraPose, dims) -> np.ndarray:
    """(mask_h, mask_w) cells whose centre direction is inside the pose's
    frustum, dilated two cells with longitude wrap (projection.py:83-108)."""
    mask_w, mask_h = dims
    dirs = direction_of_pixel(np.arange(mask_w)[None, :], np.arange(mask_h)[:, None],
                              (mask_w, mask_h))
    # roll within the dilation margin is absorbed by the 2-cell dilation
    if abs(pose.roll) > 15:
        cam_from_world = pose.rotation().T
    else:
        cam_from_world = CameraPose(pose.yaw, pose.pitch, 0.0, pose.fov_h,
                                    pose.fov_v).rotation().T
    cam = dirs @ cam_from_world.T
    x, y, z = cam[..., 0], cam[..., 1], cam[..., 2]
    lon = np.degrees(np.arctan2(x, z))
    lat = np.degrees(np.arctan2(y, np.hypot(x, z)))
    inside = (np.abs(lon) <= pose.fov_h / 2.0 + 1e-9) & (np.abs(lat) <= pose.fov_v / 2.0 + 1e-9)
    return _dilate2_wrapped(inside)


def stereo_mask(pose: CameraPose, dims) -> np.ndarray:
    """Top-bottom stereo: the eye mask stacked twice (projection.py:175-179)."""
    mask_w, mask_h = dims
    eye = viewport_to_mask(pose, (mask_w, mask_h // 2))
    return np.concatenate([eye, eye], axis=0)


# --------------------------------------------------------------- K4 (device)

def view_args(canvas: torch.Tensor, footprint_bits: torch.Tensor, row0: int, rows: int,
              width: int, channels: int, pose: CameraPose, out: torch.Tensor,
              uncovered: torch.Tensor) -> N.ViewArgs:
    """K4 arguments for one view of a planar (C, H, W) u8 canvas."""
    if not (pose.fov_h < 180 and pose.fov_v < 180):
        raise ProjectionError("perspective rendering requires FOV < 180 degrees")
    v = N.ViewArgs()
    v.d_canvas = canvas.data_ptr()
    v.d_footprint = footprint_bits.data_ptr()
    v.row0, v.rows, v.width, v.channels = row0, rows, width, channels
    v.canvas_h = int(canvas.shape[-2])
    rot = pose.rotation().reshape(-1)
    for i in range(9):
        v.rot[i] = float(rot[i])
    v.tan_h = math.tan(math.radians(pose.fov_h / 2.0))
    v.tan_v = math.tan(math.radians(pose.fov_v / 2.0))
    v.out_h, v.out_w = int(out.shape[0]), int(out.shape[1])
    v.d_out = out.data_ptr()
    v.d_uncovered = uncovered.data_ptr()
    return v


@functools.lru_cache(maxsize=4096)
def _pose_consts(yaw, pitch, roll, fov_h, fov_v):
    """Rotation (row major, the numpy product the reference forms) and FOV
    tangents of a pose; cached, since a viewer revisits poses."""
    rot = CameraPose(yaw, pitch, roll, fov_h, fov_v).rotation().reshape(-1).tolist()
    return rot, math.tan(math.radians(fov_h / 2.0)), math.tan(math.radians(fov_v / 2.0))


def set_view_pose(views: list, pose: CameraPose) -> None:
    """Re-point cached K4 arguments at a new pose (one rotation for all views)."""
    if not (pose.fov_h < 180 and pose.fov_v < 180):
        raise ProjectionError("perspective rendering requires FOV < 180 degrees")
    rot, tan_h, tan_v = _pose_consts(float(pose.yaw), float(pose.pitch), float(pose.roll),
                                     float(pose.fov_h), float(pose.fov_v))
    for v in views:
        v.rot[:] = rot
        v.tan_h, v.tan_v = tan_h, tan_v


def launch_views(views: list, stream: torch.cuda.Stream | None = None) -> None:
    lib = N.load()
    arr = (N.ViewArgs * len(views))(*views)
    s = stream if stream is not None else torch.cuda.current_stream()
    N.check(lib.wv_render_perspective(arr, len(views), C.c_void_p(s.cuda_stream)),
            "wv_render_perspective")


def pack_footprint(fp: np.ndarray) -> np.ndarray:
    """bool (H, W) -> (H, ceil(W/32)) int32 bit rows (bit i = column 32w+i)."""
    h, w = fp.shape
    wp = (w + 31) // 32
    padded = np.zeros((h, wp * 32), bool)
    padded[:, :w] = fp
    return np.packbits(padded, axis=1, bitorder="little").view(np.int32).reshape(h, wp)


def unpack_footprint(bits: np.ndarray, width: int) -> np.ndarray:
    b = np.ascontiguousarray(bits).view(np.uint8)
    return np.unpackbits(b, axis=1, bitorder="little")[:, :width].astype(bool)


def render_perspective(region: np.ndarray, footprint: np.ndarray, pose: CameraPose,
                       out_dims, device=None) -> np.ndarray:
    """Reference-compatible entry (projection.py:111-172) running K4 on the
    GPU: numpy in, numpy out, CoverageError on any uncovered tap."""
    out_w, out_h = out_dims
    if not (pose.fov_h < 180 and pose.fov_v < 180):
        raise ProjectionError("perspective rendering requires FOV < 180 degrees")
    dev = torch.device(device) if device is not None else torch.device("cuda")
    mono = region.ndim == 2
    reg = region[..., None] if mono else region
    m, n, c = reg.shape
    canvas = torch.from_numpy(np.ascontiguousarray(reg, np.uint8)).to(dev).permute(2, 0, 1).contiguous()
    fpb = torch.from_numpy(pack_footprint(np.asarray(footprint, bool))).to(dev)
    out = torch.empty((out_h, out_w, c), dtype=torch.uint8, device=dev)
    unc = torch.zeros(1, dtype=torch.int32, device=dev)
    launch_views([view_args(canvas, fpb, 0, m, n, c, pose, out, unc)])
    missing = int(unc.item())
    if missing:
        raise CoverageError(f"{missing} output pixels sample outside the footprint")
    res = out.cpu().numpy()
    return res[..., 0] if mono else res

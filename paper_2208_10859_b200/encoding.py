"""Encoder: the reference's encode_video (pkg/src/wavevid/encoding.py:36-425).

On a CUDA device each inter-frame set goes through the CUDA encoder
(``wv_encode_set``, csrc/wv_encode.cu).  The torch restatement below runs
the reference op for op in float32 with float32-rounded constants and no
fused multiply-adds; it is the CPU path (and ``backend="torch"``).  Both
reproduce the reference's files byte for byte: the golden sha256 digests
are checked in tests/test_host.py (CPU) and tests/test_gpu_encoder.py
(CUDA).  This is the mirror path of the product, not
the decode hot path.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

_F = torch.float32
# CDF 9/7 lifting constants (wavelets.py:16-22) as float32 multipliers
_ALPHA = -1.586134342059924
_BETA = -0.052980118572961
_GAMMA = 0.882911075530934
_DELTA = 0.443506852043971
_K = 1.230174104914001


class MappingKind(Enum):
    NONE = "none"
    EQUIRECTANGULAR = "equirectangular"


class EncodeError(ValueError):
    pass


def default_levels(width: int, height: int) -> int:
    """log2(N/32) - 2 clamped to [1, log2(min dims)] (encoding.py:36-39)."""
    raw = int(math.log2(max(width, 32) / 32)) - 2
    return max(1, min(raw, int(math.log2(min(width, height)))))


@dataclass
class EncodeParams:
    """Same fields and validation as encoding.py:52-83."""

    alpha: float = 0.1
    inter_threshold: float = 0.005
    levels: int | None = None
    inter_size: int = 4
    block_size: int = 32
    mapping: MappingKind = MappingKind.EQUIRECTANGULAR
    quantize: bool = True
    stereo: bool = False
    fps: float = 30.0
    mask_w: int = 64
    mask_h: int = 64

    def __post_init__(self):
        if self.alpha < 0 or self.inter_threshold < 0:
            raise EncodeError("thresholds must be >= 0")
        n = self.inter_size
        if n < 1 or n & (n - 1):
            raise EncodeError(f"inter_size must be a power of two >= 1, got {n}")
        if self.block_size < 1 or self.block_size & (self.block_size - 1):
            raise EncodeError("block_size must be a power of two")

    def resolved_levels(self, width: int, height: int) -> int:
        lv = self.levels if self.levels is not None else default_levels(width, height)
        if lv < 1:
            raise EncodeError("levels must be >= 1")
        if width % (1 << lv) or height % (1 << lv):
            raise EncodeError(f"{width}x{height} not divisible by 2^{lv}")
        if width % self.block_size or height % self.block_size:
            raise EncodeError("block_size must divide frame dimensions")
        return lv


def threshold_value(alpha: float, level: int, l_max: int, h: float = 0.0) -> float:
    """alpha * ((l_max - level) / l_max)^2 + h (encoding.py:86-98)."""
    if l_max < 1:
        raise EncodeError("l_max must be >= 1")
    if not 0 <= level <= l_max:
        raise EncodeError(f"level {level} outside [0, {l_max}]")
    if h < 0:
        raise EncodeError("mapping factor must be >= 0")
    return alpha * ((l_max - level) / l_max) ** 2 + h


def temporal_level_of(t_idx: int, n: int) -> int:
    return int(math.log2(n)) - int(math.floor(math.log2(t_idx)))


def temporal_sign(t: int, level: int) -> int:
    return 1 if ((t >> (level - 1)) & 1) == 0 else -1


def equirect_mapping_factors(height: int) -> np.ndarray:
    """H(y) = 1 - sin(y*pi/S_y) in float32 (encoding.py:359-362).  Kept in
    numpy on the host so CPU and GPU encodes share the exact table."""
    y = np.arange(height, dtype=np.float32)
    return 1.0 - np.sin(y * np.pi / height).astype(np.float32)


# -- lifting ---------------------------------------------------------------

def _c(v: float, like: torch.Tensor) -> torch.Tensor:
    return torch.tensor(v, dtype=_F, device=like.device)


def _even_odd(x: torch.Tensor, dim: int):
    idx = [slice(None)] * x.dim()
    idx[dim] = slice(0, None, 2)
    e = x[tuple(idx)]
    idx[dim] = slice(1, None, 2)
    return e.clone(), x[tuple(idx)].clone()


def _shift(x: torch.Tensor, dim: int, step: int) -> torch.Tensor:
    """x[i+1] (step=+1) or x[i-1] (step=-1) along dim, edge-clamped."""
    n = x.shape[dim]
    if step > 0:
        return torch.cat([x.narrow(dim, 1, n - 1), x.narrow(dim, n - 1, 1)], dim)
    return torch.cat([x.narrow(dim, 0, 1), x.narrow(dim, 0, n - 1)], dim)


def _analyze(x: torch.Tensor, dim: int):
    """One CDF 9/7 analysis pass along ``dim`` (wavelets.py:44-65)."""
    s, d = _even_odd(x, dim)
    d = d + _c(_ALPHA, x) * (s + _shift(s, dim, 1))
    s = s + _c(_BETA, x) * (_shift(d, dim, -1) + d)
    d = d + _c(_GAMMA, x) * (s + _shift(s, dim, 1))
    s = s + _c(_DELTA, x) * (_shift(d, dim, -1) + d)
    s = s * _c(1.0 / _K, x)
    d = d * _c(_K, x)
    return s, d


def analyze_2d(frames: torch.Tensor, levels: int) -> torch.Tensor:
    """Mallat pyramid of (..., H, W) float32 frames, rows then columns per
    level (wavelets.py:128-149)."""
    data = frames.to(_F).clone()
    h, w = data.shape[-2:]
    for _ in range(levels):
        a, d = _analyze(data[..., :h, :w], -1)
        data[..., :h, :w] = torch.cat([a, d], -1)
        a, d = _analyze(data[..., :h, :w], -2)
        data[..., :h, :w] = torch.cat([a, d], -2)
        h //= 2
        w //= 2
    return data


# -- thresholding / temporal / quantization ---------------------------------

def _threshold_grid(h: int, w: int, levels: int, alpha: float, hfac: np.ndarray,
                    device) -> torch.Tensor:
    """Spatial threshold per position; -inf in the approximation band
    (encoding.py:101-115)."""
    t = torch.empty((h, w), dtype=_F, device=device)
    hf = torch.as_tensor(np.asarray(hfac, np.float32), device=device)
    for k in range(1, levels + 1):
        base = torch.tensor(threshold_value(alpha, k - 1, levels), dtype=_F, device=device)
        hh, hw = h >> k, w >> k
        rows = hf[(torch.arange(hh, device=device) << k).clamp(0, h - 1)]
        col = (base + rows)[:, None]
        t[:hh, hw:2 * hw] = col
        t[hh:2 * hh, :2 * hw] = col
    t[: h >> levels, : w >> levels] = -math.inf
    return t


def _haar_forward(stack: torch.Tensor) -> torch.Tensor:
    """Full temporal Haar along dim 0 in Mallat order (encoding.py:153-169)."""
    n = stack.shape[0]
    out = torch.empty_like(stack)
    cur, end = stack, n
    half_c = _c(0.5, stack)
    while cur.shape[0] > 1:
        a = (cur[0::2] + cur[1::2]) * half_c
        d = (cur[0::2] - cur[1::2]) * half_c
        half = cur.shape[0] // 2
        out[end - half:end] = d
        end -= half
        cur = a
    out[0] = cur[0]
    return out


def _layer_grid(h: int, w: int, levels: int, device) -> torch.Tensor:
    """Storage layer per position: 0 approx, then coarse->fine
    (wavelets.py:202-211)."""
    g = torch.zeros((h, w), dtype=torch.int64, device=device)
    for k in range(1, levels + 1):
        layer = levels - k + 1
        hh, hw = h >> k, w >> k
        g[:hh, hw:2 * hw] = torch.clamp(g[:hh, hw:2 * hw], min=layer)
        g[hh:2 * hh, :2 * hw] = torch.clamp(g[hh:2 * hh, :2 * hw], min=layer)
    return g


@dataclass
class SparseCoefficients:
    """Records of one set in storage order (encoding.py:274-293).  The torch
    encoder also keeps ``packed`` (the on-disk record bytes) and ``counts``
    (records per (t, block)) so files are written without re-deriving them."""

    temporal: np.ndarray
    block: np.ndarray
    offset: np.ndarray
    values: np.ndarray
    packed: bytes | None = None
    counts: np.ndarray | None = None

    def __len__(self) -> int:
        return len(self.offset)

    @property
    def float_mode(self) -> bool:
        return self.values.dtype != np.uint8


@dataclass
class EncodedSet:
    records: SparseCoefficients
    extrema: np.ndarray  # (n, C, 4) float32


@dataclass
class EncodedVideo:
    width: int
    height: int
    frame_count: int
    fps: float
    channels: int
    levels: int
    inter_size: int
    block_size: int
    mask_w: int
    mask_h: int
    pad_frames: int
    float_mode: bool
    stereo: bool
    sets: list = field(default_factory=list)


def _encode_set(frames: torch.Tensor, p: EncodeParams, levels: int,
                hfac: np.ndarray, keep_arrays: bool) -> EncodedSet:
    """frames: (n, C, H, W) float32 in [0, 1] -> one encoded set
    (encoding.py:365-374 + quantize :296-332)."""
    n, c, h, w = frames.shape
    dev = frames.device
    pyr = analyze_2d(frames, levels)                           # (n, C, H, W)
    # sparsify (encoding.py:118-135): per-position channel max magnitude
    t_grid = _threshold_grid(h, w, levels, p.alpha, hfac, dev)
    keep = pyr.abs().amax(dim=1) > t_grid                       # (n, H, W)
    pyr = torch.where(keep[:, None], pyr, torch.zeros((), dtype=_F, device=dev))
    # temporal transform + threshold (encoding.py:198-236)
    data = _haar_forward(pyr)
    ah, aw = h >> levels, w >> levels
    if n > 1:
        big = int(math.log2(n))
        for ti in range(1, n):
            thr = threshold_value(p.inter_threshold, temporal_level_of(ti, n) - 1, big)
            kill = data[ti].abs().amax(dim=0) <= torch.tensor(thr, dtype=_F, device=dev)
            kill[:ah, :aw] = False
            data[ti] = torch.where(kill[None], torch.zeros((), dtype=_F, device=dev), data[ti])
    # extrema (encoding.py:239-254)
    ext = torch.zeros((n, c, 4), dtype=_F, device=dev)
    appr = data[:, :, :ah, :aw]
    ext[:, :, 0] = appr.amin(dim=(2, 3))
    ext[:, :, 1] = appr.amax(dim=(2, 3))
    dmask = torch.ones((h, w), dtype=torch.bool, device=dev)
    dmask[:ah, :aw] = False
    det = data[:, :, dmask]                                     # (n, C, P)
    ext[:, :, 2] = det.amin(dim=2)
    ext[:, :, 3] = det.amax(dim=2)
    # records (encoding.py:296-332)
    bs = p.block_size
    nbx, nb = w // bs, (w // bs) * (h // bs)
    nz = (data != 0).any(dim=1)                                 # (n, H, W)
    ti, ys, xs = torch.nonzero(nz, as_tuple=True)
    block = (ys // bs) * nbx + (xs // bs)
    offset = (ys % bs) * bs + (xs % bs)
    layer = _layer_grid(h, w, levels, dev)[ys, xs]
    key = ((ti * nb + block) * (levels + 1) + layer) * (bs * bs) + offset
    order = torch.argsort(key)
    ti, ys, xs, block, offset = ti[order], ys[order], xs[order], block[order], offset[order]
    vals = data[ti, :, ys, xs]                                  # (R, C)
    if not p.quantize:
        values = vals.contiguous()
        vbytes = values.view(torch.uint8).reshape(-1, 4 * c)
    else:
        in_appr = ((ys < ah) & (xs < aw))[:, None]
        e = ext[ti]                                             # (R, C, 4)
        lo = torch.where(in_appr, e[:, :, 0], e[:, :, 2])
        hi = torch.where(in_appr, e[:, :, 1], e[:, :, 3])
        span = hi - lo
        one = torch.ones((), dtype=_F, device=dev)
        safe = torch.where(span > 0, span, one)
        cd = torch.floor((vals - lo) / safe * _c(255.0, vals) + _c(0.5, vals))
        cd = torch.where(span > 0, cd, torch.zeros((), dtype=_F, device=dev))
        values = cd.clamp(0, 255).to(torch.uint8)
        vbytes = values
    off16 = offset.to(torch.int32)
    obytes = torch.stack([(off16 & 0xFF), (off16 >> 8) & 0xFF], 1).to(torch.uint8)
    packed = torch.cat([obytes, vbytes], 1).contiguous().cpu().numpy().tobytes()
    counts = torch.bincount(ti * nb + block, minlength=n * nb).reshape(n, nb)
    rec = SparseCoefficients(
        temporal=ti.to(torch.uint8).cpu().numpy() if keep_arrays else np.zeros(0, np.uint8),
        block=block.to(torch.int64).cpu().numpy().astype(np.uint32) if keep_arrays else np.zeros(0, np.uint32),
        offset=offset.cpu().numpy().astype(np.uint16) if keep_arrays else np.zeros(len(offset), np.uint16),
        values=values.cpu().numpy() if keep_arrays else np.zeros((0, c), np.float32 if not p.quantize else np.uint8),
        packed=packed, counts=counts.cpu().numpy())
    if not keep_arrays:
        rec.offset = np.zeros(len(offset), np.uint16)
    return EncodedSet(records=rec, extrema=ext.cpu().numpy())


def _encode_set_native(chunk: torch.Tensor, p: EncodeParams, levels: int, hfac: np.ndarray,
                       keep_arrays: bool) -> EncodedSet:
    """One set through the CUDA encoder (wv_encode_set, csrc/wv_encode.cu):
    (n, H, W, C) u8 on the device -> packed records, counts, extrema."""
    import ctypes as C
    from . import _native as nat
    lib = nat.load()
    n, h, w, c = chunk.shape
    dev = chunk.device
    ep = nat.EncodeParams()
    ep.width, ep.height, ep.channels, ep.levels = w, h, c, levels
    ep.inter_size, ep.block_size, ep.quantize = n, p.block_size, int(p.quantize)
    if n > nat.WV_ENC_MAX_N or levels > nat.WV_MAX_LEVELS:
        raise EncodeError("set geometry outside the CUDA encoder's limits")
    for k in range(1, levels + 1):
        ep.level_threshold[k - 1] = float(np.float32(threshold_value(p.alpha, k - 1, levels)))
    if n > 1:
        big = int(math.log2(n))
        for ti in range(1, n):
            ep.temporal_threshold[ti] = float(np.float32(threshold_value(
                p.inter_threshold, temporal_level_of(ti, n) - 1, big)))
    ws_bytes, cap = C.c_uint64(), C.c_uint64()
    nat.check(lib.wv_encode_workspace_bytes(C.byref(ep), C.byref(ws_bytes)), "wv_encode_workspace_bytes")
    nat.check(lib.wv_encode_payload_capacity(C.byref(ep), C.byref(cap)), "wv_encode_payload_capacity")
    frames = chunk.contiguous()
    rowf = torch.as_tensor(np.asarray(hfac, np.float32), device=dev).contiguous()
    ws = torch.empty(ws_bytes.value, dtype=torch.uint8, device=dev)
    nb = (w // p.block_size) * (h // p.block_size)
    ext = torch.empty((n, c, 4), dtype=_F, device=dev)
    counts = torch.empty((n, nb), dtype=torch.int32, device=dev)
    payload = torch.empty(cap.value, dtype=torch.uint8, device=dev)
    nrec = torch.zeros(1, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    nat.check(lib.wv_encode_set(C.byref(ep), C.c_void_p(frames.data_ptr()),
                                C.c_void_p(rowf.data_ptr()), C.c_void_p(ws.data_ptr()),
                                C.c_uint64(ws_bytes.value), C.c_void_p(ext.data_ptr()),
                                C.c_void_p(counts.data_ptr()), C.c_void_p(payload.data_ptr()),
                                C.c_uint64(cap.value), C.c_void_p(nrec.data_ptr()),
                                C.c_void_p(stream)), "wv_encode_set")
    r = int(nrec.item())
    rs = 2 + c if p.quantize else 2 + 4 * c
    packed = payload[:r * rs].cpu().numpy().tobytes()
    del ws, payload
    rec = SparseCoefficients(
        temporal=np.zeros(0, np.uint8), block=np.zeros(0, np.uint32),
        offset=np.zeros(r, np.uint16),
        values=np.zeros((0, c), np.float32 if not p.quantize else np.uint8),
        packed=packed, counts=counts.cpu().numpy().astype(np.int64))
    if keep_arrays:
        arr = np.frombuffer(packed, np.dtype([("o", "<u2"), ("v", "<f4" if not p.quantize else "u1", (c,))]))
        cnt = rec.counts.reshape(-1)
        keys = np.repeat(np.arange(n * nb, dtype=np.int64), cnt)
        rec.temporal = (keys // nb).astype(np.uint8)
        rec.block = (keys % nb).astype(np.uint32)
        rec.offset = arr["o"].copy()
        rec.values = arr["v"].copy()
    return EncodedSet(records=rec, extrema=ext.cpu().numpy())


def encode_video(frames, params: EncodeParams, device=None,
                 keep_arrays: bool = True, backend: str = "native") -> EncodedVideo:
    """Encode (F, H, W[, C]) uint8 frames into sparse sets
    (encoding.py:377-425).  ``frames`` may be a numpy array or a torch
    tensor (already on ``device``).  On a CUDA device the sets go through the
    CUDA encoder (``backend="native"``, csrc/wv_encode.cu); ``backend="torch"``
    (and every CPU encode) runs the torch restatement below."""
    if backend not in ("native", "torch"):
        raise EncodeError(f"unknown backend {backend!r}")
    if isinstance(frames, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(frames))
    else:
        x = frames
    if x.dim() == 3:
        x = x[..., None]
    if x.numel() == 0 or x.shape[0] == 0:
        raise EncodeError("empty input")
    count, h, w, c = x.shape
    levels = params.resolved_levels(w, h)
    n = params.inter_size
    pad = (-count) % n
    dev = torch.device(device) if device is not None else x.device
    hfac = (equirect_mapping_factors(h) if params.mapping is MappingKind.EQUIRECTANGULAR
            else np.zeros(h, np.float32))
    sets = []
    k255 = None
    for s0 in range(0, count + pad, n):
        idx = [min(i, count - 1) for i in range(s0, s0 + n)]
        if idx[-1] == s0 + n - 1:   # whole set present: a view (pinned sources copy async)
            chunk = x[s0:s0 + n].to(dev, non_blocking=True)      # (n, H, W, C) u8
        else:
            chunk = x[idx].to(dev)
        if dev.type == "cuda" and backend == "native":
            sets.append(_encode_set_native(chunk, params, levels, hfac, keep_arrays))
            del chunk
            continue
        if k255 is None:
            k255 = torch.tensor(255.0, dtype=_F, device=dev)
        f = (chunk.to(_F) / k255).permute(0, 3, 1, 2).contiguous()
        sets.append(_encode_set(f, params, levels, hfac, keep_arrays))
        del chunk, f
    return EncodedVideo(w, h, count, params.fps, c, levels, n, params.block_size,
                        params.mask_w, params.mask_h, pad, not params.quantize,
                        params.stereo, sets)

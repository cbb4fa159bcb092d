"""DecodeSession on the B200: the drop-in for wavevid.decoding.DecodeSession.

Public behaviour follows pkg/src/wavevid/decoding.py:184-354 (same methods,
arguments, return types, errors, stats and two-set cache bookkeeping); the
work inside ``_decode`` (decoding.py:260-307) is three C-ABI calls into the
sm_100a kernels (include/wavevid_b200.h):

  K1 wv_select            level masks, foveation windows, block work list,
                          synthesis tile lists, footprint, byte/record stats
  K2 wv_dequant_temporal  dequantise + inverse temporal Haar + inclusion
  K3 wv_synthesize        per-level inverse CDF 9/7 + u8 conversion

The compressed set payload (BlockEnd table + packed records) is read from
the file once per set into pinned memory and copied to HBM; the kernels
address records through the table in place.  One session = one CUDA stream.
There is no CPU fallback: without the extension or a GPU, construction
raises.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import functools
import math
import os
import threading
import time
from collections import OrderedDict, deque
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .fileio import COALESCE_GAP, VideoReader
from .projection import (CameraPose, CoverageError, launch_views, set_view_pose, unpack_footprint,
                         view_args)


class DecodeError(ValueError):
    pass


class CorruptStreamError(DecodeError):
    pass


@dataclass
class FoveationSchedule:
    """Per-level retained viewport fraction, coarsest first, plus the gaze
    point in viewport coordinates (decoding.py:93-121)."""

    fractions: tuple
    gaze_u: float = 0.5
    gaze_v: float = 0.5

    def __post_init__(self):
        f = tuple(float(x) for x in self.fractions)
        if not f or f[0] != 1.0:
            raise DecodeError("coarsest fraction must be 1.0")
        if any(b > a for a, b in zip(f, f[1:])):
            raise DecodeError("fractions must be non-increasing toward finer levels")
        if not (0.0 <= self.gaze_u <= 1.0 and 0.0 <= self.gaze_v <= 1.0):
            raise DecodeError("gaze must lie inside the viewport")
        self.fractions = f

    @classmethod
    def default(cls, levels: int, gaze_u: float = 0.5, gaze_v: float = 0.5):
        if levels == 6:
            fr = (1.0, 0.65, 0.40, 0.22, 0.10, 0.04, 0.02)
        elif levels == 1:
            fr = (1.0, 0.02)
        else:
            fr = (1.0,) + tuple(np.geomspace(0.65, 0.02, levels))
        return cls(fr, gaze_u, gaze_v)


@dataclass
class DecodeStats:
    bytes_loaded: int = 0
    records_processed: int = 0
    load_ms: float = 0.0
    temporal_ms: float = 0.0
    synthesis_ms: float = 0.0

    @property
    def decode_ms(self) -> float:
        return self.load_ms + self.temporal_ms + self.synthesis_ms


@dataclass
class SessionStats:
    bytes_loaded: int = 0
    records_processed: int = 0
    frames_decoded: int = 0
    total_ms: float = 0.0


@functools.lru_cache(maxsize=16)
def _upscale_ranges(n: int, m: int):
    """For the nearest upscale of m cells to n pixels (index map
    ``arange(n) * m // n``, fileio.py:430-436): per cell the pixel range
    [start, end) that maps to it (empty when n < m skips the cell)."""
    idx = np.arange(n, dtype=np.int64) * m // n
    cells = np.arange(m)
    return np.searchsorted(idx, cells, "left"), np.searchsorted(idx, cells, "right")


def _axis_extent(any_cells: np.ndarray, n: int):
    start, end = _upscale_ranges(n, any_cells.size)
    hit = np.flatnonzero(any_cells & (end > start))
    if hit.size == 0:
        return None
    return int(start[hit[0]]), int(end[hit[-1]])


def mask_bbox(mask: np.ndarray, width: int, height: int):
    """Bounding box (y0, y1, x0, x1) of the upscaled pixel mask, computed
    from the low-resolution mask through the nearest-neighbour index maps
    (fileio.py:430-436) without materialising the full-resolution mask: the
    first and last set cells per axis whose pixel range is not empty."""
    m = np.asarray(mask, bool)
    ys = _axis_extent(m.any(axis=1), height)
    xs = _axis_extent(m.any(axis=0), width) if ys is not None else None
    if ys is None or xs is None:
        return None
    return ys[0], ys[1], xs[0], xs[1]


def fovea_rects(bbox, height: int, width: int, schedule: FoveationSchedule, levels: int):
    """Per detail level (finest first) the gaze window (r0, r1, c0, c1) in
    pixels, float64 arithmetic as decoding.py:133-151."""
    y0, y1, x0, x1 = bbox
    gw, gh = x1 - x0, y1 - y0
    cx = x0 + schedule.gaze_u * gw
    cy = y0 + schedule.gaze_v * gh
    fr = list(schedule.fractions[1:])
    while len(fr) < levels:
        fr.append(fr[-1] if fr else 1.0)
    out = []
    for k in range(1, levels + 1):
        f = fr[levels - k]
        hw, hh = f * gw / 2.0, f * gh / 2.0
        out.append((max(0, int(cy - hh)), min(height, int(math.ceil(cy + hh))),
                    max(0, int(cx - hw)), min(width, int(math.ceil(cx + hw)))))
    return out


class _Entry:
    """Reference cache entry (decoding.py:168-173): which blocks of a set
    have been accounted and their cumulative span bytes, kept on device."""

    def __init__(self, set_index: int, nb: int, device):
        self.set_index = set_index
        self.loaded = torch.zeros(max(1, (nb + 31) // 32), dtype=torch.int32, device=device)
        self.nbytes = torch.zeros(1, dtype=torch.int64, device=device)
        self.bytes_loaded = 0


class _Pending:
    __slots__ = ("slot", "set_index", "entry", "existed", "may_evict", "event", "ev",
                 "account_only", "stats", "raw", "spanq")

    def __init__(self):
        self.stats = None
        self.raw = None
        self.spanq = None


class _Prefetcher:
    """Span residency's prefetch engine (DecodeSession.advance,
    decoding.py:335-354): a selection-only workspace, its own descriptor,
    fetch-list buffers and read queue, all driven on the session's copy
    stream -- the next set's block selection, file reads and host -> HBM
    copies overlap the current set's decodes on the session stream."""

    def __init__(self, sess):
        lib, g = sess._lib, sess._geom
        nbytes = C.c_uint64()
        N.check(lib.wv_workspace_bytes_select(C.byref(g), C.byref(nbytes)),
                "wv_workspace_bytes_select")
        h = sess.header
        with torch.cuda.stream(sess._copy_stream):
            self.ws = torch.zeros(int(nbytes.value), dtype=torch.uint8, device=sess.device)
            self.mask = torch.zeros(h.mask_h * h.mask_w, dtype=torch.uint8, device=sess.device)
        self.mask_host = torch.zeros(h.mask_h * h.mask_w, dtype=torch.uint8).pin_memory()
        self.args_host = torch.zeros(_FA_BYTES, dtype=torch.uint8).pin_memory()
        self.args = N.FrameArgs.from_address(self.args_host.data_ptr())
        self.flist = torch.zeros(max(1, h.num_blocks), dtype=torch.int32).pin_memory()
        self.fcount = torch.zeros(4, dtype=torch.int32).pin_memory()
        self.spanq = N.SpanQueue()


class DeviceFrame:
    """Device-resident decode result.  ``canvas`` planar (C, H, W) u8 and
    ``footprint_bits`` (H, ceil(W/32)) int32 are the session's buffers and
    stay valid until the next decode call on the session."""

    def __init__(self, session, pending: _Pending, canvas, footprint_bits):
        self._session = session
        self._pending = pending
        self.canvas = canvas
        self.footprint_bits = footprint_bits

    def stats(self) -> DecodeStats:
        self._session._settle_until(self._pending)
        return self._pending.stats

    def result(self) -> N.FrameResult:
        """Raw device result (tile/block counts) after settling."""
        self._session._settle_until(self._pending)
        return self._pending.raw


_RESULT_BYTES = C.sizeof(N.FrameResult)
_FA_BYTES = C.sizeof(N.FrameArgs)
_VA_BYTES = C.sizeof(N.ViewArgs)
_DESC_BYTES = _FA_BYTES + 4 * _VA_BYTES
_RING = 64
_NO_CTX = contextlib.nullcontext()
_MODES = {"full": N.WV_MODE_FULL, "viewport": N.WV_MODE_VIEWPORT, "foveated": N.WV_MODE_FOVEATED}


class DecodeSession:
    """Single-owner decode session on one GPU stream with one-slot prefetch."""

    def __init__(self, path, device=None, max_resident_sets: int = 4, residency: str = "set",
                 tile_strips: int = 1):
        """``residency``: "set" reads a set's whole payload and uploads it to
        HBM when it is first decoded; "spans" reads and uploads only its
        BlockEnd table, and each decode streams the record spans of newly
        selected blocks from the file (VideoReader.load_blocks,
        fileio.py:346-390, 4 KiB coalescing) inside the frame's stream order:
        the GPU lists the blocks, a stream-ordered host function reads their
        spans into pinned memory, and the fetch kernel copies them to HBM.
        ``tile_strips``: synthesis tile width in 28-column warp strips -- 2
        (56 columns, the ``_wvb200_wide.so`` build) is faster for sessions
        that decode whole frames, 1 for viewport decodes; results are
        identical."""
        if residency not in ("set", "spans"):
            raise ValueError(f"residency {residency!r} not in ('set', 'spans')")
        self.residency = residency
        self.bytes_fetched = 0         # spans residency: record bytes copied host -> HBM
        if not torch.cuda.is_available():
            raise RuntimeError("the B200 decode path needs a CUDA device (no CPU fallback)")
        self._lib = N.load_tiles(tile_strips)
        self.reader = VideoReader(path)
        h = self.reader.header
        self.header = h
        self._fd = None
        if residency == "spans":
            # span streaming: a private descriptor for pread, the job queue of
            # the stream-ordered reads, and the GPU's fetch list in host memory
            self._fd = os.open(path, os.O_RDONLY)
            self._spanq = N.SpanQueue()
            self._h_flist = torch.zeros(max(1, h.num_blocks), dtype=torch.int32).pin_memory()
            self._h_fcount = torch.zeros(4, dtype=torch.int32).pin_memory()
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self._geom = N.Geometry(h.width, h.height, h.channels, h.levels, h.inter_size,
                                h.block_size, int(h.float_mode), h.mask_w, h.mask_h)
        nbytes = C.c_uint64()
        N.check(self._lib.wv_workspace_bytes(C.byref(self._geom), C.byref(nbytes)),
                "wv_workspace_bytes")
        self.stream = torch.cuda.Stream(self.device)
        self._copy_stream = torch.cuda.Stream(self.device)
        self._io_lock = threading.Lock()
        wpr0 = (h.width + 31) // 32
        with torch.cuda.stream(self.stream):
            self._ws = torch.empty(int(nbytes.value), dtype=torch.uint8, device=self.device)
            N.check(self._lib.wv_workspace_reset(C.byref(self._geom), C.c_void_p(self._ws.data_ptr()),
                                                 C.c_void_p(self.stream.cuda_stream)),
                    "wv_workspace_reset")
            # planar (C, H, W): K3 writes each channel plane with coalesced stores
            self._canvas = torch.zeros((h.channels, h.height, h.width), dtype=torch.uint8,
                                       device=self.device)
            self._footprint = torch.zeros((h.height, wpr0), dtype=torch.int32, device=self.device)
            self._mask_dev = torch.zeros((_RING, h.mask_h * h.mask_w), dtype=torch.uint8,
                                         device=self.device)
            self._results = torch.zeros((_RING, _RESULT_BYTES), dtype=torch.uint8,
                                        device=self.device)
            self._uncovered = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._mask_host = torch.zeros((_RING, h.mask_h * h.mask_w), dtype=torch.uint8).pin_memory()
        # descriptor slot: wv_frame_args, 4 wv_view_args, mask bytes (wv_desc_layout)
        moff, sbytes = C.c_uint64(), C.c_uint64()
        N.check(self._lib.wv_desc_layout(C.byref(self._geom), C.byref(moff), C.byref(sbytes)),
                "wv_desc_layout")
        self._desc_mask_off, self._desc_bytes = int(moff.value), int(sbytes.value)
        self._desc_host = torch.zeros((_RING, self._desc_bytes), dtype=torch.uint8).pin_memory()
        dptr = C.c_void_p()
        N.check(self._lib.wv_desc_view(C.byref(self._geom), C.c_void_p(self._ws.data_ptr()),
                                       C.byref(dptr)), "wv_desc_view")
        doff = dptr.value - self._ws.data_ptr()
        self._desc_dev = self._ws[doff: doff + self._desc_bytes]
        self._desc_dev_ptr = self._desc_dev.data_ptr()
        # per ring slot: the frame arguments live directly in the pinned slot;
        # masks are copied next to them, so one H2D per frame carries both
        self._slot_args = [N.FrameArgs.from_address(self._desc_host[i].data_ptr())
                           for i in range(_RING)]
        self._slot_mask = [self._desc_host[i].numpy()[self._desc_mask_off:
                                                      self._desc_mask_off + h.mask_h * h.mask_w]
                           for i in range(_RING)]
        self._graphs: dict = {}
        self.use_graphs = True
        with torch.cuda.stream(self.stream):
            # all-ones footprint for foveated writeout (cli.py:177, service.py:135)
            self._ones_fp = torch.full_like(self._footprint, -1)
        self.shared_view_geometry = int(os.environ.get("WV_SHARED_VIEW_GEOMETRY", "1"))
        self.fork_footprint = int(os.environ.get("WV_FORK_FOOTPRINT", "1")) != 0
        self._aux_stream = torch.cuda.Stream(self.device)
        self._aux_stream2 = torch.cuda.Stream(self.device)
        self._results_host = torch.zeros((_RING, _RESULT_BYTES), dtype=torch.uint8).pin_memory()
        # one completion event per ring slot, materialised (recorded once) so
        # that wv_enqueue_frame can record its handle
        self._slot_events = []
        for _ in range(_RING):
            ev = torch.cuda.Event()
            ev.record(self.stream)
            self._slot_events.append(ev)
        # wv_enqueue_frame arguments that never change, per ring slot
        self._enq_desc = C.c_void_p(self._desc_dev_ptr)
        self._enq_bytes = C.c_uint64(self._desc_bytes)
        self._enq_stream = C.c_void_p(self.stream.cuda_stream)
        self._enq_args = [(C.c_void_p(self._desc_host[i].data_ptr()),
                           C.c_void_p(self._results[i].data_ptr()),
                           C.c_void_p(self._results_host[i].data_ptr()),
                           C.c_void_p(self._slot_events[i].cuda_event)) for i in range(_RING)]
        self._slot = 0
        self._cache: dict[int, _Entry] = {}
        self._resident: OrderedDict = OrderedDict()
        self._max_resident = max(2, max_resident_sets)
        self._pending: deque = deque()
        self._n_may_evict = 0          # pending launches whose settle may evict
        self._view_cache = {}          # (footprint, out, out shape) -> eye ViewArgs
        self._stats = SessionStats()
        self._prefetch_thread: threading.Thread | None = None
        self._prefetch_job = None
        self._prefetcher = None          # spans residency: created by the first advance()
        self._counts_cache: dict = {}    # spans residency: set -> (host payload, u16 counts)
        self._prefetch_ready: dict = {}  # set -> event of its prefetch on the copy stream
        self.time_stages = True
        self.kernel_timing = False
        self.kernel_events: list = []

    # -- lifecycle ------------------------------------------------------------

    def close(self):
        self.join_prefetch()
        if self._pending:
            self._settle_until(None)
        self.reader.close()
        if self.residency == "spans" and self._fd is not None:
            os.close(self._fd)
            self._fd = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def stats(self) -> SessionStats:
        self._settle_until(None)
        return self._stats

    # -- set payloads -----------------------------------------------------------

    def _read_payload(self, set_index: int) -> torch.Tensor:
        """The set payload in pinned host memory, zero-padded to 16 bytes (the
        span fetch copies 16-byte chunks).  Span residency reads only the
        BlockEnd table here; record spans are read per decode."""
        n = self.reader.payload_length(set_index)
        host = torch.zeros((n + 15) // 16 * 16, dtype=torch.uint8).pin_memory()
        with self._io_lock:
            if self.residency == "spans":
                self.reader.read_set_table(set_index, memoryview(host.numpy()[:n]))
            else:
                self.reader.read_set_payload(set_index, memoryview(host.numpy()[:n]))
        return host

    def _table_counts(self, set_index: int, host: torch.Tensor):
        """Per-(t, block) record counts of a set's BlockEnd table as pinned
        u16 (a quarter of the table's bytes), or None when the table is not
        monotone / record-aligned / small enough (then it is uploaded as is,
        so a corrupt table still reports the reference's errors)."""
        hit = self._counts_cache.get(set_index)
        if hit is not None and hit[0] is host:
            return hit[1]
        h = self.header
        ends = np.frombuffer(host.numpy()[: h.table_bytes].tobytes(), dtype="<u8")
        rs = h.record_size
        out = None
        if ends.size and np.all(ends[1:] >= ends[:-1]):
            d = np.diff(ends, prepend=np.uint64(0))
            if not np.any(d % rs) and int(d.max()) // rs < 65536:
                out = torch.from_numpy((d // rs).astype(np.uint16).view(np.int16)).pin_memory()
        self._counts_cache[set_index] = (host, out)
        return out

    @property
    def table_upload_bytes(self) -> int:
        """Host -> HBM bytes of one set's BlockEnd table under span residency
        (the compact counts when the table allows it)."""
        h = self.header
        return h.table_bytes // 4 if self._counts_cache and all(
            v[1] is not None for v in self._counts_cache.values()) else h.table_bytes

    def _push_span_job(self, set_index: int, host: torch.Tensor, slot: int,
                       q=None, flist=None, fcount=None) -> None:
        """Queue the file read of this frame's fetch list (consumed in stream
        order by the host function that wv_span_queue_enqueue placed)."""
        q = self._spanq if q is None else q
        flist = self._h_flist if flist is None else flist
        fcount = self._h_fcount if fcount is None else fcount
        h = self.header
        tb = h.table_bytes
        j = N.SpanJob()
        j.fd, j.n, j.nb = self._fd, h.inter_size, h.num_blocks
        j.payload_offset = self.reader.set_meta[set_index].payload_offset
        j.payload_bytes = self.reader.payload_length(set_index)
        j.table_bytes = tb
        j.table = host.data_ptr()
        j.dst = host.data_ptr()
        j.ids, j.count = flist.data_ptr(), fcount.data_ptr()
        j.coalesce_gap = COALESCE_GAP
        N.check(self._lib.wv_span_queue_push(C.byref(q), C.byref(j), slot),
                "wv_span_queue_push")

    def _span_read_then_fetch(self, stream) -> None:
        """Stream-ordered: read the listed spans from the file, then copy
        them to HBM (the host-argument call paths)."""
        N.check(self._lib.wv_span_queue_enqueue(C.byref(self._spanq),
                                                C.c_void_p(stream.cuda_stream)),
                "wv_span_queue_enqueue")
        mode = N.WV_MODE_FULL   # the fetch stage ignores the mode
        N.check(self._lib.wv_decode_stages_desc(
            C.byref(self._geom), mode, N.WV_FLAG_FETCH, N.WV_STAGE_FETCH,
            C.c_void_p(self._ws.data_ptr()), C.c_void_p(stream.cuda_stream)),
            "wv_decode_stages_desc")

    def pinned_payload(self, set_index: int) -> torch.Tensor:
        """The set's payload (BlockEnd table + records) read into pinned host
        memory, for callers that stream sets themselves (upload_set)."""
        return self._read_payload(set_index)

    def upload_set(self, set_index: int, host: torch.Tensor) -> None:
        """Copy a set payload from (pinned) host memory to HBM on the session
        stream, replacing any resident copy (end-to-end host-buffer path)."""
        self._resident.pop(set_index, None)
        self._make_resident(set_index, host)

    def _make_resident(self, set_index: int, host: torch.Tensor | None = None, stream=None):
        if set_index in self._resident:
            self._resident.move_to_end(set_index)
            return self._resident[set_index]
        if host is None:
            host = self._read_payload(set_index)
        meta = self.reader.set_meta[set_index]
        ext_host = torch.from_numpy(np.ascontiguousarray(meta.extrema, np.float32)).pin_memory()
        fetched = None
        with torch.cuda.stream(stream or self.stream):
            dev = torch.empty(host.numel(), dtype=torch.uint8, device=self.device)
            if self.residency == "set":
                dev.copy_(host, non_blocking=True)
            else:
                # BlockEnd table only; record bytes arrive per selected block.
                # Unfetched bytes read as 0xFF (offset 65535: a decode reading
                # them would report a corrupt stream).
                tb = self.header.table_bytes
                dev.fill_(0xFF)
                counts = self._table_counts(set_index, host)
                if counts is None:   # not a well-formed table: upload it as it is
                    dev[:tb].copy_(host[:tb], non_blocking=True)
                else:
                    # 2-byte record counts, cumulative ends rebuilt in HBM
                    dc = torch.empty(counts.numel(), dtype=torch.int16, device=self.device)
                    dc.copy_(counts, non_blocking=True)
                    N.check(self._lib.wv_table_expand(
                        C.c_void_p(dc.data_ptr()), C.c_uint64(counts.numel()),
                        self.header.record_size, C.c_void_p(dev.data_ptr()),
                        C.c_void_p(torch.cuda.current_stream().cuda_stream)), "wv_table_expand")
                fetched = torch.zeros(max(1, (self.header.num_blocks + 31) // 32),
                                      dtype=torch.int32, device=self.device)
            ext = torch.empty(ext_host.shape, dtype=torch.float32, device=self.device)
            ext.copy_(ext_host, non_blocking=True)
        self._resident[set_index] = (dev, ext, (host, ext_host, fetched))
        while len(self._resident) > self._max_resident:
            self._resident.popitem(last=False)
        return self._resident[set_index]

    # -- reference cache bookkeeping -------------------------------------------

    def _store(self, entry: _Entry):
        """decoding.py:236-241."""
        self._cache[entry.set_index] = entry
        if len(self._cache) > 2:
            oldest = min(self._cache)
            if oldest != entry.set_index:
                del self._cache[oldest]

    def _entry_for(self, set_index: int) -> tuple[_Entry, bool, bool]:
        if self._n_may_evict:
            self._settle_until(None)
        entry = self._cache.get(set_index)
        if entry is None:
            with torch.cuda.stream(self.stream):
                entry = _Entry(set_index, self.header.num_blocks, self.device)
            self._store(entry)
            return entry, False, False
        return entry, True, len(self._cache) > 2

    # -- decode core ------------------------------------------------------------

    def _frame_set(self, frame: int) -> tuple[int, int]:
        if not 0 <= frame < self.header.frame_count:
            raise DecodeError(f"frame {frame} out of range [0, {self.header.frame_count})")
        return frame // self.header.inter_size, frame % self.header.inter_size

    def _check_mask(self, mask: np.ndarray) -> np.ndarray:
        h = self.header
        m = np.asarray(mask)
        if m.shape != (h.mask_h, h.mask_w):
            raise DecodeError(f"mask dims {m.shape} != header ({h.mask_h}, {h.mask_w})")
        return m if m.dtype == np.bool_ else m.astype(bool)

    def _mode_args(self, mode: str, mask, schedule, slot: int, in_desc: bool = False):
        """Frame arguments in ring slot ``slot``.  ``in_desc``: the mask
        travels inside the descriptor slot (graph path, one H2D per frame);
        otherwise it is copied to its own device buffer now."""
        h = self.header
        args = self._slot_args[slot]
        C.memset(C.addressof(args), 0, _FA_BYTES)
        if mode == "full":
            args.mode = N.WV_MODE_FULL
            return args
        m = self._check_mask(mask)
        if in_desc:
            np.copyto(self._slot_mask[slot], m.reshape(-1), casting="unsafe")
            args.d_mask = self._desc_dev_ptr + self._desc_mask_off
        else:
            np.copyto(self._mask_host[slot].numpy(), m.reshape(-1), casting="unsafe")
            self._mask_dev[slot].copy_(self._mask_host[slot], non_blocking=True)
            args.d_mask = self._mask_dev[slot].data_ptr()
        args.mode = N.WV_MODE_VIEWPORT
        if mode == "foveated":
            bbox = mask_bbox(m, h.width, h.height)
            if bbox is not None:   # empty viewport: plain masks (decoding.py:131-132)
                args.mode = N.WV_MODE_FOVEATED
                for k, rect in enumerate(fovea_rects(bbox, h.height, h.width, schedule, h.levels)):
                    for q in range(4):
                        args.fovea[k][q] = rect[q]
        return args

    def _run_fast(self, slot: int, args: N.FrameArgs, mode: str, views=None, out_dims=None,
                  flags: int = 0) -> bool:
        """Per-frame inputs (already in pinned ring slot ``slot``: arguments,
        views, mask) -> the workspace descriptor, then the fixed launch
        sequence of this mode.  After its first direct run the sequence is a
        CUDA graph, and a frame is ONE C call (wv_enqueue_frame: descriptor
        H2D, graph launch, result D2H, completion event); returns True then."""
        host = self._desc_host[slot]
        hptr = host.data_ptr()
        nv = len(views) if views else 0
        for i in range(nv):
            C.memmove(hptr + _FA_BYTES + i * _VA_BYTES, C.addressof(views[i]), _VA_BYTES)
        key = (_MODES[mode], nv, tuple(out_dims) if nv else None, flags)
        g = self._graphs.get(key)
        if g is not None:
            ea = self._enq_args[slot]
            st = self._lib.wv_enqueue_frame(self._enq_desc, ea[0], self._enq_bytes, g[1],
                                            self._enq_stream, ea[1], ea[2], ea[3])
            if st:
                N.check(st, "wv_enqueue_frame")
            return True
        with torch.cuda.stream(self.stream):
            return self._first_run(host, key, flags, nv, views, out_dims)

    def _first_run(self, host, key, flags, nv, views, out_dims) -> bool:
        """Direct run of a mode's launch sequence, then its graph capture."""
        self._desc_dev.copy_(host, non_blocking=True)
        spans = self.residency == "spans"

        def run(stages, stream):
            N.check(self._lib.wv_decode_stages_desc(
                C.byref(self._geom), key[0], flags, stages, C.c_void_p(self._ws.data_ptr()),
                C.c_void_p(stream.cuda_stream)), "wv_decode_stages_desc")

        def seq():
            cur = torch.cuda.current_stream()
            if self.fork_footprint:
                # rows -> {tile lists} || cascades -> {footprint chain} ||
                # block selection -> K2; K3 joins the tile lists, the finest
                # footprint step joins the footprint chain
                aux, aux2 = self._aux_stream, self._aux_stream2
                run(N.WV_STAGE_ROWS, cur)
                ev_r = torch.cuda.Event()
                ev_r.record(cur)
                aux2.wait_event(ev_r)
                run(N.WV_STAGE_TILES, aux2)
                ev_t = torch.cuda.Event()
                ev_t.record(aux2)
                run(N.WV_STAGE_CASCADES, cur)
                ev_c = torch.cuda.Event()
                ev_c.record(cur)
                aux.wait_event(ev_c)
                run(N.WV_STAGE_FOOTPRINT, aux)
                # the finest footprint step needs the level-1 tile list, not
                # K3: it runs beside synthesis and only K4 waits for it
                aux.wait_event(ev_t)
                run(N.WV_STAGE_FOOTPRINT_TILES, aux)
                ev_f = torch.cuda.Event()
                ev_f.record(aux)
                if spans:
                    # span streaming: the GPU's fetch list -> file reads
                    # (stream-ordered host function) -> fetch kernel -> K2
                    run(N.WV_STAGE_BLOCKS, cur)
                    N.check(self._lib.wv_span_queue_enqueue(
                        C.byref(self._spanq), C.c_void_p(cur.cuda_stream)),
                        "wv_span_queue_enqueue")
                    run(N.WV_STAGE_FETCH | N.WV_STAGE_DEQUANT, cur)
                else:
                    run(N.WV_STAGE_BLOCKS | N.WV_STAGE_FETCH | N.WV_STAGE_DEQUANT, cur)
                cur.wait_event(ev_t)
                run(N.WV_STAGE_SYNTH, cur)
                cur.wait_event(ev_f)
            elif spans:
                run(N.WV_STAGE_SELECT, cur)
                N.check(self._lib.wv_span_queue_enqueue(
                    C.byref(self._spanq), C.c_void_p(cur.cuda_stream)),
                    "wv_span_queue_enqueue")
                run(N.WV_STAGE_FETCH | N.WV_STAGE_DEQUANT | N.WV_STAGE_SYNTH, cur)
            else:
                N.check(self._lib.wv_decode_frame_desc(
                    C.byref(self._geom), key[0], flags, C.c_void_p(self._ws.data_ptr()),
                    C.c_void_p(cur.cuda_stream)), "wv_decode_frame_desc")
            if nv:
                # all eyes of a session share pose and region size (stereo pair)
                N.check(self._lib.wv_render_perspective_desc(
                    C.c_void_p(self._desc_dev.data_ptr() + _FA_BYTES), nv, out_dims[0],
                    out_dims[1], self.shared_view_geometry,
                    C.c_void_p(cur.cuda_stream)),
                    "wv_render_perspective_desc")

        seq()
        if self.use_graphs:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=self.stream, capture_error_mode="relaxed"):
                seq()
            self._graphs[key] = (graph, C.c_void_p(graph.raw_cuda_graph_exec()))
        return False

    def _launch(self, frame: int, mode: str, mask=None, schedule=None,
                account_only: bool = False, time_stages: bool = False,
                views=None, out_dims=None, out_rows=None) -> _Pending:
        self.join_prefetch()
        si, t = self._frame_set(frame)
        if mode != "full":
            self._check_mask(mask)
        s = self.stream
        p = _Pending()
        if len(self._pending) >= _RING:
            self._settle_until(self._pending[0])
        slot = self._slot
        self._slot = (self._slot + 1) % _RING
        fast = not (account_only or self.kernel_timing or time_stages)
        # the graph fast path enqueues through the C ABI with the stream
        # passed explicitly; only the other paths issue torch ops here
        ready = self._prefetch_ready.pop(si, None)
        if ready is not None:   # the set's prefetch (copy stream) precedes its decodes
            s.wait_event(ready)
        with (_NO_CTX if fast else torch.cuda.stream(s)):
            ev0 = torch.cuda.Event(enable_timing=True) if time_stages else None
            if ev0 is not None:
                ev0.record(s)
            dev, ext, keep = self._make_resident(si)
            args = self._mode_args(mode, mask, schedule, slot, in_desc=fast)
            entry, existed, may_evict = self._entry_for(si)
            args.t = t
            args.flags = N.WV_FLAG_ACCOUNT_ONLY if account_only else 0
            if out_rows is not None:
                args.out_row0, args.out_row1 = out_rows
            spans = self.residency == "spans"
            if spans:
                args.flags |= N.WV_FLAG_FETCH
                args.h_payload = keep[0].data_ptr()
                args.d_fetched = keep[2].data_ptr()
                args.h_fetch_list = self._h_flist.data_ptr()
                args.h_fetch_count = self._h_fcount.data_ptr()
                self._push_span_job(si, keep[0], slot)
            args.d_payload = dev.data_ptr()
            args.payload_bytes = self.reader.payload_length(si)
            args.d_extrema = ext.data_ptr()
            args.d_set_loaded = entry.loaded.data_ptr()
            args.d_set_bytes = entry.nbytes.data_ptr()
            args.d_canvas = self._canvas.data_ptr()
            args.d_footprint = self._footprint.data_ptr()
            args.d_result = self._results[slot].data_ptr()
            g, ws, cs = C.byref(self._geom), C.c_void_p(self._ws.data_ptr()), C.c_void_p(s.cuda_stream)
            evs = None
            done = None
            if account_only:
                N.check(self._lib.wv_select(g, C.byref(args), ws, cs), "wv_select")
                if spans:
                    self._span_read_then_fetch(s)
            elif self.kernel_timing:
                # per-kernel CUDA events on this stream: K1, K2, K3 levels L..2, K3 level 1
                e = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
                e[0].record(s)
                N.check(self._lib.wv_select(g, C.byref(args), ws, cs), "wv_select")
                if spans:
                    self._span_read_then_fetch(s)
                e[1].record(s)
                N.check(self._lib.wv_decode_stages_desc(g, args.mode, args.flags,
                                                        N.WV_STAGE_DEQUANT, ws, cs),
                        "wv_decode_stages_desc")
                e[2].record(s)
                # (the arguments are in the descriptor since wv_dequant_temporal:
                # the level launches are timed without an argument copy)
                for k in range(self.header.levels, 1, -1):
                    N.check(self._lib.wv_synthesize_level_desc(g, ws, k, cs),
                            "wv_synthesize_level_desc")
                e[3].record(s)
                N.check(self._lib.wv_synthesize_level_desc(g, ws, 1, cs),
                        "wv_synthesize_level_desc")
                e[4].record(s)
                self.kernel_events.append(e)
            elif time_stages:
                evs = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                N.check(self._lib.wv_select(g, C.byref(args), ws, cs), "wv_select")
                if spans:
                    self._span_read_then_fetch(s)
                evs[0].record(s)
                N.check(self._lib.wv_dequant_temporal(g, C.byref(args), ws, cs),
                        "wv_dequant_temporal")
                evs[1].record(s)
                N.check(self._lib.wv_synthesize(g, C.byref(args), ws, cs), "wv_synthesize")
                evs[2].record(s)
            elif self._run_fast(slot, args, mode, views, out_dims, args.flags):
                done = self._slot_events[slot]   # recorded by wv_enqueue_frame
            if done is None:
                with torch.cuda.stream(s):
                    self._results_host[slot].copy_(self._results[slot], non_blocking=True)
                done = torch.cuda.Event()
                done.record(s)
        p.slot, p.set_index, p.entry, p.existed, p.may_evict = slot, si, entry, existed, may_evict
        p.event, p.ev, p.account_only = done, (ev0, evs), account_only
        self._pending.append(p)
        self._n_may_evict += bool(may_evict)
        return p

    def _settle_until(self, target: _Pending | None):
        """Apply results of launched decodes in order (stats, corrupt-stream
        errors, cache store/eviction of existing entries)."""
        while self._pending:
            p = self._pending.popleft()
            self._n_may_evict -= bool(p.may_evict)
            p.event.synchronize()
            r = N.FrameResult.from_buffer_copy(bytes(self._results_host[p.slot].numpy()))
            entry = p.entry
            if p.existed and r.n_missing and self._cache.get(p.set_index) is entry:
                self._store(entry)
            entry.bytes_loaded = int(r.set_bytes)
            st = DecodeStats(bytes_loaded=int(r.new_bytes if r.new_bytes else r.set_bytes),
                             records_processed=int(r.records))
            ev0, evs = p.ev
            if evs is not None:
                st.load_ms = ev0.elapsed_time(evs[0])
                st.temporal_ms = evs[0].elapsed_time(evs[1])
                st.synthesis_ms = evs[1].elapsed_time(evs[2])
            p.stats = st
            p.raw = r
            self.bytes_fetched += int(r.fetched_bytes)
            if self.residency == "spans":
                job = (p.spanq or self._spanq).jobs[p.slot]
                if job.done and job.bytes_read:
                    self.reader.io_trace.append((p.set_index, int(job.bytes_read)))
                if job.done and job.status:
                    raise CorruptStreamError(
                        f"span read failed ({N.status_name(job.status)}): BlockEnd table "
                        "inconsistent with the file")
            if not p.account_only:
                self._stats.bytes_loaded += st.bytes_loaded
                self._stats.records_processed += st.records_processed
                self._stats.frames_decoded += 1
                self._stats.total_ms += st.decode_ms
            if r.error:
                raise CorruptStreamError(
                    "record offset outside block" if r.error & N.WV_DERR_OFFSET
                    else "BlockEnd table inconsistent with payload")
            if p is target:
                return

    def _decode(self, frame: int, mode: str, mask=None, schedule=None):
        p = self._launch(frame, mode, mask, schedule, time_stages=self.time_stages)
        self._settle_until(p)
        h = self.header
        with torch.cuda.stream(self.stream):
            hwc = self._canvas.permute(1, 2, 0).contiguous()
        self.stream.synchronize()
        pixels = hwc.cpu().numpy()
        footprint = unpack_footprint(self._footprint.cpu().numpy(), h.width)
        return pixels, footprint, p.stats

    # -- public API (decoding.py:309-354) ----------------------------------------

    def decode_viewport(self, frame: int, mask: np.ndarray):
        """Full-quality decode of the masked region: (pixels, footprint, stats)."""
        return self._decode(frame, "viewport", mask)

    def decode_foveated(self, frame: int, mask: np.ndarray,
                        schedule: FoveationSchedule | None = None):
        schedule = schedule or FoveationSchedule.default(self.header.levels)
        return self._decode(frame, "foveated", mask, schedule)

    def decode_full(self, frame: int):
        return self._decode(frame, "full")

    # device-resident variants for throughput (no host sync, no D2H)
    def decode_viewport_device(self, frame: int, mask: np.ndarray) -> DeviceFrame:
        return DeviceFrame(self, self._launch(frame, "viewport", mask), self._canvas,
                           self._footprint)

    def decode_foveated_device(self, frame: int, mask: np.ndarray,
                               schedule: FoveationSchedule | None = None) -> DeviceFrame:
        schedule = schedule or FoveationSchedule.default(self.header.levels)
        return DeviceFrame(self, self._launch(frame, "foveated", mask, schedule), self._canvas,
                           self._footprint)

    def decode_full_device(self, frame: int) -> DeviceFrame:
        return DeviceFrame(self, self._launch(frame, "full"), self._canvas, self._footprint)

    def _eyes(self):
        h = self.header
        return [(0, h.height)] if not h.stereo else [(0, h.height // 2),
                                                     (h.height // 2, h.height // 2)]

    def decode_render_device(self, frame: int, mode: str, mask, pose: CameraPose, out_dims,
                             out: torch.Tensor, schedule: FoveationSchedule | None = None,
                             eye: int | None = None) -> DeviceFrame:
        """Decode + per-eye perspective writeout as one graph replay (the
        throughput path of a viewer).  ``out`` is (views, out_h, out_w, C) u8
        on the device; coverage is counted in ``uncovered()``.  ``eye`` (0 or
        1, stereo only): synthesise and render that eye alone (its half of
        the canvas, out[0]) -- the per-GPU share of a stereo eye split; its
        pixels and footprint equal the whole-frame decode's."""
        h = self.header
        if mode == "foveated" and schedule is None:
            schedule = FoveationSchedule.default(h.levels)
        # a foveated frame is exact only near the gaze; its callers render with
        # an all-ones footprint (cli.py:177, service.py:135)
        fp = self._footprint
        if mode == "foveated":
            if self._ones_fp is None:
                self._ones_fp = torch.full_like(self._footprint, -1)
            fp = self._ones_fp
        eyes = self._eyes()
        out_rows = None
        if eye is not None:
            if not h.stereo or eye not in (0, 1):
                raise ValueError("eye must be 0 or 1 for a stereo file")
            eyes = [eyes[eye]]
            out_rows = (eyes[0][0], eyes[0][0] + eyes[0][1])
        key = (fp.data_ptr(), out.data_ptr(), tuple(out.shape), eye)
        views = self._view_cache.get(key)
        if views is None:
            views = [view_args(self._canvas, fp, r0, rows, h.width, h.channels, pose,
                               out[i], self._uncovered) for i, (r0, rows) in enumerate(eyes)]
            self._view_cache[key] = views
        else:
            set_view_pose(views, pose)
        p = self._launch(frame, mode, mask, schedule, views=views, out_dims=tuple(out_dims),
                         out_rows=out_rows)
        return DeviceFrame(self, p, self._canvas, self._footprint)

    def uncovered(self, reset: bool = False) -> int:
        """Output pixels whose taps left the footprint, accumulated over
        decode_render_device calls since the last reset."""
        self.stream.synchronize()
        n = int(self._uncovered.item())
        if reset:
            self._uncovered.zero_()
        return n

    def render_views(self, pose: CameraPose, out_dims, out: torch.Tensor | None = None,
                     check: bool = True, all_covered: bool = False,
                     events: tuple | None = None) -> torch.Tensor:
        """Perspective writeout (K4) of the current canvas: one view, or one
        per eye for top-bottom stereo.  Returns
        (views, out_h, out_w, C) u8 on the device.  ``all_covered``: coverage
        against an all-ones footprint, as the reference's foveated callers do
        (cli.py:177, service.py:135)."""
        h = self.header
        out_w, out_h = out_dims
        eyes = [(0, h.height)] if not h.stereo else [(0, h.height // 2),
                                                     (h.height // 2, h.height // 2)]
        if out is None:
            out = torch.empty((len(eyes), out_h, out_w, h.channels), dtype=torch.uint8,
                              device=self.device)
        with torch.cuda.stream(self.stream):
            self._uncovered.zero_()
            fp = self._footprint
            if all_covered:
                if self._ones_fp is None:
                    self._ones_fp = torch.full_like(self._footprint, -1)
                fp = self._ones_fp
            views = [view_args(self._canvas, fp, r0, rows, h.width, h.channels,
                               pose, out[i], self._uncovered) for i, (r0, rows) in enumerate(eyes)]
            if events is not None:   # (start, end) CUDA events around the K4 launch only
                events[0].record(self.stream)
            launch_views(views, self.stream)
            if events is not None:
                events[1].record(self.stream)
        if check:
            self.stream.synchronize()
            missing = int(self._uncovered.item())
            if missing:
                raise CoverageError(f"{missing} output pixels sample outside the footprint")
        return out

    def plane(self) -> torch.Tensor:
        """K2 output (C, H, W) float32 of the last decode (parity tests)."""
        ptr = C.c_void_p()
        N.check(self._lib.wv_plane_view(C.byref(self._geom), C.c_void_p(self._ws.data_ptr()),
                                        C.byref(ptr)), "wv_plane_view")
        h = self.header
        off = ptr.value - self._ws.data_ptr()
        n = h.channels * h.height * h.width
        return self._ws[off: off + 4 * n].view(torch.float32).view(h.channels, h.height, h.width)

    def block_work(self) -> np.ndarray:
        """K2 work list of the last decode (block ids; ZERO_FLAG bit = clear
        only), after the stream has finished."""
        lst, cnt = C.c_void_p(), C.c_void_p()
        N.check(self._lib.wv_block_list_view(C.byref(self._geom), C.c_void_p(self._ws.data_ptr()),
                                             C.byref(lst), C.byref(cnt)), "wv_block_list_view")
        self.stream.synchronize()
        base = self._ws.data_ptr()
        n = int(self._ws[cnt.value - base: cnt.value - base + 4].view(torch.int32).item())
        off = lst.value - base
        return self._ws[off: off + 4 * n].view(torch.int32).cpu().numpy().view(np.uint32)

    def tile_counts(self) -> list:
        """Synthesis tiles listed per level [k = 1..L] by the last decode
        (level 1 includes the tiles only cleared because they left the
        request), after the stream has finished."""
        lst, cnt = C.c_void_p(), C.c_void_p()
        N.check(self._lib.wv_block_list_view(C.byref(self._geom), C.c_void_p(self._ws.data_ptr()),
                                             C.byref(lst), C.byref(cnt)), "wv_block_list_view")
        self.stream.synchronize()
        off = cnt.value - self._ws.data_ptr()   # counters[CNT_BLOCKS]; tiles at [1 + k]
        ctr = self._ws[off: off + 4 * 64].view(torch.int32).cpu().numpy()
        return [int(ctr[1 + k]) for k in range(1, self.header.levels + 1)]

    # -- prefetch (decoding.py:335-354) -------------------------------------------

    def advance(self, current_frame: int, next_mask: np.ndarray) -> None:
        """Read the next inter-frame set in the background; its payload goes
        to HBM and its blocks for ``next_mask`` are accounted in the cache."""
        set_index = current_frame // self.header.inter_size + 1
        if set_index >= self.header.num_sets:
            return
        mask = self._check_mask(next_mask)
        self.join_prefetch()
        if self.residency == "spans":
            self._prefetch_spans(set_index, mask)
            return
        job = {"set": set_index, "mask": mask, "host": None}

        def work():
            if set_index not in self._resident:
                job["host"] = self._read_payload(set_index)

        self._prefetch_job = job
        self._prefetch_thread = threading.Thread(target=work, daemon=True)
        self._prefetch_thread.start()

    def _prefetch_spans(self, si: int, mask: np.ndarray) -> None:
        """Span residency: the next set's BlockEnd table, then -- on the copy
        stream, with the selection-only workspace -- its block selection for
        the predicted mask (accounted in the cache as the reference's
        prefetch does), the file reads of those spans (stream-ordered host
        function) and their copy to HBM.  The set's decodes wait for it."""
        pf = self._prefetcher
        if pf is None:
            pf = self._prefetcher = _Prefetcher(self)
        cs = self._copy_stream
        h = self.header
        # the previous prefetch's list / queue slot must be consumed first
        for p in list(self._pending):
            if p.spanq is pf.spanq:
                self._settle_until(p)
        dev, ext, keep = self._make_resident(si, stream=cs)
        entry, existed, may_evict = self._entry_for(si)
        if len(self._pending) >= _RING:
            self._settle_until(self._pending[0])
        slot = self._slot
        self._slot = (self._slot + 1) % _RING
        np.copyto(pf.mask_host.numpy(), mask.reshape(-1), casting="unsafe")
        a = pf.args
        C.memset(C.addressof(a), 0, _FA_BYTES)
        a.mode, a.t = N.WV_MODE_VIEWPORT, 0
        a.flags = N.WV_FLAG_ACCOUNT_ONLY | N.WV_FLAG_FETCH
        a.d_mask = pf.mask.data_ptr()
        a.d_payload, a.payload_bytes = dev.data_ptr(), self.reader.payload_length(si)
        a.d_extrema = ext.data_ptr()
        a.d_set_loaded, a.d_set_bytes = entry.loaded.data_ptr(), entry.nbytes.data_ptr()
        a.d_canvas, a.d_footprint = self._canvas.data_ptr(), self._footprint.data_ptr()
        a.d_result = self._results[slot].data_ptr()
        a.h_payload, a.d_fetched = keep[0].data_ptr(), keep[2].data_ptr()
        a.h_fetch_list, a.h_fetch_count = pf.flist.data_ptr(), pf.fcount.data_ptr()
        self._push_span_job(si, keep[0], slot, pf.spanq, pf.flist, pf.fcount)
        g, ws, css = C.byref(self._geom), C.c_void_p(pf.ws.data_ptr()), C.c_void_p(cs.cuda_stream)
        with torch.cuda.stream(cs):
            pf.mask.copy_(pf.mask_host, non_blocking=True)
            N.check(self._lib.wv_select(g, C.byref(a), ws, css), "wv_select")
            N.check(self._lib.wv_span_queue_enqueue(C.byref(pf.spanq), css),
                    "wv_span_queue_enqueue")
            N.check(self._lib.wv_decode_stages_desc(g, a.mode, a.flags, N.WV_STAGE_FETCH, ws, css),
                    "wv_decode_stages_desc")
            self._results_host[slot].copy_(self._results[slot], non_blocking=True)
            done = torch.cuda.Event()
            done.record(cs)
        p = _Pending()
        p.slot, p.set_index, p.entry, p.existed, p.may_evict = slot, si, entry, existed, may_evict
        p.event, p.ev, p.account_only, p.spanq = done, (None, None), True, pf.spanq
        self._pending.append(p)
        self._n_may_evict += bool(may_evict)
        self._prefetch_ready[si] = done

    def join_prefetch(self):
        if self._prefetch_thread is not None:
            self._prefetch_thread.join()
            self._prefetch_thread = None
        job, self._prefetch_job = self._prefetch_job, None
        if job is not None:
            si = job["set"]
            self._make_resident(si, job["host"])
            # the set's first frame is always a real frame (pad < inter_size)
            p = self._launch(si * self.header.inter_size, "viewport", job["mask"],
                             account_only=True)
            self._settle_until(p)

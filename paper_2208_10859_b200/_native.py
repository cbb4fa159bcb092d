"""ctypes binding of the C ABI in include/wavevid_b200.h.

The decode path has no CPU fallback: if the library is missing or a call
fails, this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_wvb200.so")
LIB_WIDE_PATH = os.path.join(HERE, "_wvb200_wide.so")   # 56-column synthesis tiles

WV_OK, WV_ERR_ARG, WV_ERR_CUDA, WV_ERR_UNSUPPORTED, WV_ERR_FORMAT, WV_ERR_IO = 0, 1, 2, 3, 4, 5
WV_MODE_FULL, WV_MODE_VIEWPORT, WV_MODE_FOVEATED = 0, 1, 2
WV_FLAG_ACCOUNT_ONLY, WV_FLAG_FETCH = 1, 2
WV_ABI_VERSION = 4
WV_ENC_MAX_N = 64
(WV_STAGE_ROWS, WV_STAGE_CASCADES, WV_STAGE_FOOTPRINT, WV_STAGE_BLOCKS, WV_STAGE_TILES,
 WV_STAGE_FOOTPRINT_TILES, WV_STAGE_DEQUANT, WV_STAGE_SYNTH, WV_STAGE_FETCH) = (
    1, 2, 4, 8, 16, 32, 64, 128, 256)
WV_DERR_OFFSET, WV_DERR_TABLE = 1, 2
WV_MAX_LEVELS = 12

EXPORTS = ["wv_abi_version", "wv_status_string", "wv_workspace_bytes", "wv_workspace_reset",
           "wv_select", "wv_dequant_temporal", "wv_synthesize", "wv_decode_frame",
           "wv_synthesize_level",
           "wv_render_perspective", "wv_plane_view", "wv_level_mask_view",
           "wv_block_list_view", "wv_desc_view", "wv_decode_frame_desc",
           "wv_render_perspective_desc", "wv_file_info_read", "wv_file_set_read",
           "wv_file_payload_read", "wv_decode_stages_desc", "wv_encode_workspace_bytes",
           "wv_encode_payload_capacity", "wv_encode_set", "wv_enqueue_frame",
           "wv_desc_layout", "wv_synthesize_2d", "wv_spans_read", "wv_span_queue_push",
           "wv_span_queue_enqueue", "wv_fetch_list_view", "wv_synthesize_level_desc",
           "wv_workspace_bytes_select", "wv_table_expand", "wv_synthesis_tile"]


class Geometry(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("width", "height", "channels", "levels", "inter_size",
                                         "block_size", "float_mode", "mask_w", "mask_h")]


class EncodeParams(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("width", "height", "channels", "levels", "inter_size",
                                         "block_size", "quantize", "reserved")] + [
        ("level_threshold", C.c_float * WV_MAX_LEVELS),
        ("temporal_threshold", C.c_float * WV_ENC_MAX_N)]


class FileInfo(C.Structure):
    _fields_ = [("geom", Geometry), ("frame_count", C.c_int32), ("pad_frames", C.c_int32),
                ("num_sets", C.c_int32), ("stereo", C.c_int32), ("fps", C.c_float),
                ("version", C.c_uint32), ("table_bytes", C.c_uint64)]


class SetInfo(C.Structure):
    _fields_ = [("payload_offset", C.c_uint64), ("payload_length", C.c_uint64),
                ("record_count", C.c_uint64)]


class FrameResult(C.Structure):
    _fields_ = [("new_bytes", C.c_uint64), ("set_bytes", C.c_uint64), ("records", C.c_uint64),
                ("n_missing", C.c_uint32), ("n_selected", C.c_uint32), ("error", C.c_uint32),
                ("n_tiles", C.c_uint32), ("fetched_bytes", C.c_uint64)]


class FrameArgs(C.Structure):
    _fields_ = [("mode", C.c_int32), ("t", C.c_int32), ("flags", C.c_int32),
                ("reserved", C.c_int32), ("d_mask", C.c_void_p),
                ("fovea", (C.c_int32 * 4) * WV_MAX_LEVELS),
                ("d_payload", C.c_void_p), ("payload_bytes", C.c_uint64),
                ("d_extrema", C.c_void_p), ("d_set_loaded", C.c_void_p),
                ("d_set_bytes", C.c_void_p), ("d_canvas", C.c_void_p),
                ("d_footprint", C.c_void_p), ("d_result", C.c_void_p),
                ("h_payload", C.c_void_p), ("d_fetched", C.c_void_p),
                ("h_fetch_list", C.c_void_p), ("h_fetch_count", C.c_void_p),
                ("out_row0", C.c_int32), ("out_row1", C.c_int32)]


WV_SPAN_QUEUE = 64


class SpanJob(C.Structure):
    _fields_ = [("fd", C.c_int32), ("n", C.c_int32), ("nb", C.c_int32), ("status", C.c_int32),
                ("payload_offset", C.c_uint64), ("payload_bytes", C.c_uint64),
                ("table_bytes", C.c_uint64), ("table", C.c_void_p), ("dst", C.c_void_p),
                ("ids", C.c_void_p), ("count", C.c_void_p),
                ("coalesce_gap", C.c_uint64), ("bytes_read", C.c_uint64),
                ("bytes_spans", C.c_uint64), ("done", C.c_int32), ("reserved", C.c_int32)]


class SpanQueue(C.Structure):
    _fields_ = [("jobs", SpanJob * WV_SPAN_QUEUE), ("fifo", C.c_uint32 * WV_SPAN_QUEUE),
                ("head", C.c_uint32), ("tail", C.c_uint32)]


class ViewArgs(C.Structure):
    _fields_ = [("d_canvas", C.c_void_p), ("d_footprint", C.c_void_p), ("row0", C.c_int32),
                ("rows", C.c_int32), ("width", C.c_int32), ("channels", C.c_int32),
                ("canvas_h", C.c_int32), ("reserved", C.c_int32),
                ("rot", C.c_double * 9), ("tan_h", C.c_double), ("tan_v", C.c_double),
                ("out_w", C.c_int32), ("out_h", C.c_int32), ("d_out", C.c_void_p),
                ("d_uncovered", C.c_void_p)]


class NativeError(RuntimeError):
    pass


_libs: dict = {}


def load(path: str | None = None):
    """Load the decode library (raises if it is absent: no fallback).
    ``WV_LIB`` selects an experimental build variant (build.build(out=...))."""
    path = path or os.environ.get("WV_LIB") or LIB_PATH
    lib = _libs.get(path)
    if lib is not None:
        return lib
    if not os.path.exists(path):
        raise NativeError(
            f"B200 decode library not built: {path} (run python -m paper_2208_10859_b200.build)")
    lib = C.CDLL(path)
    G, A, V = C.POINTER(Geometry), C.POINTER(FrameArgs), C.POINTER(ViewArgs)
    lib.wv_abi_version.restype = C.c_int
    lib.wv_status_string.restype = C.c_char_p
    lib.wv_status_string.argtypes = [C.c_int]
    lib.wv_workspace_bytes.argtypes = [G, C.POINTER(C.c_uint64)]
    lib.wv_workspace_reset.argtypes = [G, C.c_void_p, C.c_void_p]
    for fn in ("wv_select", "wv_dequant_temporal", "wv_synthesize", "wv_decode_frame"):
        getattr(lib, fn).argtypes = [G, A, C.c_void_p, C.c_void_p]
    lib.wv_synthesize_level.argtypes = [G, A, C.c_void_p, C.c_int, C.c_void_p]
    lib.wv_render_perspective.argtypes = [V, C.c_int, C.c_void_p]
    lib.wv_plane_view.argtypes = [G, C.c_void_p, C.POINTER(C.c_void_p)]
    lib.wv_level_mask_view.argtypes = [G, C.c_void_p, C.c_int, C.POINTER(C.c_void_p),
                                       C.POINTER(C.c_int32)]
    lib.wv_block_list_view.argtypes = [G, C.c_void_p, C.POINTER(C.c_void_p),
                                       C.POINTER(C.c_void_p)]
    lib.wv_desc_view.argtypes = [G, C.c_void_p, C.POINTER(C.c_void_p)]
    lib.wv_decode_frame_desc.argtypes = [G, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    lib.wv_render_perspective_desc.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int,
                                               C.c_int, C.c_void_p]
    lib.wv_decode_stages_desc.argtypes = [G, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    lib.wv_file_info_read.argtypes = [C.c_char_p, C.POINTER(FileInfo)]
    lib.wv_file_set_read.argtypes = [C.c_char_p, C.c_int, C.POINTER(SetInfo), C.c_void_p]
    lib.wv_file_payload_read.argtypes = [C.c_char_p, C.c_int, C.c_void_p, C.c_uint64]
    lib.wv_synthesis_tile.argtypes = [C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    for fn in EXPORTS[2:]:
        getattr(lib, fn).restype = C.c_int
    if lib.wv_abi_version() != WV_ABI_VERSION:
        raise NativeError("decode library ABI mismatch")
    _libs[path] = lib
    return lib


def load_tiles(strips: int = 1):
    """The library whose synthesis tiles are ``strips`` warp strips wide:
    1 -> 28 columns (the default build), 2 -> 56 columns (``_wvb200_wide.so``,
    faster for full-frame decodes, slower for viewports)."""
    if strips == 1:
        return load()
    if strips == 2:
        return load(LIB_WIDE_PATH)
    raise ValueError(f"tile_strips must be 1 or 2, not {strips}")


def check(status: int, what: str) -> None:
    if status != WV_OK:
        msg = load().wv_status_string(status).decode()
        raise NativeError(f"{what} failed: {msg} (status {status})")


def synthesis_tile(lib=None) -> tuple:
    """(ty, tx): coefficients per subband of one K3 work item (wv_synthesis_tile)."""
    ty, tx = C.c_int32(), C.c_int32()
    check((lib or load()).wv_synthesis_tile(C.byref(ty), C.byref(tx)), "wv_synthesis_tile")
    return ty.value, tx.value


def status_name(status: int) -> str:
    return load().wv_status_string(status).decode()

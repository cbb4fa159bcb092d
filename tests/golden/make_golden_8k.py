"""Pin parity at the benchmarked sizes by running the REAL reference
(/root/reference) on the benchmark clips.  Run in the build container (the
reference is not on the GPU boxes); takes ~10 min on 8 cores:

    python tests/golden/make_golden_8k.py

Inputs: the bench clips made by ``scripts/make_bench_input.py`` (CPU torch
restatement of the reference encoder):
  * C3/C4/C5: 8192x8192x3 stereo, L6, n 4, 256x256 mask, 4 sets, 120 fps
  * C2:       4096x2048x3 mono,   L5, n 4, 64x64 mask,  4 sets, 120 fps
They are committed xz-compressed (``bench_c3_8k.wvv.xz``,
``bench_c2.wvv.xz``) so that neither bench arm nor the GPU tests encode
anything.

Outputs (committed):
  * ``bench_8k.json``: sha256 of each clip; set 0 of the 8K clip re-encoded
    by the reference encoder (encoding.py:377-425 + fileio.py:196-237) and
    its payload/extrema sha256 (pins our encoders at 8K); per scripted
    decode call of the reference DecodeSession (fresh session per call):
    sha256 of pixels (H, W, C) u8 and of the packed footprint,
    bytes_loaded, records_processed, the PSNR over the footprint against
    the source frame (bench.py:22-30), and the fraction of the frame
    in the footprint.
  * ``bench_8k_renders.npz``: reference render_perspective (projection.py:
    111-172) per eye at 256x256 for the viewport calls (perspective parity
    on the 8K canvas geometry, +-1 LSB).
"""
from __future__ import annotations

import hashlib
import json
import lzma
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
sys.path.insert(0, REF)

import make_bench_input as mbi  # noqa: E402
from wavevid.bench import psnr as ref_psnr  # noqa: E402
from wavevid.decoding import DecodeSession, FoveationSchedule  # noqa: E402
from wavevid.encoding import EncodeParams, MappingKind, encode_video  # noqa: E402
from wavevid.fileio import VideoReader, write_video  # noqa: E402
from wavevid.projection import CameraPose, render_perspective, stereo_mask, viewport_to_mask  # noqa: E402

CACHE = "/tmp/wvb"
CLIPS = {"c3": ("bench_c3_8k.wvv.xz", "c3_8192_s4.wvv"),
         "c2": ("bench_c2.wvv.xz", "c2_4096x2048_s4.wvv")}
RENDER = 256

# (name, clip, kind, display step or frame, pose override, gaze override)
CASES = [
    ("c3_viewport_step0", "c3", "viewport", 0, None, None),
    ("c3_viewport_step37", "c3", "viewport", 37, None, None),
    ("c3_viewport_fixed_f3", "c3", "viewport", 3, (30.0, 10.0, 0.0), None),
    ("c4_foveated_step130", "c3", "foveated", 130, None, None),
    ("c4_foveated_gaze_f9", "c3", "foveated", 9, (-20.0, 5.0, 0.0), (0.3, 0.65)),
    ("c5_full_f6", "c3", "full", 6, None, None),
    ("c2_full_f1", "c2", "full", 1, None, None),
    ("c2_full_f13", "c2", "full", 13, None, None),
    ("c2_viewport_step50", "c2", "viewport", 50, None, None),
]


def sha_bytes(b) -> str:
    return hashlib.sha256(b).hexdigest()


def clip_path(cfg: str) -> str:
    xz, raw = CLIPS[cfg]
    p = os.path.join(CACHE, raw)
    if not os.path.exists(p):
        mbi.make(cfg, p)
    packed = os.path.join(HERE, xz)
    if not os.path.exists(packed):
        with open(p, "rb") as fh:
            data = fh.read()
        with open(packed, "wb") as fh:
            fh.write(lzma.compress(data, preset=9))
    return p


def case_inputs(case, header):
    name, cfg, kind, step, pose_o, gaze_o = case
    if pose_o is None:
        frame, yaw, pitch, roll, gu, gv = mbi.display_step(step, header.frame_count)
    else:
        frame, (yaw, pitch, roll), (gu, gv) = step, pose_o, (0.5, 0.5)
    if gaze_o is not None:
        gu, gv = gaze_o
    pose = CameraPose(yaw=yaw, pitch=pitch, roll=roll, fov_h=90, fov_v=90)
    dims = (header.mask_w, header.mask_h)
    mask = stereo_mask(pose, dims) if header.stereo else viewport_to_mask(pose, dims)
    return frame, (yaw, pitch, roll), (gu, gv), pose, mask


def reference_encoder_check(path: str) -> dict:
    """Set 0 of the 8K clip through the reference encoder."""
    frames = mbi.clip_frames("c3", 0).numpy()
    p = EncodeParams(alpha=0.1, inter_threshold=0.005, inter_size=4, block_size=32,
                     mapping=MappingKind.EQUIRECTANGULAR, stereo=True, fps=120.0,
                     mask_w=256, mask_h=256)
    t0 = time.perf_counter()
    video = encode_video(frames, p)
    tmp = os.path.join(CACHE, "ref_enc_c3_set0.wvv")
    write_video(video, tmp)
    el = time.perf_counter() - t0
    with VideoReader(tmp) as r_ref, VideoReader(path) as r_ours:
        m_ref = r_ref.set_meta[0]
        m_our = r_ours.set_meta[0]
        with open(tmp, "rb") as fh:
            fh.seek(m_ref.payload_offset)
            ref_payload = fh.read(m_ref.payload_length)
        with open(path, "rb") as fh:
            fh.seek(m_our.payload_offset)
            our_payload = fh.read(m_our.payload_length)
        ref_ext = np.ascontiguousarray(m_ref.extrema, np.float32).tobytes()
        our_ext = np.ascontiguousarray(m_our.extrema, np.float32).tobytes()
    out = {"payload_sha256": sha_bytes(ref_payload), "extrema_sha256": sha_bytes(ref_ext),
           "payload_bytes": len(ref_payload), "records": int(m_ref.record_count),
           "frames_sha256": sha_bytes(frames.tobytes()), "encode_s": round(el, 1),
           "bench_clip_set0_equal": ref_payload == our_payload and ref_ext == our_ext}
    print("[golden8k] reference encoder set 0:", out, flush=True)
    return out


def main():
    out = {"clips": {}, "cases": {}, "render": RENDER}
    renders = {}
    paths = {cfg: clip_path(cfg) for cfg in CLIPS}
    for cfg, p in paths.items():
        with open(p, "rb") as fh:
            out["clips"][cfg] = {"file": CLIPS[cfg][0], "sha256": sha_bytes(fh.read()),
                                 "bytes": os.path.getsize(p)}
    if "--skip-encoder" not in sys.argv:
        out["reference_encoder_set0"] = reference_encoder_check(paths["c3"])
    sources = {}
    for case in CASES:
        name, cfg, kind = case[:3]
        t0 = time.perf_counter()
        with DecodeSession(paths[cfg]) as sess:
            h = sess.header
            frame, ypr, gaze, pose, mask = case_inputs(case, h)
            if kind == "full":
                pix, fp, st = sess.decode_full(frame)
            elif kind == "viewport":
                pix, fp, st = sess.decode_viewport(frame, mask)
            else:
                pix, fp, st = sess.decode_foveated(
                    frame, mask, FoveationSchedule.default(h.levels, *gaze))
        el = time.perf_counter() - t0
        key = (cfg, frame // 4)
        if key not in sources:
            sources = {key: mbi.clip_frames(cfg, frame // 4).numpy()}
        src = sources[key][frame % 4]
        rec = {"clip": cfg, "kind": kind, "frame": frame, "pose": list(ypr), "gaze": list(gaze),
               "pixels_sha256": sha_bytes(np.ascontiguousarray(pix).tobytes()),
               "footprint_sha256": sha_bytes(np.packbits(fp).tobytes()),
               "footprint_count": int(fp.sum()),
               "bytes_loaded": int(st.bytes_loaded), "records_processed": int(st.records_processed),
               "psnr_footprint_db": (float(ref_psnr(pix[fp], src[fp])) if fp.any() else None),
               "reference_decode_s": round(el, 2)}
        if kind == "viewport":
            half = h.height // 2 if h.stereo else h.height
            for e in range(2 if h.stereo else 1):
                sl = slice(e * half, (e + 1) * half)
                renders[f"{name}|eye{e}"] = render_perspective(pix[sl], fp[sl], pose,
                                                               (RENDER, RENDER))
        out["cases"][name] = rec
        print(f"[golden8k] {name}: {el:.1f} s", rec, flush=True)
    with open(os.path.join(HERE, "bench_8k.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "bench_8k_renders.npz"), **renders)


if __name__ == "__main__":
    main()

"""Generate parity fixtures by running the REAL reference (/root/reference).

Run in the build container (the reference is not available on GPU boxes):

    python tests/golden/make_golden.py

Outputs (committed):
  * ``*.wvv``            small files encoded by the reference encoder
                          (the three golden.json files reproduce their
                          published sha256)
  * ``manifest.json``     sha256 of every file + encode parameters
  * ``decode_cases.npz``  reference DecodeSession outputs (pixels,
                          footprint, bytes_loaded, records_processed) for a
                          scripted list of decode calls per file
  * ``temporal.npz``      reference temporal_inverse_sparse planes
  * ``projection.npz``    reference viewport_to_mask / stereo_mask /
                          render_perspective outputs
  * ``synthetic.json``    sha256 of reference make_synthetic_clip outputs
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from wavevid.bench import make_synthetic_clip  # noqa: E402
from wavevid.decoding import (DecodeSession, FoveationSchedule,  # noqa: E402
                              temporal_inverse_sparse)
from wavevid.encoding import EncodeParams, MappingKind, encode_video  # noqa: E402
from wavevid.fileio import VideoReader, write_video  # noqa: E402
from wavevid.projection import (CameraPose, CoverageError,  # noqa: E402
                                render_perspective, stereo_mask,
                                viewport_to_mask)


def sha(path):
    return hashlib.sha256(open(path, "rb").read()).hexdigest()


def noise(seed, frames, size, channels):
    return np.random.default_rng(seed).integers(
        0, 256, (frames, size, size, channels), dtype=np.uint8)


# file name -> (clip factory, encode params)
FILES = {
    # the three frozen files of pkg/tests/data/golden.json
    "golden_quantized.wvv": (lambda: noise(11, 4, 64, 3),
                             dict(alpha=0.1, inter_threshold=0.005, levels=2,
                                  mapping="NONE")),
    "golden_float.wvv": (lambda: noise(12, 2, 64, 1),
                         dict(alpha=0.0, inter_threshold=0.0, quantize=False,
                              levels=2, inter_size=2, mapping="NONE")),
    "golden_stereo.wvv": (lambda: noise(13, 4, 128, 3),
                          dict(alpha=0.25, inter_threshold=0.005, levels=3,
                               stereo=True, mapping="EQUIRECTANGULAR",
                               fps=60.0)),
    # conftest.py quantized_file / lossless_file equivalents
    "smooth_hq.wvv": (lambda: make_synthetic_clip(frames=8, size=128),
                      dict(alpha=0.1, inter_threshold=0.005, levels=3,
                           mapping="NONE")),
    "smooth_lossless.wvv": (lambda: make_synthetic_clip(frames=4, size=64),
                            dict(alpha=0.0, inter_threshold=0.0,
                                 quantize=False, levels=3, mapping="NONE")),
    # 16-px blocks, dense records (test_decoding.py big_file, shrunk)
    "noise_bs16.wvv": (lambda: noise(5, 4, 128, 3),
                       dict(alpha=0.3, inter_threshold=0.01, levels=4,
                            block_size=16, mapping="NONE")),
    # temporal depth n=8 and n=1, equirect mapping, padded last set
    "smooth_n8.wvv": (lambda: make_synthetic_clip(frames=10, size=64),
                      dict(alpha=0.1, inter_threshold=0.005, levels=2,
                           inter_size=8)),
    "smooth_n1_mono.wvv": (lambda: make_synthetic_clip(frames=3, size=64,
                                                      channels=1),
                           dict(alpha=0.05, inter_threshold=0.0, levels=3,
                                inter_size=1)),
    # non-square frame with 64x32 mask grid (equirect 2:1)
    "wide_equirect.wvv": (lambda: make_synthetic_clip(frames=4, size=128)[:, :64],
        dict(alpha=0.1, inter_threshold=0.005, levels=3, mask_w=64,
             mask_h=32)),
}


def params_of(spec):
    p = dict(spec)
    p["mapping"] = MappingKind[p.get("mapping", "EQUIRECTANGULAR")]
    return EncodeParams(**p)


def rect_mask(h, w, y, x, hh, ww):
    m = np.zeros((h, w), bool)
    m[y:y + hh, x:x + ww] = True
    return m


def decode_script(name, header):
    """List of (kind, frame, mask, schedule-args) decode calls per file,
    executed in order on ONE session (so cache/bytes semantics are pinned)."""
    mh, mw = header.mask_h, header.mask_w
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    calls = []
    nf = header.frame_count
    calls.append(("full", 0, None, None))
    calls.append(("full", nf - 1, None, None))
    for i in range(6):
        hh, ww = rng.integers(2, max(3, mh // 2)), rng.integers(2, max(3, mw // 2))
        y, x = rng.integers(0, mh - hh + 1), rng.integers(0, mw - ww + 1)
        calls.append(("viewport", int(rng.integers(0, nf)),
                      rect_mask(mh, mw, y, x, hh, ww), None))
    calls.append(("viewport", 0, np.zeros((mh, mw), bool), None))
    calls.append(("viewport", 1 % nf, rng.random((mh, mw)) < 0.05, None))
    for pose in [dict(yaw=30, pitch=10), dict(yaw=-100, pitch=-40, roll=5),
                 dict(yaw=170, pitch=60)]:
        cp = CameraPose(fov_h=90, fov_v=90, **pose)
        mk = (stereo_mask(cp, (mw, mh)) if header.stereo
              else viewport_to_mask(cp, (mw, mh)))
        calls.append(("viewport", int(rng.integers(0, nf)), mk, None))
        calls.append(("foveated", int(rng.integers(0, nf)), mk,
                      (None, float(rng.uniform(0, 1)), float(rng.uniform(0, 1)))))
    big = rect_mask(mh, mw, mh // 8, mw // 8, 3 * mh // 4, 3 * mw // 4)
    calls.append(("foveated", 0, big, (None, 0.5, 0.5)))
    calls.append(("foveated", 0, big, (tuple([1.0] * (header.levels + 1)), 0.5, 0.5)))
    calls.append(("foveated", nf - 1, big, ((1.0, 0.5), 0.2, 0.9)))
    # growing masks inside one set, then revisit (bytes bookkeeping)
    small = rect_mask(mh, mw, mh // 3, mw // 3, max(1, mh // 6), max(1, mw // 6))
    calls.append(("viewport", 0, small, None))
    calls.append(("viewport", 0, big, None))
    calls.append(("viewport", 0, small, None))
    return calls


def main():
    manifest = {}
    cases = {}
    for name, (clip_fn, spec) in FILES.items():
        path = os.path.join(HERE, name)
        clip = clip_fn()
        write_video(encode_video(clip, params_of(spec)), path)
        manifest[name] = {"sha256": sha(path), "params": spec,
                          "clip_shape": list(clip.shape)}
        with DecodeSession(path) as s:
            h = s.header
            for i, (kind, frame, mask, sched) in enumerate(decode_script(name, h)):
                key = f"{name}|{i}"
                if kind == "full":
                    pix, fp, st = s.decode_full(frame)
                elif kind == "viewport":
                    pix, fp, st = s.decode_viewport(frame, mask)
                else:
                    fr, gu, gv = sched
                    sc = (FoveationSchedule.default(h.levels, gu, gv) if fr is None
                          else FoveationSchedule(fr, gu, gv))
                    pix, fp, st = s.decode_foveated(frame, mask, sc)
                    cases[key + "|fractions"] = np.array(sc.fractions)
                    cases[key + "|gaze"] = np.array([gu, gv])
                cases[key + "|kind"] = np.array(kind)
                cases[key + "|frame"] = np.array(frame)
                if mask is not None:
                    cases[key + "|mask"] = np.packbits(mask)
                cases[key + "|pixels"] = pix
                cases[key + "|footprint"] = np.packbits(fp)
                cases[key + "|stats"] = np.array([st.bytes_loaded,
                                                  st.records_processed])
        print(name, manifest[name]["sha256"][:16])
    np.savez_compressed(os.path.join(HERE, "decode_cases.npz"), **cases)

    # temporal planes (decoding.py:53-90) straight from the reference
    tplanes = {}
    for name in ("golden_quantized.wvv", "golden_float.wvv", "smooth_n8.wvv",
                 "noise_bs16.wvv"):
        with VideoReader(os.path.join(HERE, name)) as r:
            h = r.header
            recs, _ = r.load_all(0)
            for t in range(h.inter_size):
                pyr = temporal_inverse_sparse(
                    recs, r.set_meta[0].extrema, t, h.width, h.height,
                    h.levels, h.inter_size, h.block_size, h.channels)
                tplanes[f"{name}|{t}"] = pyr.data
    np.savez_compressed(os.path.join(HERE, "temporal.npz"), **tplanes)

    # projection: masks for poses and perspective renders of decoded canvases
    proj = {}
    rng = np.random.default_rng(42)
    poses = [CameraPose(yaw=30, pitch=10), CameraPose(yaw=0, pitch=0),
             CameraPose(pitch=90), CameraPose(fov_h=360, fov_v=180)]
    for _ in range(12):
        poses.append(CameraPose(yaw=rng.uniform(-180, 180),
                                pitch=rng.uniform(-85, 85),
                                roll=rng.uniform(-25, 25),
                                fov_h=rng.uniform(60, 120),
                                fov_v=rng.uniform(60, 120)))
    for i, p in enumerate(poses):
        proj[f"pose|{i}"] = np.array([p.yaw, p.pitch, p.roll, p.fov_h, p.fov_v])
        for dims in ((64, 64), (48, 48), (64, 32), (256, 256)):
            proj[f"vmask|{i}|{dims[0]}x{dims[1]}"] = np.packbits(
                viewport_to_mask(p, dims))
            proj[f"smask|{i}|{dims[0]}x{dims[1]}"] = np.packbits(
                stereo_mask(p, dims))
    for fname in ("smooth_hq.wvv", "golden_stereo.wvv"):
        with DecodeSession(os.path.join(HERE, fname)) as s:
            h = s.header
            for i, p in enumerate(poses[:10]):
                if not (p.fov_h < 180 and p.fov_v < 180):
                    continue
                if h.stereo:
                    mk = stereo_mask(p, (h.mask_w, h.mask_h))
                else:
                    mk = viewport_to_mask(p, (h.mask_w, h.mask_h))
                pix, fp, _ = s.decode_viewport(i % h.frame_count, mk)
                eyes = [(pix, fp)] if not h.stereo else [
                    (pix[: h.height // 2], fp[: h.height // 2]),
                    (pix[h.height // 2:], fp[h.height // 2:])]
                for e, (reg, f) in enumerate(eyes):
                    try:
                        out = render_perspective(reg, f, p, (40, 24))
                        proj[f"persp|{fname}|{i}|{e}"] = out
                    except CoverageError:
                        proj[f"persp|{fname}|{i}|{e}"] = np.array("coverage")
    np.savez_compressed(os.path.join(HERE, "projection.npz"), **proj)

    synth = {}
    for args in [(8, 128, 3, 7), (3, 64, 1, 7), (4, 128, 3, 9), (2, 256, 3, 7)]:
        clip = make_synthetic_clip(*args)
        synth["x".join(map(str, args))] = hashlib.sha256(clip.tobytes()).hexdigest()
    with open(os.path.join(HERE, "synthetic.json"), "w") as fh:
        json.dump(synth, fh, indent=1)
    with open(os.path.join(HERE, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1)


if __name__ == "__main__":
    main()

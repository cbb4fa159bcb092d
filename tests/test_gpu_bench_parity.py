"""Parity at the benchmarked configurations: the bench's own
committed clips (C3/C4/C5 8192x8192 stereo L6, C2 4096x2048 RGB L5)
decoded on the GPU and compared with outputs of the REAL reference decoder
run on the same files (tests/golden/make_golden_8k.py -> bench_8k.json):
pixels (sha256 of the (H, W, C) u8 array), footprint (sha256 of the packed
bool array), bytes_loaded and records_processed, all exact; PSNR against
the source frame equal to 0.01 dB; per-eye perspective renders of the 8K
canvas within +-1 LSB of the reference's render_perspective.  The 8K CUDA
encoder is pinned to the reference encoder's set-0 sha256 and the numpy
oracle is pinned at 8K on one viewport frame."""
import hashlib
import json
import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

sys.path.insert(0, os.path.join(ROOT, "scripts"))
import make_bench_input as mbi  # noqa: E402

pytestmark = pytest.mark.gpu

CACHE = os.environ.get("WV_BENCH_CACHE", "/tmp/wvb200_bench")


@pytest.fixture(scope="module")
def fixture():
    with open(os.path.join(GOLDEN, "bench_8k.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def wv():
    import paper_2208_10859_b200 as p
    from paper_2208_10859_b200 import build
    build.build()
    return p


def _sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _inputs(wv, rec, h):
    pose = wv.CameraPose(yaw=rec["pose"][0], pitch=rec["pose"][1], roll=rec["pose"][2],
                         fov_h=90, fov_v=90)
    dims = (h.mask_w, h.mask_h)
    mask = wv.stereo_mask(pose, dims) if h.stereo else wv.viewport_to_mask(pose, dims)
    return pose, mask


def _decode(wv, sess, rec, mask):
    if rec["kind"] == "full":
        return sess.decode_full(rec["frame"])
    if rec["kind"] == "viewport":
        return sess.decode_viewport(rec["frame"], mask)
    sc = wv.FoveationSchedule.default(sess.header.levels, *rec["gaze"])
    return sess.decode_foveated(rec["frame"], mask, sc)


CASES = ["c3_viewport_step0", "c3_viewport_step37", "c3_viewport_fixed_f3",
         "c4_foveated_step130", "c4_foveated_gaze_f9", "c5_full_f6",
         "c2_full_f1", "c2_full_f13", "c2_viewport_step50"]


# the 56-column synthesis tiles (tile_strips=2, the full-frame bench's
# sessions) on every kind of case
WIDE = ["c3_viewport_step37", "c4_foveated_gaze_f9", "c5_full_f6", "c2_full_f13"]


@pytest.mark.parametrize("name,strips", [(n, 1) for n in CASES] + [(n, 2) for n in WIDE])
def test_bench_clip_decode_equals_reference(wv, fixture, name, strips):
    """GPU decode of the benchmarked clip == the reference decoder, bit for
    bit (pixels, footprint, stats); fresh session as in the fixture."""
    rec = fixture["cases"][name]
    path = mbi.ensure_clip(rec["clip"], CACHE)
    with wv.DecodeSession(path, device="cuda:0", tile_strips=strips) as sess:
        h = sess.header
        pose, mask = _inputs(wv, rec, h)
        pix, fp, st = _decode(wv, sess, rec, mask)
        assert (st.bytes_loaded, st.records_processed) == (rec["bytes_loaded"],
                                                           rec["records_processed"])
        assert int(fp.sum()) == rec["footprint_count"]
        assert _sha(np.packbits(fp)) == rec["footprint_sha256"], "footprint differs"
        assert _sha(pix) == rec["pixels_sha256"], "pixels differ from the reference"
        if rec["kind"] == "viewport":
            # per-eye writeout of the 8K canvas vs the reference render (+-1 LSB)
            want = np.load(os.path.join(GOLDEN, "bench_8k_renders.npz"))
            R = fixture["render"]
            out = sess.render_views(pose, (R, R)).cpu().numpy()
            for e in range(2 if h.stereo else 1):
                ref = want[f"{name}|eye{e}"]
                d = np.abs(out[e].astype(np.int16) - ref.astype(np.int16))
                assert d.max() <= 1, f"eye {e}: max diff {d.max()}"


@pytest.mark.parametrize("name", ["c5_full_f6", "c2_full_f1"])
def test_bench_clip_psnr_equals_reference(wv, fixture, name):
    """PSNR of the GPU decode against the source frame (bench.py:22-30)
    equal to the reference's within 0.01 dB."""
    from paper_2208_10859_b200.synthetic import make_synthetic_clip_torch, psnr
    rec = fixture["cases"][name]
    cfg = rec["clip"]
    w, hh, _, n_sets, _ = mbi.CONFIGS[cfg]
    src = make_synthetic_clip_torch(1, hh, w, 3, seed=7, device="cpu", first_frame=rec["frame"],
                                    total_frames=4 * n_sets)[0].numpy()
    path = mbi.ensure_clip(cfg, CACHE)
    with wv.DecodeSession(path, device="cuda:0") as sess:
        pix, fp, _ = sess.decode_full(rec["frame"])
    assert abs(psnr(pix[fp], src[fp]) - rec["psnr_footprint_db"]) < 0.01


def test_bench_clip_oracle_pinned_at_8k(fixture):
    """The numpy oracle (the checker of every other GPU test) reproduces the
    reference decoder at 8K too."""
    from oracle import wavevid_oracle as wo
    import paper_2208_10859_b200 as wv
    rec = fixture["cases"]["c3_viewport_step37"]
    path = mbi.ensure_clip("c3", CACHE)
    sess = wo.OracleSession(path)
    _, mask = _inputs(wv, rec, sess.header)
    pix, fp, st = sess.decode(rec["frame"], "viewport", mask)
    assert (st.bytes_loaded, st.records_processed) == (rec["bytes_loaded"],
                                                       rec["records_processed"])
    assert _sha(np.packbits(fp)) == rec["footprint_sha256"]
    assert _sha(pix) == rec["pixels_sha256"]


def test_cuda_encoder_equals_reference_encoder_at_8k(wv, fixture):
    """Set 0 of the 8K clip re-encoded by the CUDA encoder (the bench's
    input generator) is byte-identical to the reference encoder's set 0."""
    import torch
    ref = fixture["reference_encoder_set0"]
    frames = mbi.clip_frames("c3", 0)
    assert _sha(frames.numpy()) == ref["frames_sha256"]
    v = wv.encode_video(frames.to("cuda:0"), mbi.params_for("c3"), device="cuda:0",
                        keep_arrays=False)
    tmp = os.path.join(CACHE, "enc_check.wvv")
    os.makedirs(CACHE, exist_ok=True)
    v.frame_count, v.pad_frames = 4, 0
    wv.write_video(v, tmp)
    with wv.VideoReader(tmp) as r:
        m = r.set_meta[0]
        with open(tmp, "rb") as fh:
            fh.seek(m.payload_offset)
            payload = fh.read(m.payload_length)
        ext = np.ascontiguousarray(m.extrema, np.float32).tobytes()
    torch.cuda.synchronize()
    assert hashlib.sha256(payload).hexdigest() == ref["payload_sha256"]
    assert hashlib.sha256(ext).hexdigest() == ref["extrema_sha256"]

"""Pin the CPU oracle against fixtures produced by the real reference.

Every decode call the reference made in tests/golden/make_golden.py is
replayed on one OracleSession per file, in the same order, and must match
bit for bit: u8 pixels, footprint, bytes_loaded, records_processed.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, case_calls, unpack_mask
from oracle import wavevid_oracle as wo

FILES = ["golden_quantized.wvv", "golden_float.wvv", "golden_stereo.wvv",
         "smooth_hq.wvv", "smooth_lossless.wvv", "noise_bs16.wvv",
         "smooth_n8.wvv", "smooth_n1_mono.wvv", "wide_equirect.wvv"]


@pytest.mark.parametrize("name", FILES)
def test_fixture_files_unchanged(manifest, name):
    digest = hashlib.sha256(open(os.path.join(GOLDEN, name), "rb").read()).hexdigest()
    assert digest == manifest[name]["sha256"]


def test_published_golden_digests(manifest):
    # pkg/tests/data/golden.json:3,41,81 (the reference's frozen files)
    assert manifest["golden_quantized.wvv"]["sha256"].startswith("798cf686c201")
    assert manifest["golden_float.wvv"]["sha256"].startswith("83f78953c069")
    assert manifest["golden_stereo.wvv"]["sha256"].startswith("8618e871a4bf")


@pytest.mark.parametrize("name", FILES)
def test_oracle_replays_reference_decodes(decode_cases, name):
    sess = wo.OracleSession(os.path.join(GOLDEN, name))
    h = sess.header
    calls = case_calls(decode_cases, name)
    assert calls
    for i, c in enumerate(calls):
        mask = None
        if c["mask_packed"] is not None:
            mask = unpack_mask(c["mask_packed"], (h.mask_h, h.mask_w))
        kw = {}
        if c["kind"] == "foveated":
            kw = dict(fractions=c["fractions"], gaze=c["gaze"])
        pix, fp, st = sess.decode(c["frame"], c["kind"], mask, **kw)
        want_fp = unpack_mask(c["footprint"], (h.height, h.width))
        np.testing.assert_array_equal(pix, c["pixels"], err_msg=f"call {i}")
        np.testing.assert_array_equal(fp, want_fp, err_msg=f"call {i}")
        assert (st.bytes_loaded, st.records_processed) == c["stats"], i


@pytest.mark.parametrize("name", ["golden_quantized.wvv", "smooth_hq.wvv",
                                  "golden_stereo.wvv"])
def test_full_synthesis_equals_windowed(decode_cases, name):
    """windowed synthesis == full synthesis of the masked
    pyramid inside the request; the GPU tiling relies on it."""
    a = wo.OracleSession(os.path.join(GOLDEN, name))
    b = wo.OracleSession(os.path.join(GOLDEN, name), full_synthesis=True)
    h = a.header
    for c in case_calls(decode_cases, name):
        mask = None
        if c["mask_packed"] is not None:
            mask = unpack_mask(c["mask_packed"], (h.mask_h, h.mask_w))
        kw = {}
        if c["kind"] == "foveated":
            kw = dict(fractions=c["fractions"], gaze=c["gaze"])
        pa, fa, _ = a.decode(c["frame"], c["kind"], mask, **kw)
        pb, fb, _ = b.decode(c["frame"], c["kind"], mask, **kw)
        np.testing.assert_array_equal(pa, pb)


def test_temporal_planes_match_reference():
    want = np.load(os.path.join(GOLDEN, "temporal.npz"))
    names = sorted({k.split("|")[0] for k in want.files})
    for name in names:
        hd, sets = wo.read_file(os.path.join(GOLDEN, name))
        blocks = np.arange(hd.num_blocks)
        for t in range(hd.inter_size):
            got = wo.temporal_plane(hd, sets[0], blocks, t)
            ref = want[f"{name}|{t}"]
            # bitwise, including the sign of zero
            assert got.dtype == ref.dtype == np.float32
            np.testing.assert_array_equal(got.view(np.uint32), ref.view(np.uint32))


def _dense_haar_inverse(coeffs):
    """Independent dense inverse (encoding.py:172-184 semantics)."""
    cur = [coeffs[0]]
    start = 1
    while start < len(coeffs):
        det = coeffs[start:2 * start]
        cur = [v for a, d in zip(cur, det) for v in (a + d, a - d)]
        start *= 2
    return cur


def test_haar_series_known_answer():
    # test_decoding.py:56-60: approx 5, level-2 detail -2, level-1 detail +1
    w = wo.temporal_weights(0, 4)
    assert float(np.dot(w, [5.0, -2.0, 1.0, 0.0])) == 4.0
    rng = np.random.default_rng(0)
    for n in (1, 2, 4, 8, 16):
        c = list(rng.integers(-9, 9, n).astype(float))
        dense = _dense_haar_inverse(c)
        for t in range(n):
            w = wo.temporal_weights(t, n)
            assert float(np.dot(w, c)) == dense[t]
            assert int((w != 0).sum()) == n.bit_length()


def test_perspective_matches_reference():
    want = np.load(os.path.join(GOLDEN, "projection.npz"))
    for fname in ("smooth_hq.wvv", "golden_stereo.wvv"):
        sess = wo.OracleSession(os.path.join(GOLDEN, fname))
        h = sess.header
        keys = [k for k in want.files if k.startswith(f"persp|{fname}|")]
        assert keys
        done = set()
        for k in keys:
            _, _, i, e = k.split("|")
            i, e = int(i), int(e)
            if (i, e) in done:
                continue
            done.add((i, e))
            yaw, pitch, roll, fh, fv = want[f"pose|{i}"]
            dims = (h.mask_w, h.mask_h)
            mk = unpack_mask(want[f"{'smask' if h.stereo else 'vmask'}|{i}|"
                                  f"{dims[0]}x{dims[1]}"], (h.mask_h, h.mask_w)) \
                if f"{'smask' if h.stereo else 'vmask'}|{i}|{dims[0]}x{dims[1]}" in want.files \
                else None
            if mk is None:
                continue
            pix, fp, _ = sess.decode(i % h.frame_count, "viewport", mk)
            if h.stereo:
                half = h.height // 2
                reg, f = (pix[:half], fp[:half]) if e == 0 else (pix[half:], fp[half:])
            else:
                reg, f = pix, fp
            rot = wo.pose_rotation(yaw, pitch, roll)
            ref = want[k]
            if ref.dtype.kind == "U":
                with pytest.raises(wo.Uncovered):
                    wo.perspective(reg, f, rot, fh, fv, 40, 24)
            else:
                got = wo.perspective(reg, f, rot, fh, fv, 40, 24)
                np.testing.assert_array_equal(got, ref)

"""GPU decode path: perspective parity, reference-suite behaviours
(pkg/tests/test_decoding.py, test_acceptance.py, test_projection.py) and
larger-frame parity against the CPU oracle."""
import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN, unpack_mask
from oracle import wavevid_oracle as wo

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wv():
    import paper_2208_10859_b200 as p
    from paper_2208_10859_b200 import build
    build.build()
    return p


@pytest.fixture(scope="module")
def clip512():
    from paper_2208_10859_b200.synthetic import make_synthetic_clip
    return make_synthetic_clip(16, 512)


@pytest.fixture(scope="module")
def hq512(wv, clip512, tmp_path_factory):
    """test_acceptance.py hq_file: 512^2, 16 frames, L5, HQ params."""
    path = tmp_path_factory.mktemp("acc") / "hq.wvv"
    p = wv.EncodeParams(levels=5, mapping=wv.MappingKind.NONE, alpha=0.1, inter_threshold=0.005)
    wv.write_video(wv.encode_video(clip512, p), path)
    return path


# ------------------------------------------------------------ perspective

def test_perspective_matches_reference_fixtures(wv):
    want = np.load(os.path.join(GOLDEN, "projection.npz"))
    for fname in ("smooth_hq.wvv", "golden_stereo.wvv"):
        sess = wv.DecodeSession(os.path.join(GOLDEN, fname))
        h = sess.header
        done = set()
        for k in sorted(k for k in want.files if k.startswith(f"persp|{fname}|")):
            _, _, i, e = k.split("|")
            i, e = int(i), int(e)
            yaw, pitch, roll, fh, fv = want[f"pose|{i}"]
            pose = wv.CameraPose(float(yaw), float(pitch), float(roll), float(fh), float(fv))
            key = f"{'smask' if h.stereo else 'vmask'}|{i}|{h.mask_w}x{h.mask_h}"
            mk = unpack_mask(want[key], (h.mask_h, h.mask_w))
            if (i, 0) not in done:
                pix, fp, _ = sess.decode_viewport(i % h.frame_count, mk)
                done.add((i, 0))
            half = h.height // 2 if h.stereo else h.height
            reg, f = pix[e * half:(e + 1) * half], fp[e * half:(e + 1) * half]
            ref = want[k]
            if ref.dtype.kind == "U":
                with pytest.raises(wv.CoverageError):
                    wv.render_perspective(reg, f, pose, (40, 24))
            else:
                got = wv.render_perspective(reg, f, pose, (40, 24))
                d = np.abs(got.astype(int) - ref.astype(int))
                assert d.max() <= 1, (fname, i, e, d.max())
        sess.close()


def test_perspective_against_oracle_random_poses(wv):
    rng = np.random.default_rng(5)
    region = rng.integers(0, 256, (256, 512, 3), dtype=np.uint8)
    fp = np.ones((256, 512), bool)
    for _ in range(25):
        pose = wv.CameraPose(yaw=rng.uniform(-180, 180), pitch=rng.uniform(-89, 89),
                             roll=rng.uniform(-30, 30), fov_h=rng.uniform(30, 150),
                             fov_v=rng.uniform(30, 150))
        got = wv.render_perspective(region, fp, pose, (97, 61))
        ref = wo.perspective(region, fp, pose.rotation(), pose.fov_h, pose.fov_v, 97, 61)
        assert np.abs(got.astype(int) - ref.astype(int)).max() <= 1


def test_perspective_coverage_matches_oracle(wv):
    """Partial footprints: CoverageError exactly when the oracle raises."""
    rng = np.random.default_rng(9)
    region = rng.integers(0, 256, (128, 256, 3), dtype=np.uint8)
    for _ in range(30):
        fp = np.zeros((128, 256), bool)
        y, x = rng.integers(0, 100), rng.integers(0, 220)
        fp[y:y + rng.integers(10, 128), x:x + rng.integers(10, 256)] = True
        pose = wv.CameraPose(yaw=rng.uniform(-180, 180), pitch=rng.uniform(-60, 60),
                             fov_h=rng.uniform(20, 90), fov_v=rng.uniform(20, 90))
        try:
            ref = wo.perspective(region, fp, pose.rotation(), pose.fov_h, pose.fov_v, 48, 32)
        except wo.Uncovered:
            with pytest.raises(wv.CoverageError):
                wv.render_perspective(region, fp, pose, (48, 32))
            continue
        got = wv.render_perspective(region, fp, pose, (48, 32))
        assert np.abs(got.astype(int) - ref.astype(int)).max() <= 1


def test_perspective_constant_and_identity(wv):
    # test_projection.py:139-155
    region = np.full((128, 256, 3), 77, np.uint8)
    fp = np.ones((128, 256), bool)
    out = wv.render_perspective(region, fp, wv.CameraPose(yaw=12, pitch=-5), (64, 64))
    assert (out == 77).all()
    region = np.zeros((128, 256, 3), np.uint8)
    region[63:65, 127:129] = (200, 10, 30)
    out = wv.render_perspective(region, fp, wv.CameraPose(), (65, 65))
    assert tuple(out[32, 32]) == (200, 10, 30)


def test_perspective_errors(wv):
    region = np.zeros((64, 128), np.uint8)
    with pytest.raises(wv.ProjectionError):
        wv.render_perspective(region, np.ones((64, 128), bool), wv.CameraPose(fov_h=180), (32, 32))
    with pytest.raises(wv.CoverageError):
        wv.render_perspective(np.zeros((64, 128, 3), np.uint8), np.zeros((64, 128), bool),
                              wv.CameraPose(), (16, 16))


def test_hundred_random_poses_covered(wv):
    # test_projection.py:159-176 on the conftest quantized file
    rng = np.random.default_rng(42)
    sess = wv.DecodeSession(os.path.join(GOLDEN, "smooth_hq.wvv"))
    h = sess.header
    for _ in range(100):
        pose = wv.CameraPose(yaw=rng.uniform(-180, 180), pitch=rng.uniform(-85, 85),
                             roll=rng.uniform(-10, 10), fov_h=rng.uniform(60, 120),
                             fov_v=rng.uniform(60, 120))
        mask = wv.viewport_to_mask(pose, (h.mask_w, h.mask_h))
        sess.decode_viewport_device(0, mask)
        sess.render_views(pose, (32, 32))       # raises CoverageError if not covered
    sess.close()


# --------------------------------------------------- reference behaviours

def test_roi_exactness_hundred_masks(wv, hq512):
    """test_acceptance.py:96-117, plus every pixel == oracle."""
    rng = np.random.default_rng(99)
    full, _, _ = wv.DecodeSession(hq512).decode_full(3)
    sess = wv.DecodeSession(hq512)
    ref = wo.OracleSession(hq512)
    for i in range(100):
        mask = np.zeros((64, 64), bool)
        w, h = rng.integers(4, 40, 2)
        x, y = rng.integers(0, 64 - w), rng.integers(0, 64 - h)
        mask[y:y + h, x:x + w] = True
        pix, fp, st = sess.decode_viewport(3, mask)
        assert (pix[fp] == full[fp]).all()
        rp, rf, rs = ref.decode(3, "viewport", mask)     # same call history: same stats
        assert (st.bytes_loaded, st.records_processed) == (rs.bytes_loaded, rs.records_processed)
        if i % 10 == 0:
            np.testing.assert_array_equal(pix, rp)
            np.testing.assert_array_equal(fp, rf)


def test_quantized_psnr_and_oracle_psnr_equal(wv, clip512, hq512):
    """PSNR >= 40 dB (test_acceptance.py:84-93) and identical to the oracle's
    PSNR to 0.01 dB (north-star parity bar)."""
    sess = wv.DecodeSession(hq512)
    ref = wo.OracleSession(hq512)
    for f in (0, 8, 15):
        pix, _, _ = sess.decode_full(f)
        rp, _, _ = ref.decode(f, "full")
        a, b = wv.psnr(pix, clip512[f]), wv.psnr(rp, clip512[f])
        assert a >= 40.0 and abs(a - b) < 0.01


def test_lossless_path(wv, clip512, tmp_path):
    path = tmp_path / "lossless.wvv"
    p = wv.EncodeParams(levels=5, mapping=wv.MappingKind.NONE, alpha=0.0, inter_threshold=0.0,
                        quantize=False)
    wv.write_video(wv.encode_video(clip512, p), path)
    sess = wv.DecodeSession(path)
    for f in (0, 7, 15):
        pix, _, _ = sess.decode_full(f)
        assert np.abs(pix.astype(int) - clip512[f].astype(int)).max() <= 1
        assert wv.psnr(pix, clip512[f]) >= 60.0


def test_foveation_savings(wv, hq512):
    # test_acceptance.py:183-197
    pose = wv.CameraPose(yaw=30, pitch=10, fov_h=90, fov_v=90)
    mask = wv.viewport_to_mask(pose, (64, 64))
    _, _, vs = wv.DecodeSession(hq512).decode_viewport(0, mask)
    s = wv.DecodeSession(hq512)
    _, _, fs = s.decode_foveated(0, mask, wv.FoveationSchedule.default(s.header.levels))
    assert 1.0 - fs.bytes_loaded / vs.bytes_loaded >= 0.5


def test_keyframe_freedom_and_cache(wv, hq512):
    mask = np.ones((64, 64), bool)
    sess = wv.DecodeSession(hq512)
    n = sess.header.inter_size
    for frame in [13, 2, 9, 0, 15, 6]:
        before = len(sess.reader.io_trace)
        sess.decode_viewport(frame, mask)
        assert {e[0] for e in sess.reader.io_trace[before:]} <= {frame // n}
    sess2 = wv.DecodeSession(hq512)
    for frame in (0, 4, 0, 4, 0):
        sess2.decode_viewport(frame, mask)
        assert len(sess2._cache) <= 2


def test_stats_monotone_and_errors(wv):
    path = os.path.join(GOLDEN, "smooth_hq.wvv")
    mask = np.zeros((64, 64), bool)
    mask[10:50, 10:50] = True
    with wv.DecodeSession(path) as s:
        seen = []
        for frame in range(4):
            s.decode_viewport(frame, mask)
            st = s.stats
            seen.append((st.bytes_loaded, st.records_processed, st.frames_decoded))
        assert seen == sorted(seen)
        with pytest.raises(wv.DecodeError):
            s.decode_viewport(0, np.ones((32, 32), bool))
        with pytest.raises(wv.DecodeError):
            s.decode_full(99)
        with pytest.raises(wv.DecodeError):
            wv.FoveationSchedule((1.0, 0.2, 0.5))


def test_prefetch_mask_enlarged(wv):
    # test_decoding.py:233-247
    path = os.path.join(GOLDEN, "smooth_hq.wvv")
    small = np.zeros((64, 64), bool)
    small[24:40, 24:40] = True
    large = np.zeros((64, 64), bool)
    large[8:56, 8:56] = True
    with wv.DecodeSession(path) as s:
        s.decode_viewport(0, small)
        s.advance(0, small)
        s.join_prefetch()
        grown, gf, gs = s.decode_viewport(4, large)
    with wv.DecodeSession(path) as f:
        want, wf, ws = f.decode_viewport(4, large)
    np.testing.assert_array_equal(gf, wf)
    np.testing.assert_array_equal(grown, want)
    # the prefetched blocks were already accounted in the set's cache entry
    assert gs.bytes_loaded <= ws.bytes_loaded


def test_corrupt_offset_raises(wv, tmp_path):
    src = os.path.join(GOLDEN, "golden_quantized.wvv")
    dst = tmp_path / "corrupt.wvv"
    shutil.copy(src, dst)
    raw = bytearray(open(dst, "rb").read())
    from paper_2208_10859_b200.fileio import read_header
    h, metas = read_header(src)
    rec0 = metas[0].payload_offset + h.table_bytes
    raw[rec0:rec0 + 2] = (0xFFFF).to_bytes(2, "little")   # offset 65535 >= 32*32
    open(dst, "wb").write(bytes(raw))
    with wv.DecodeSession(dst) as s:
        with pytest.raises(wv.CorruptStreamError):
            s.decode_full(0)


@pytest.mark.parametrize("mode", ["full", "viewport"])
def test_blockend_past_payload_raises(wv, tmp_path, mode):
    """A BlockEnd entry pointing past the set payload is a corrupt stream:
    K2 and the span fetch skip the span (no out-of-bounds read) and the
    decode raises CorruptStreamError; the session stays usable."""
    src = os.path.join(GOLDEN, "golden_quantized.wvv")
    dst = tmp_path / "corrupt_table.wvv"
    shutil.copy(src, dst)
    raw = bytearray(open(dst, "rb").read())
    from paper_2208_10859_b200.fileio import read_header
    h, metas = read_header(src)
    t0 = metas[0].payload_offset
    raw[t0 + 8 * 5:t0 + 8 * 6] = (1 << 40).to_bytes(8, "little")   # (t=0, block 5) end
    open(dst, "wb").write(bytes(raw))
    mask = np.ones((h.mask_h, h.mask_w), bool)
    for residency in ("set", "spans"):
        with wv.DecodeSession(dst, residency=residency) as s:
            with pytest.raises(wv.CorruptStreamError):
                s.decode_full(0) if mode == "full" else s.decode_viewport(0, mask)
            # the context is intact: a good file still decodes afterwards
        with wv.DecodeSession(src) as s:
            s.decode_full(1)


# ------------------------------------------------------ larger frames

@pytest.mark.parametrize("mode", ["viewport", "foveated", "full"])
def test_stereo_2048_vs_oracle(wv, tmp_path_factory, mode):
    """8K-shaped path at 2048^2 stereo (L4, 256^2 mask grid): GPU == oracle."""
    import torch
    d = tmp_path_factory.mktemp("s2048")
    path = d / "s.wvv"
    if not path.exists():
        from paper_2208_10859_b200.synthetic import make_synthetic_clip_torch
        clip = make_synthetic_clip_torch(4, 2048, 2048, 3, device="cuda")
        p = wv.EncodeParams(stereo=True, fps=120.0, mask_w=256, mask_h=256)
        wv.write_video(wv.encode_video(clip, p, device="cuda"), path)
    sess = wv.DecodeSession(path)
    ref = wo.OracleSession(path)
    h = sess.header
    pose = wv.CameraPose(yaw=30, pitch=10)
    mask = wv.stereo_mask(pose, (h.mask_w, h.mask_h))
    for frame in (0, 2):
        if mode == "full":
            pix, fp, st = sess.decode_full(frame)
            rp, rf, rs = ref.decode(frame, "full")
        elif mode == "viewport":
            pix, fp, st = sess.decode_viewport(frame, mask)
            rp, rf, rs = ref.decode(frame, "viewport", mask)
        else:
            sc = wv.FoveationSchedule.default(h.levels, 0.3, 0.6)
            pix, fp, st = sess.decode_foveated(frame, mask, sc)
            rp, rf, rs = ref.decode(frame, "foveated", mask, fractions=sc.fractions,
                                    gaze=(0.3, 0.6))
        np.testing.assert_array_equal(pix, rp)
        np.testing.assert_array_equal(fp, rf)
        assert (st.bytes_loaded, st.records_processed) == (rs.bytes_loaded, rs.records_processed)
    if mode == "viewport":
        out = sess.render_views(pose, (500, 500)).cpu().numpy()
        half = h.height // 2
        for e in range(2):
            r = wo.perspective(rp[e * half:(e + 1) * half], rf[e * half:(e + 1) * half],
                               pose.rotation(), 90.0, 90.0, 500, 500)
            assert np.abs(out[e].astype(int) - r.astype(int)).max() <= 1
    torch.cuda.synchronize()


def test_c1_full_decode_vs_oracle(wv, tmp_path):
    """BASELINE configs[0]: 1024x512, 16 frames, L3 full decode."""
    from paper_2208_10859_b200.synthetic import make_synthetic_clip
    clip = make_synthetic_clip(16, height=512, width=1024)
    path = tmp_path / "c1.wvv"
    wv.write_video(wv.encode_video(clip, wv.EncodeParams(levels=3)), path)
    sess = wv.DecodeSession(path)
    ref = wo.OracleSession(path)
    for f in (0, 5, 15):
        pix, fp, st = sess.decode_full(f)
        rp, rf, rs = ref.decode(f, "full")
        np.testing.assert_array_equal(pix, rp)
        assert abs(wv.psnr(pix, clip[f]) - wv.psnr(rp, clip[f])) < 0.01
        assert (st.bytes_loaded, st.records_processed) == (rs.bytes_loaded, rs.records_processed)


# ------------------------------------------------ incremental device state

def _random_call(rng, h, wv):
    """One decode request: (frame, mode, mask, schedule, pose)."""
    pose = wv.CameraPose(yaw=float(rng.uniform(-180, 180)), pitch=float(rng.uniform(-60, 60)),
                         roll=float(rng.uniform(-20, 20)), fov_h=float(rng.uniform(60, 110)),
                         fov_v=float(rng.uniform(60, 110)))
    mask = wv.stereo_mask(pose, (h.mask_w, h.mask_h)) if h.stereo else \
        wv.viewport_to_mask(pose, (h.mask_w, h.mask_h))
    mode = ["viewport", "viewport", "foveated", "full"][int(rng.integers(0, 4))]
    sc = wv.FoveationSchedule.default(h.levels, float(rng.uniform()), float(rng.uniform()))
    return int(rng.integers(0, h.frame_count)), mode, mask, sc, pose


def _decode(sess, frame, mode, mask, sc):
    if mode == "full":
        return sess.decode_full(frame)
    if mode == "viewport":
        return sess.decode_viewport(frame, mask)
    return sess.decode_foveated(frame, mask, sc)


@pytest.mark.parametrize("content", ["smooth", "noise"])
def test_history_independence(wv, tmp_path, content):
    """The device state carried between calls (dirty plane blocks, canvas and
    footprint tiles, cache entries) never leaks into a result: a random
    sequence of viewport / foveated / full decodes across sets, modes and
    poses equals, call by call, a fresh session's decode of that call alone."""
    import torch
    from paper_2208_10859_b200.synthetic import make_synthetic_clip_torch
    if content == "smooth":
        clip = make_synthetic_clip_torch(8, 1024, 1024, 3, device="cuda")
    else:
        g = torch.Generator(device="cuda").manual_seed(5)
        clip = torch.randint(0, 256, (8, 1024, 1024, 3), dtype=torch.uint8, device="cuda",
                             generator=g)
    path = tmp_path / "h.wvv"
    p = wv.EncodeParams(stereo=True, levels=4, mask_w=128, mask_h=128)
    wv.write_video(wv.encode_video(clip, p, device="cuda"), path)
    rng = np.random.default_rng(11)
    sess = wv.DecodeSession(path)
    h = sess.header
    for _ in range(14):
        frame, mode, mask, sc, pose = _random_call(rng, h, wv)
        pix, fp, _ = _decode(sess, frame, mode, mask, sc)
        with wv.DecodeSession(path) as fresh:
            rp, rf, _ = _decode(fresh, frame, mode, mask, sc)
        np.testing.assert_array_equal(fp, rf, err_msg=f"{frame} {mode}")
        np.testing.assert_array_equal(pix, rp, err_msg=f"{frame} {mode}")
    # device path (graph replays) after the same kind of history
    out = torch.empty((2, 300, 300, 3), dtype=torch.uint8, device="cuda")
    for _ in range(6):
        frame, mode, mask, sc, pose = _random_call(rng, h, wv)
        mode = "viewport" if mode == "full" else mode
        sess.decode_render_device(frame, mode, mask, pose, (300, 300), out,
                                  schedule=sc if mode == "foveated" else None).result()
        got = out.cpu().numpy()
        with wv.DecodeSession(path) as fresh:
            want = torch.empty_like(out)
            fresh.decode_render_device(frame, mode, mask, pose, (300, 300), want,
                                       schedule=sc if mode == "foveated" else None).result()
        np.testing.assert_array_equal(got, want.cpu().numpy(), err_msg=f"{frame} {mode}")


def test_c2_mono_full_vs_oracle(wv, tmp_path):
    """BASELINE C2 shape: 4096x2048 mono, L5 full decode == oracle."""
    from paper_2208_10859_b200.synthetic import make_synthetic_clip_torch
    clip = make_synthetic_clip_torch(4, 2048, 4096, 1, device="cuda")
    path = tmp_path / "c2.wvv"
    wv.write_video(wv.encode_video(clip, wv.EncodeParams(levels=5), device="cuda"), path)
    sess = wv.DecodeSession(path)
    ref = wo.OracleSession(path)
    host = clip.cpu().numpy()
    for f in (0, 3):
        pix, fp, st = sess.decode_full(f)
        rp, rf, rs = ref.decode(f, "full")
        np.testing.assert_array_equal(pix, rp)
        assert fp.all() and rf.all()
        assert abs(wv.psnr(pix, host[f]) - wv.psnr(rp, host[f])) < 0.01
        assert (st.bytes_loaded, st.records_processed) == (rs.bytes_loaded, rs.records_processed)


def test_8k_viewport_and_foveated_equal_full_inside_footprint(wv, tmp_path):
    """Bench-size property (8192^2 stereo, L6, 256^2 mask): inside its
    footprint a viewport or foveated decode equals the full-frame decode
    (decoding.py:296-299: the footprint marks where the result is exact), the
    footprint lies inside the request, and the writeout is fully covered."""
    import torch
    from paper_2208_10859_b200.synthetic import make_synthetic_clip_torch
    clip = make_synthetic_clip_torch(4, 8192, 8192, 3, device="cuda")
    path = tmp_path / "k8.wvv"
    p = wv.EncodeParams(stereo=True, fps=120.0, mask_w=256, mask_h=256)
    wv.write_video(wv.encode_video(clip, p, device="cuda"), path)
    del clip
    torch.cuda.empty_cache()
    sess = wv.DecodeSession(path)
    h = sess.header
    full = sess.decode_full(1)[0]
    for pose in (wv.CameraPose(yaw=30, pitch=10), wv.CameraPose(yaw=-150, pitch=-35, roll=8)):
        mask = wv.stereo_mask(pose, (h.mask_w, h.mask_h))
        req = wo.upscale(mask, h.width, h.height)
        for mode in ("viewport", "foveated"):
            if mode == "viewport":
                pix, fp, _ = sess.decode_viewport(1, mask)
            else:
                pix, fp, _ = sess.decode_foveated(
                    1, mask, wv.FoveationSchedule.default(h.levels, 0.4, 0.5))
            # (the default foveation keeps full detail only in a ~2% window,
            # which the 4-pixel synthesis support can erode to nothing)
            assert (fp.any() or mode == "foveated") and not (fp & ~req).any(), mode
            np.testing.assert_array_equal(pix[fp], full[fp])
            assert not pix[~req].any()
        # writeout: same uncovered-pixel count as the reference geometry, and
        # +-1 LSB where covered (2 eyes, 2000^2 each)
        pix, fp, _ = sess.decode_viewport(1, mask)
        out = sess.render_views(pose, (2000, 2000), check=False).cpu().numpy()
        got = sess.uncovered(reset=True)
        half = h.height // 2
        want = 0
        for e in range(2):
            try:
                r = wo.perspective(pix[e * half:(e + 1) * half], fp[e * half:(e + 1) * half],
                                   pose.rotation(), pose.fov_h, pose.fov_v, 2000, 2000)
                assert np.abs(out[e].astype(int) - r.astype(int)).max() <= 1
            except wo.Uncovered as u:
                want += u.args[0]
        assert got == want


def test_span_streaming_residency(wv, tmp_path):
    """residency="spans" (VideoReader.load_blocks, fileio.py:346-390): only the
    BlockEnd table is uploaded per set and the GPU copies the record spans of
    newly selected blocks from pinned host memory.  Results and statistics
    equal the whole-set residency call by call; a block's spans are copied
    once; unfetched HBM bytes are 0xFF, so reading one would fail loudly."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(9)
    clip = torch.randint(0, 256, (8, 1024, 1024, 3), dtype=torch.uint8, device="cuda", generator=g)
    path = tmp_path / "sp.wvv"
    wv.write_video(wv.encode_video(clip, wv.EncodeParams(stereo=True, levels=4, mask_w=128,
                                                         mask_h=128), device="cuda"), path)
    rng = np.random.default_rng(3)
    a = wv.DecodeSession(path)
    b = wv.DecodeSession(path, residency="spans")
    h = a.header
    total_records = sum(m.payload_length - h.table_bytes for m in a.reader.set_meta)
    for _ in range(12):
        frame, mode, mask, sc, pose = _random_call(rng, h, wv)
        pa, fa, sa = _decode(a, frame, mode, mask, sc)
        before = b.bytes_fetched
        pb, fb, sb = _decode(b, frame, mode, mask, sc)
        np.testing.assert_array_equal(pb, pa, err_msg=f"{frame} {mode}")
        np.testing.assert_array_equal(fb, fa)
        assert (sb.bytes_loaded, sb.records_processed) == (sa.bytes_loaded, sa.records_processed)
        assert b.bytes_fetched - before <= total_records
        # the same request again: everything is already in HBM
        again = b.bytes_fetched
        _decode(b, frame, mode, mask, sc)
        assert b.bytes_fetched == again
    assert 0 < b.bytes_fetched <= total_records
    # the file reads: the BlockEnd table, then the coalesced spans of the
    # blocks a decode newly needs -- one viewport decode reads far less than
    # the set's records
    assert len(b.reader.io_trace) > h.num_sets
    with wv.DecodeSession(path, residency="spans") as c:
        pose = wv.CameraPose(yaw=30, pitch=10)
        c.decode_viewport(1, wv.stereo_mask(pose, (h.mask_w, h.mask_h)))
        trace = c.reader.io_trace
        assert trace[0] == (0, h.table_bytes) and len(trace) == 2 and trace[1][0] == 0
        assert 0 < trace[1][1] < 0.8 * (a.reader.set_meta[0].payload_length - h.table_bytes)
    # device path (graph replay with the fetch step)
    out_a = torch.empty((2, 256, 256, 3), dtype=torch.uint8, device="cuda")
    out_b = torch.empty_like(out_a)
    for _ in range(4):
        frame, mode, mask, sc, pose = _random_call(rng, h, wv)
        mode = "viewport" if mode == "full" else mode
        s_ = sc if mode == "foveated" else None
        a.decode_render_device(frame, mode, mask, pose, (256, 256), out_a, schedule=s_).result()
        b.decode_render_device(frame, mode, mask, pose, (256, 256), out_b, schedule=s_).result()
        assert torch.equal(out_a, out_b)


def test_bounds_checked_build_runs_clean(wv):
    """Debug build with shared-memory index checks (WV_CHECK=1: K3 box /
    column / output tiles, K4 window) runs every mode, the render path and
    span streaming on the golden files without trapping."""
    import subprocess
    import sys
    from paper_2208_10859_b200 import build
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_2208_10859_b200", "variants", "checked.so")
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    if build._stale(lib):
        build.build(defines=["WV_CHECK=1"], out=lib)
    env = dict(os.environ, WV_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(root, "scripts", "sanitize.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.count(" ok") == 4


def test_direct_cascade_build_matches_reference():
    """The one-launch cascade (WV_K1_DIRECT=1: every level as a box OR of the
    low-res mask) replays all scripted reference decodes exactly, like the
    default step-by-step cascade."""
    import subprocess
    import sys
    from paper_2208_10859_b200 import build
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_2208_10859_b200", "variants", "k1direct.so")
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    if build._stale(lib):
        build.build(defines=["WV_K1_DIRECT=1"], out=lib)
    env = dict(os.environ, WV_LIB=lib)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        os.path.join(root, "tests", "test_gpu_parity.py")],
                       env=env, capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


# ------------------------------------------------------ stereo eye split

@pytest.mark.parametrize("clip", ["golden_stereo", "bench_c3"])
def test_eye_split_equals_whole_frame(wv, clip):
    """Each eye decoded alone (out_rows = that eye's half; the per-GPU share
    of a stereo eye split): its canvas rows, footprint rows and rendered eye
    image equal the whole-frame decode's, bit for bit, for viewport and
    foveated frames."""
    import sys
    import torch
    sys.path.insert(0, os.path.join(os.path.dirname(GOLDEN), "..", "scripts"))
    import make_bench_input as mbi
    path = (os.path.join(GOLDEN, "golden_stereo.wvv") if clip == "golden_stereo"
            else mbi.ensure_clip("c3", os.environ.get("WV_BENCH_CACHE", "/tmp/wvb200_bench")))
    whole = wv.DecodeSession(path)
    eyes = [wv.DecodeSession(path), wv.DecodeSession(path)]
    h = whole.header
    half = h.height // 2
    R = 200 if clip == "golden_stereo" else 1000
    outw = torch.empty((2, R, R, h.channels), dtype=torch.uint8, device="cuda")
    oute = [torch.empty((1, R, R, h.channels), dtype=torch.uint8, device="cuda") for _ in range(2)]
    for i, (yaw, pitch, mode) in enumerate([(30, 10, "viewport"), (-40, -60, "viewport"),
                                             (100, 75, "foveated"), (0, 0, "foveated")]):
        frame = i % h.frame_count
        pose = wv.CameraPose(yaw=yaw, pitch=pitch)
        mask = wv.stereo_mask(pose, (h.mask_w, h.mask_h))
        sc = wv.FoveationSchedule.default(h.levels, 0.4, 0.6) if mode == "foveated" else None
        whole.decode_render_device(frame, mode, mask, pose, (R, R), outw, schedule=sc)
        torch.cuda.synchronize()
        cw, fw = whole._canvas.clone(), whole._footprint.clone()
        for e in range(2):
            eyes[e].decode_render_device(frame, mode, mask, pose, (R, R), oute[e], schedule=sc,
                                         eye=e)
            torch.cuda.synchronize()
            rows = slice(e * half, (e + 1) * half)
            assert torch.equal(eyes[e]._canvas[:, rows], cw[:, rows]), (i, e, "canvas")
            assert torch.equal(eyes[e]._footprint[rows], fw[rows]), (i, e, "footprint")
            assert torch.equal(oute[e][0], outw[e]), (i, e, "eye image")
    for s in [whole] + eyes:
        s.close()


@pytest.mark.parametrize("name", ["smooth_hq.wvv", "smooth_n8.wvv"])
def test_prefetch_spans_overlapped(wv, name):
    """advance() under span residency (decoding.py:335-354): the next set's
    selection, file reads and HBM copies run on the copy stream with the
    selection-only workspace; the next set's decodes then equal a
    whole-set-residency session's, call for call, including the cache
    accounting of the prefetched blocks, and its file reads are spans."""
    import torch
    path = os.path.join(GOLDEN, name)
    with wv.DecodeSession(path) as ref_s, wv.DecodeSession(path, residency="spans") as s:
        h = s.header
        pose = wv.CameraPose(yaw=20, pitch=5)
        m = (wv.stereo_mask(pose, (h.mask_w, h.mask_h)) if h.stereo
             else wv.viewport_to_mask(pose, (h.mask_w, h.mask_h)))
        big = np.ones_like(m)
        for sess in (ref_s, s):
            sess.decode_viewport(0, m)
            sess.advance(0, m)
        # decodes of the current set run while the prefetch is in flight
        out = torch.empty((2 if h.stereo else 1, 64, 64, h.channels), dtype=torch.uint8,
                          device="cuda")
        s.decode_render_device(1, "viewport", m, pose, (64, 64), out)
        for sess in (ref_s, s):
            sess.join_prefetch()
        n = h.inter_size
        for frame, mask in ((n, m), (n + 1, big), (n + 2, m)):
            if frame >= h.frame_count:
                continue
            a = ref_s.decode_viewport(frame, mask)
            b = s.decode_viewport(frame, mask)
            np.testing.assert_array_equal(b[0], a[0])
            np.testing.assert_array_equal(b[1], a[1])
            assert (b[2].bytes_loaded, b[2].records_processed) == (
                a[2].bytes_loaded, a[2].records_processed)
        reads = [v for si, v in s.reader.io_trace if si == 1]
        assert reads[0] == h.table_bytes and len(reads) >= 2


@pytest.mark.parametrize("name", ["noise_bs16.wvv", "golden_float.wvv", "smooth_n8.wvv"])
def test_table_expand_rebuilds_blockend_table(wv, name):
    """wv_table_expand (span residency's compact table upload): the u16
    record counts expand to the file's BlockEnd table bit for bit."""
    import ctypes as C
    import torch
    from paper_2208_10859_b200 import _native as N
    lib = N.load()
    with wv.VideoReader(os.path.join(GOLDEN, name)) as r:
        h = r.header
        for si in range(h.num_sets):
            raw = bytes(r.read_set_payload(si))[: h.table_bytes]
            ends = np.frombuffer(raw, "<u8")
            counts = (np.diff(ends, prepend=np.uint64(0)) // h.record_size).astype(np.uint16)
            dc = torch.from_numpy(counts.view(np.int16)).cuda()
            out = torch.zeros(ends.size, dtype=torch.int64, device="cuda")
            assert lib.wv_table_expand(C.c_void_p(dc.data_ptr()), C.c_uint64(ends.size),
                                       h.record_size, C.c_void_p(out.data_ptr()), None) == 0
            torch.cuda.synchronize()
            assert out.cpu().numpy().view(np.uint64).tobytes() == raw

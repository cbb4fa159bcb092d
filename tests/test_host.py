"""CPU-only checks: the C ABI library loads and exports every declared
symbol (no compute calls), the .wvv reader, the package encoder's byte
exactness against reference-produced files, host-side mask geometry, and the
foveation window arithmetic against the oracle."""
import ctypes as C
import hashlib
import json
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, unpack_mask
from oracle import wavevid_oracle as wo


@pytest.fixture(scope="module")
def lib():
    from paper_2208_10859_b200 import _native, build
    build.build()
    return _native.load()


def _declared_functions():
    text = open(os.path.join(ROOT, "include", "wavevid_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(wv_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol(lib):
    names = _declared_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n
    from paper_2208_10859_b200 import _native
    assert sorted(_native.EXPORTS) == names


def test_abi_host_functions(lib):
    from paper_2208_10859_b200 import _native as N
    assert lib.wv_abi_version() == N.WV_ABI_VERSION == 4
    assert lib.wv_status_string(0) == b"ok"
    g = N.Geometry(8192, 8192, 3, 6, 4, 32, 0, 256, 256)
    b = C.c_uint64()
    assert lib.wv_workspace_bytes(C.byref(g), C.byref(b)) == 0
    # plane 805 MB + level buffers + masks: about 1.1 GB at 8K
    assert 1.0e9 < b.value < 1.3e9
    bad = N.Geometry(100, 64, 3, 6, 4, 32, 0, 64, 64)          # not divisible by 2^6
    assert lib.wv_workspace_bytes(C.byref(bad), C.byref(b)) == N.WV_ERR_ARG
    # decode entry points reject missing pointers before touching the GPU
    a = N.FrameArgs()
    assert lib.wv_decode_frame(C.byref(g), C.byref(a), None, None) == N.WV_ERR_ARG
    # K3 work item: 32 rows x 28 columns per subband (a warp = 28 columns + 2 x 2 halo);
    # the wide build (full-frame sessions) puts two warp strips side by side
    assert N.synthesis_tile() == (32, 28)
    wide = N.load_tiles(2)
    assert wide is not lib and N.synthesis_tile(wide) == (32, 56)
    assert wide.wv_abi_version() == N.WV_ABI_VERSION
    assert all(hasattr(wide, n) for n in _declared_functions())
    assert lib.wv_synthesis_tile(None, None) == N.WV_ERR_ARG


def test_encode_abi_host_checks(lib):
    """wv_encode_*: sizing and argument validation (no GPU needed)."""
    from paper_2208_10859_b200 import _native as N
    ep = N.EncodeParams()
    ep.width = ep.height = 8192
    ep.channels, ep.levels, ep.inter_size, ep.block_size, ep.quantize = 3, 6, 4, 32, 1
    ws, cap = C.c_uint64(), C.c_uint64()
    assert lib.wv_encode_workspace_bytes(C.byref(ep), C.byref(ws)) == 0
    assert lib.wv_encode_payload_capacity(C.byref(ep), C.byref(cap)) == 0
    samples = 4 * 8192 * 8192 * 3
    assert 8 * samples <= ws.value < 8 * samples * 1.05     # two f32 pyramids + tables
    assert cap.value == 4 * 8192 * 8192 * (2 + 3)           # every coefficient a record
    for field, value in (("inter_size", 3), ("block_size", 48), ("levels", 0), ("channels", 5)):
        badp = N.EncodeParams.from_buffer_copy(ep)
        setattr(badp, field, value)
        assert lib.wv_encode_workspace_bytes(C.byref(badp), C.byref(ws)) == N.WV_ERR_ARG
    odd = N.EncodeParams.from_buffer_copy(ep)
    odd.width = 8192 + 32                                     # not divisible by 2^6
    assert lib.wv_encode_payload_capacity(C.byref(odd), C.byref(cap)) == N.WV_ERR_ARG
    # missing device pointers are rejected before any launch
    assert lib.wv_encode_set(C.byref(ep), None, None, None, C.c_uint64(0), None, None, None,
                             C.c_uint64(0), None, None) == N.WV_ERR_ARG


def test_struct_layouts_match_header():
    from paper_2208_10859_b200 import _native as N
    assert C.sizeof(N.Geometry) == 36
    assert C.sizeof(N.FrameResult) == 48
    assert N.FrameArgs.h_payload.offset == N.FrameArgs.d_result.offset + 8
    assert N.FrameArgs.d_mask.offset == 16
    assert N.FrameArgs.d_payload.offset == 16 + 8 + 12 * 4 * 4
    assert C.sizeof(N.EncodeParams) == 8 * 4 + 4 * N.WV_MAX_LEVELS + 4 * N.WV_ENC_MAX_N


@pytest.mark.parametrize("name", ["golden_quantized.wvv", "golden_float.wvv",
                                  "golden_stereo.wvv", "noise_bs16.wvv", "smooth_n8.wvv"])
def test_reader_parses_fixture(manifest, name):
    from paper_2208_10859_b200.fileio import VideoReader
    with VideoReader(os.path.join(GOLDEN, name)) as r:
        h = r.header
        assert list(r.header.__dict__.keys())[:4] == ["width", "height", "frame_count", "fps"]
        assert h.num_sets == len(r.set_meta)
        total = 0
        for si in range(h.num_sets):
            buf = r.read_set_payload(si)
            t = r.block_table(si)
            assert len(buf) == r.set_meta[si].payload_length
            assert t.total_bytes() + h.table_bytes == len(buf)
            total += r.set_meta[si].record_count
        assert total > 0


def test_golden_header_fields():
    # pkg/tests/data/golden.json header entries
    from paper_2208_10859_b200.fileio import VideoReader
    with VideoReader(os.path.join(GOLDEN, "golden_stereo.wvv")) as r:
        h = r.header
        assert (h.width, h.height, h.channels, h.levels, h.inter_size, h.block_size) == \
            (128, 128, 3, 3, 4, 32)
        assert h.stereo and not h.float_mode and h.fps == 60.0
    with VideoReader(os.path.join(GOLDEN, "golden_quantized.wvv")) as r:
        assert [m.record_count for m in r.set_meta] == [16383]
        assert [m.payload_offset for m in r.set_meta] == [280]
        assert [m.payload_length for m in r.set_meta] == [82043]


def _clip(spec_name):
    from paper_2208_10859_b200.synthetic import make_synthetic_clip

    def noise(seed, frames, size, channels):
        return np.random.default_rng(seed).integers(0, 256, (frames, size, size, channels),
                                                    dtype=np.uint8)
    return {
        "golden_quantized.wvv": lambda: noise(11, 4, 64, 3),
        "golden_float.wvv": lambda: noise(12, 2, 64, 1),
        "golden_stereo.wvv": lambda: noise(13, 4, 128, 3),
        "smooth_hq.wvv": lambda: make_synthetic_clip(8, 128),
        "smooth_lossless.wvv": lambda: make_synthetic_clip(4, 64),
        "noise_bs16.wvv": lambda: noise(5, 4, 128, 3),
        "smooth_n8.wvv": lambda: make_synthetic_clip(10, 64),
        "smooth_n1_mono.wvv": lambda: make_synthetic_clip(3, 64, 1),
        "wide_equirect.wvv": lambda: make_synthetic_clip(4, 128)[:, :64],
    }[spec_name]()


@pytest.mark.parametrize("name", ["golden_quantized.wvv", "golden_float.wvv",
                                  "golden_stereo.wvv", "smooth_hq.wvv", "smooth_lossless.wvv",
                                  "noise_bs16.wvv", "smooth_n8.wvv", "smooth_n1_mono.wvv",
                                  "wide_equirect.wvv"])
def test_encoder_reproduces_reference_bytes(manifest, name, tmp_path):
    """The package encoder (torch, CPU here) writes the reference encoder's
    exact bytes; the first three digests are pkg/tests/data/golden.json's."""
    from paper_2208_10859_b200.encoding import EncodeParams, MappingKind, encode_video
    from paper_2208_10859_b200.fileio import write_video
    spec = dict(manifest[name]["params"])
    spec["mapping"] = MappingKind[spec.get("mapping", "EQUIRECTANGULAR")]
    out = tmp_path / "x.wvv"
    write_video(encode_video(_clip(name), EncodeParams(**spec)), out)
    assert hashlib.sha256(out.read_bytes()).hexdigest() == manifest[name]["sha256"]


def test_synthetic_clip_matches_reference():
    from paper_2208_10859_b200.synthetic import make_synthetic_clip
    want = json.load(open(os.path.join(GOLDEN, "synthetic.json")))
    for k, v in want.items():
        f, size, c, seed = (int(x) for x in k.split("x"))
        got = make_synthetic_clip(f, size, c, seed)
        assert hashlib.sha256(got.tobytes()).hexdigest() == v


def test_viewport_and_stereo_masks_match_reference():
    from paper_2208_10859_b200.projection import CameraPose, stereo_mask, viewport_to_mask
    want = np.load(os.path.join(GOLDEN, "projection.npz"))
    n = 0
    for k in want.files:
        if not (k.startswith("vmask|") or k.startswith("smask|")):
            continue
        kind, i, dims = k.split("|")
        mw, mh = (int(x) for x in dims.split("x"))
        yaw, pitch, roll, fh, fv = want[f"pose|{i}"]
        pose = CameraPose(float(yaw), float(pitch), float(roll), float(fh), float(fv))
        fn = viewport_to_mask if kind == "vmask" else stereo_mask
        got = fn(pose, (mw, mh))
        np.testing.assert_array_equal(got, unpack_mask(want[k], (mh, mw)), err_msg=k)
        n += 1
    assert n >= 100


def test_mask_bbox_and_fovea_rects_match_oracle(rng):
    from paper_2208_10859_b200.decoding import FoveationSchedule, fovea_rects, mask_bbox
    for H, W, mh, mw in [(128, 128, 64, 64), (8192, 8192, 256, 256), (512, 1024, 32, 64),
                         (96, 64, 128, 128)]:
        for _ in range(20):
            m = np.zeros((mh, mw), bool)
            y, x = rng.integers(0, mh), rng.integers(0, mw)
            m[y:y + rng.integers(1, mh), x:x + rng.integers(1, mw)] = True
            pm = wo.upscale(m, W, H)
            want = wo.pixel_bbox(pm)
            assert mask_bbox(m, W, H) == want
            if want is None:
                continue
            L = 3
            sc = FoveationSchedule.default(L, float(rng.uniform()), float(rng.uniform()))
            assert fovea_rects(want, H, W, sc, L) == wo.fovea_rects(
                want, H, W, sc.fractions, sc.gaze_u, sc.gaze_v, L)


def test_schedule_and_pose_validation():
    from paper_2208_10859_b200 import CameraPose, DecodeError, FoveationSchedule, ProjectionError
    assert FoveationSchedule.default(6).fractions == (1.0, 0.65, 0.40, 0.22, 0.10, 0.04, 0.02)
    for levels in range(1, 8):
        f = FoveationSchedule.default(levels).fractions
        assert f[0] == 1.0 and all(a >= b for a, b in zip(f, f[1:]))
    for bad in [((1.0, 0.2, 0.5),), ((0.9, 0.5),)]:
        with pytest.raises(DecodeError):
            FoveationSchedule(*bad)
    with pytest.raises(DecodeError):
        FoveationSchedule((1.0, 0.5), gaze_u=1.5)
    with pytest.raises(ProjectionError):
        CameraPose(fov_h=0)
    with pytest.raises(ProjectionError):
        CameraPose(pitch=95)
    r = CameraPose(yaw=33, pitch=-20, roll=7).rotation()
    np.testing.assert_allclose(r @ r.T, np.eye(3), atol=1e-12)
    np.testing.assert_allclose(r, wo.pose_rotation(33, -20, 7), atol=0)


def test_footprint_bit_packing_roundtrip(rng):
    from paper_2208_10859_b200.projection import pack_footprint, unpack_footprint
    for shape in [(5, 7), (64, 64), (33, 100)]:
        fp = rng.random(shape) < 0.5
        np.testing.assert_array_equal(unpack_footprint(pack_footprint(fp), shape[1]), fp)


def test_decode_session_requires_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2208_10859_b200 import DecodeSession
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        DecodeSession(os.path.join(GOLDEN, "golden_quantized.wvv"))


def test_lifting_kernels_have_no_fused_multiply_add(lib):
    """Bit-exact synthesis needs every product rounded before its add: in the
    K3 kernels' SASS every FFMA2 is a product with the run-time -0.0 addend,
    a scalar broadcast to both lanes (a*b + -0 rounds like mul.rn), and there
    is no scalar FFMA.  A contracted paired multiply-add would show a packed
    (F32x2) addend."""
    import re
    import subprocess
    from paper_2208_10859_b200 import _native
    sass = subprocess.run(["cuobjdump", "-sass", _native.LIB_PATH], capture_output=True,
                          text=True).stdout
    fn, bad, n_ffma2 = None, [], 0
    for line in sass.splitlines():
        if "Function :" in line:
            fn = line.split(":")[1].strip()
        elif fn and "k_level" in fn:
            if re.search(r"\bFFMA\b", line):
                bad.append((fn, line.strip()[:60]))
            m = re.search(r"FFMA2 [^;]*,\s*(\S+)\s*;", line)
            if m:
                n_ffma2 += 1
                if not m.group(1).endswith(".F32"):   # broadcast scalar addend
                    bad.append((fn, line.strip()[:80]))
    assert "k_level" in sass and not bad, bad[:3]
    assert n_ffma2 > 0
    assert "UTMALDG" in sass      # the synthesis tiles are TMA-fed


# ------------------------------------------------ C++ .wvv reader (§8f row 3)

@pytest.mark.parametrize("name", ["golden_quantized.wvv", "golden_float.wvv", "golden_stereo.wvv",
                                  "smooth_hq.wvv", "smooth_lossless.wvv", "noise_bs16.wvv",
                                  "smooth_n8.wvv", "smooth_n1_mono.wvv", "wide_equirect.wvv"])
def test_native_reader_matches_python_reader(lib, name):
    """wv_file_* (C++) parse every fixture exactly like fileio.VideoReader."""
    from paper_2208_10859_b200 import _native as N
    from paper_2208_10859_b200.fileio import VideoReader
    path = os.path.join(GOLDEN, name).encode()
    info = N.FileInfo()
    assert lib.wv_file_info_read(path, C.byref(info)) == 0
    with VideoReader(os.path.join(GOLDEN, name)) as r:
        h = r.header
        g = info.geom
        assert (g.width, g.height, g.channels, g.levels, g.inter_size, g.block_size,
                g.float_mode, g.mask_w, g.mask_h) == (h.width, h.height, h.channels, h.levels,
                                                     h.inter_size, h.block_size, int(h.float_mode),
                                                     h.mask_w, h.mask_h)
        assert (info.frame_count, info.pad_frames, info.num_sets, bool(info.stereo)) == \
            (h.frame_count, h.pad_frames, h.num_sets, h.stereo)
        assert np.float32(info.fps) == np.float32(h.fps) and info.table_bytes == h.table_bytes
        for si, m in enumerate(r.set_meta):
            si_info = N.SetInfo()
            ext = np.zeros((h.inter_size, h.channels, 4), np.float32)
            assert lib.wv_file_set_read(path, si, C.byref(si_info), ext.ctypes.data) == 0
            assert (si_info.payload_offset, si_info.payload_length, si_info.record_count) == \
                (m.payload_offset, m.payload_length, m.record_count)
            np.testing.assert_array_equal(ext, m.extrema)
            buf = np.zeros(m.payload_length, np.uint8)
            assert lib.wv_file_payload_read(path, si, buf.ctypes.data, buf.size) == 0
            assert bytes(buf) == bytes(r.read_set_payload(si))
            assert lib.wv_file_payload_read(path, si, buf.ctypes.data, buf.size - 1) == N.WV_ERR_ARG
        assert lib.wv_file_set_read(path, h.num_sets, C.byref(N.SetInfo()), None) == N.WV_ERR_ARG


def test_native_reader_rejects_malformed(lib, tmp_path):
    """fileio.py:34 FormatError cases: bad magic, bad version, truncation,
    non-contiguous payloads; missing file -> WV_ERR_IO."""
    from paper_2208_10859_b200 import _native as N
    raw = bytearray(open(os.path.join(GOLDEN, "smooth_n8.wvv"), "rb").read())
    info = N.FileInfo()
    cases = {
        "magic": (lambda b: b.__setitem__(slice(0, 4), b"XXXX"), N.WV_ERR_FORMAT),
        "version": (lambda b: b.__setitem__(slice(4, 6), (7).to_bytes(2, "little")), N.WV_ERR_FORMAT),
        "truncated": (lambda b: b.__delitem__(slice(70, None)), N.WV_ERR_IO),
        # second SetMeta entry (n 8, C 3: 408 bytes each) -> payload_offset moved
        "contiguity": (lambda b: b.__setitem__(slice(64 + 408, 64 + 416),
                                               (12345).to_bytes(8, "little")), N.WV_ERR_FORMAT),
    }
    for what, (mutate, want) in cases.items():
        b = bytearray(raw)
        mutate(b)
        p = tmp_path / f"{what}.wvv"
        p.write_bytes(bytes(b))
        assert lib.wv_file_info_read(str(p).encode(), C.byref(info)) == want, what
    assert lib.wv_file_info_read(str(tmp_path / "none.wvv").encode(), C.byref(info)) == N.WV_ERR_IO


def test_c_only_consumer_builds_and_reads(lib, tmp_path):
    """examples/c_consumer.c: a plain-C program linked against the library
    reads a .wvv through the C ABI (no Python, no torch)."""
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    from paper_2208_10859_b200 import _native
    exe = tmp_path / "c_consumer"
    libdir = os.path.dirname(_native.LIB_PATH)
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "c_consumer.c"), "-L", libdir, "-l:_wvb200.so",
                    f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), os.path.join(GOLDEN, "smooth_n8.wvv")], capture_output=True,
                         text=True, check=True).stdout
    assert "64x64 C3 L2 n8 bs32 frames 10 sets 2" in out and "set 1:" in out


def test_q255_table_matches_numpy():
    """K2's compiled q/255 table is numpy's float32 division, bit for bit
    (dequantize_values, encoding.py:270-271)."""
    src = open(os.path.join(ROOT, "paper_2208_10859_b200", "csrc", "wv_temporal.cu")).read()
    body = src[src.index("kQ255Bits[256] = {"):]
    body = body[:body.index("};")]
    got = np.array([int(x, 16) for x in re.findall(r"0x([0-9a-f]{8})u", body)], np.uint32)
    want = (np.arange(256, dtype=np.float32) / np.float32(255.0)).view(np.uint32)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("name", ["noise_bs16.wvv", "smooth_hq.wvv", "golden_stereo.wvv"])
def test_spans_read_matches_load_blocks(lib, name):
    """wv_spans_read (span streaming's file reader, host-only): the records
    of the listed blocks land at their payload offsets, and the byte counts
    follow VideoReader.load_blocks (fileio.py:346-390: spans per (t, run),
    coalesced through 4 KiB gaps)."""
    from paper_2208_10859_b200 import _native as N
    from paper_2208_10859_b200.fileio import VideoReader
    path = os.path.join(GOLDEN, name)
    rng = np.random.default_rng(len(name))
    with VideoReader(path) as r:
        h = r.header
        for si in range(h.num_sets):
            m = r.set_meta[si]
            full = bytes(r.read_set_payload(si))
            table = np.frombuffer(full[:h.table_bytes], "<u8").reshape(h.inter_size, h.num_blocks)
            ids = np.unique(rng.integers(0, h.num_blocks, max(1, h.num_blocks // 3))).astype(np.uint32)
            ids = rng.permutation(ids)                       # any order, as the GPU lists them
            buf = np.zeros(m.payload_length + 16, np.uint8)
            buf[:h.table_bytes] = np.frombuffer(full[:h.table_bytes], np.uint8)
            cnt = np.array([len(ids)], np.uint32)
            fd = os.open(path, os.O_RDONLY)
            try:
                j = N.SpanJob(fd=fd, n=h.inter_size, nb=h.num_blocks,
                              payload_offset=m.payload_offset, payload_bytes=m.payload_length,
                              table_bytes=h.table_bytes, table=buf.ctypes.data, dst=buf.ctypes.data,
                              ids=ids.ctypes.data, count=cnt.ctypes.data, coalesce_gap=4096)
                br, bs = C.c_uint64(), C.c_uint64()
                assert lib.wv_spans_read(C.byref(j), C.byref(br), C.byref(bs)) == 0
            finally:
                os.close(fd)
            flat = table.reshape(-1)
            srt = np.sort(ids)
            runs, i = [], 0
            while i < len(srt):
                e = i
                while e + 1 < len(srt) and srt[e + 1] == srt[e] + 1:
                    e += 1
                runs.append((int(srt[i]), int(srt[e])))
                i = e + 1
            spans = []
            for t in range(h.inter_size):
                for a, b in runs:
                    k = t * h.num_blocks + a
                    st = int(flat[k - 1]) if k else 0
                    spans.append((st, int(flat[t * h.num_blocks + b])))
            tb = h.table_bytes
            for st, en in spans:                             # every record in place
                assert bytes(buf[tb + st:tb + en]) == full[tb + st:tb + en]
            merged = []
            for st, en in sorted(spans):
                if st >= en:
                    continue
                if merged and st - merged[-1][1] <= 4096:
                    merged[-1][1] = max(merged[-1][1], en)
                else:
                    merged.append([st, en])
            assert bs.value == sum(e - s for s, e in spans)
            assert br.value == sum(e - s for s, e in merged)

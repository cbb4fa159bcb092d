"""GPU parity: the B200 decode path against the reference fixtures and the
CPU oracle.  Bars (north star): dequantised coefficients bit-exact, u8
pixels exact (bar +-1 LSB), footprint/stats exact, perspective +-1 LSB."""
import os

import numpy as np
import pytest

from conftest import GOLDEN, case_calls, unpack_mask
from oracle import wavevid_oracle as wo

pytestmark = pytest.mark.gpu

FILES = ["golden_quantized.wvv", "golden_float.wvv", "golden_stereo.wvv",
         "smooth_hq.wvv", "smooth_lossless.wvv", "noise_bs16.wvv",
         "smooth_n8.wvv", "smooth_n1_mono.wvv", "wide_equirect.wvv"]


@pytest.fixture(scope="module")
def pkg():
    import paper_2208_10859_b200 as p
    from paper_2208_10859_b200 import build
    build.build()
    return p


def _replay(pkg, name, decode_cases, device_api=False, tile_strips=1):
    from paper_2208_10859_b200.decoding import FoveationSchedule
    sess = pkg.DecodeSession(os.path.join(GOLDEN, name), tile_strips=tile_strips)
    h = sess.header
    for i, c in enumerate(case_calls(decode_cases, name)):
        mask = None
        if c["mask_packed"] is not None:
            mask = unpack_mask(c["mask_packed"], (h.mask_h, h.mask_w))
        if c["kind"] == "full":
            pix, fp, st = sess.decode_full(c["frame"])
        elif c["kind"] == "viewport":
            pix, fp, st = sess.decode_viewport(c["frame"], mask)
        else:
            sc = FoveationSchedule(c["fractions"], *c["gaze"])
            pix, fp, st = sess.decode_foveated(c["frame"], mask, sc)
        want_fp = unpack_mask(c["footprint"], (h.height, h.width))
        np.testing.assert_array_equal(fp, want_fp, err_msg=f"{name} call {i} footprint")
        np.testing.assert_array_equal(pix, c["pixels"], err_msg=f"{name} call {i} pixels")
        assert (st.bytes_loaded, st.records_processed) == c["stats"], (name, i)
        assert len(sess._cache) <= 3
    sess.close()


@pytest.mark.parametrize("name", FILES)
def test_replay_reference_decodes(pkg, decode_cases, name):
    _replay(pkg, name, decode_cases)


@pytest.mark.parametrize("name", ["golden_quantized.wvv", "golden_stereo.wvv", "smooth_n8.wvv",
                                  "noise_bs16.wvv", "wide_equirect.wvv"])
def test_replay_reference_decodes_wide_tiles(pkg, decode_cases, name):
    """The same reference call sequences through the 56-column synthesis
    tiles (the _wvb200_wide.so build): identical pixels, footprints, stats."""
    _replay(pkg, name, decode_cases, tile_strips=2)


@pytest.mark.parametrize("name", ["golden_quantized.wvv", "golden_float.wvv",
                                  "smooth_n8.wvv", "noise_bs16.wvv", "smooth_n1_mono.wvv"])
def test_dequantized_plane_bit_exact(pkg, name):
    """K2 output == oracle temporal plane x inclusion, bitwise (all t)."""
    path = os.path.join(GOLDEN, name)
    hd, sets = wo.read_file(path)
    sess = pkg.DecodeSession(path)
    for frame in range(min(hd.frame_count, 2 * hd.inter_size)):
        si, t = divmod(frame, hd.inter_size)
        sess.decode_full(frame)
        got = sess.plane().permute(1, 2, 0).cpu().numpy()
        want = wo.temporal_plane(hd, sets[si], np.arange(hd.num_blocks), t)
        np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32),
                                      err_msg=f"{name} frame {frame}")
    sess.close()


def test_dequantized_plane_masked(pkg):
    """Viewport decode: selected blocks carry plane x inclusion, the rest 0."""
    path = os.path.join(GOLDEN, "noise_bs16.wvv")
    hd, sets = wo.read_file(path)
    sess = pkg.DecodeSession(path)
    rng = np.random.default_rng(3)
    for _ in range(6):
        m = np.zeros((hd.mask_h, hd.mask_w), bool)
        y, x = rng.integers(0, 48, 2)
        m[y:y + 12, x:x + 20] = True
        frame = int(rng.integers(0, hd.frame_count))
        sess.decode_viewport(frame, m)
        got = sess.plane().permute(1, 2, 0).cpu().numpy()
        pm = wo.upscale(m, hd.width, hd.height)
        detail = wo.detail_masks(pm, hd.levels)
        incl = wo.inclusion(detail, hd.width, hd.height)
        blocks = wo.select_blocks(incl, hd.block_size)
        want = wo.temporal_plane(hd, sets[frame // hd.inter_size], blocks, frame % hd.inter_size)
        want = want * incl[:, :, None]
        np.testing.assert_array_equal(got, want)
    sess.close()

"""K3 at odd sizes: wavelets.synthesize_2d (the decode's K3 kernels in
float32) against the oracle's full-frame inverse (oracle synth_full, pinned
to the reference by tests/test_oracle_golden.py) on seeded random pyramids,
bitwise.  The shapes put partial 32x28 tiles at every level, subband widths
that are not multiples of 4 floats (plain-load boxes) next to TMA-fed ones,
and level borders inside column segments."""
import numpy as np
import pytest

from oracle import wavevid_oracle as wo

pytestmark = pytest.mark.gpu

SHAPES = [((1000, 1400, 3), 3), ((504, 616), 3), ((2048, 1792, 3), 6), ((96, 4056), 3)]


@pytest.mark.parametrize("shape,levels", SHAPES)
def test_synthesize_2d_random_matches_oracle(shape, levels):
    import paper_2208_10859_b200 as wv
    from paper_2208_10859_b200 import build
    build.build()
    rng = np.random.default_rng(sum(shape) + levels)
    # coefficient magnitudes like a real pyramid: O(1) approximation band,
    # small details, many exact zeros (the sparse planes K2 writes)
    pyr = rng.normal(0.0, 0.05, shape).astype(np.float32)
    pyr[rng.random(shape) < 0.6] = 0.0
    h, w = shape[0] >> levels, shape[1] >> levels
    pyr[:h, :w] = rng.random((h, w) + shape[2:]).astype(np.float32)
    got = wv.synthesize_2d(wv.CoefficientPyramid(pyr, levels), wv.WaveletKind.CDF97)
    data = pyr if pyr.ndim == 3 else pyr[..., None]
    want = wo.synth_full(data, levels)
    want = want if pyr.ndim == 3 else want[..., 0]
    assert got.shape == want.shape
    bad = np.flatnonzero(got.view(np.uint32) != want.view(np.uint32))
    assert bad.size == 0, f"{bad.size} mismatches, first at {np.unravel_index(bad[0], got.shape)}"

"""The reference's wavelet API exported by the package (wavelets.py):
analysis on the host/encoder path (CPU test), synthesis through the C ABI's
K3 kernels (GPU test), both bitwise against reference outputs
(tests/golden/make_wavelet_golden.py)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN

CASES = ["rgb_cdf97", "mono_cdf97", "rgb_haar", "odd_cdf97", "tall_cdf97", "tiny_cdf97",
         "wide_cdf97"]


@pytest.fixture(scope="module")
def fx():
    return dict(np.load(os.path.join(GOLDEN, "wavelets.npz")))


def _kind(wv, fx, name):
    levels, k = (int(v) for v in fx[f"{name}|meta"])
    return levels, (wv.WaveletKind.CDF97 if k == 0 else wv.WaveletKind.HAAR)


@pytest.mark.parametrize("name", CASES)
def test_analyze_2d_matches_reference(fx, name):
    import paper_2208_10859_b200 as wv
    levels, kind = _kind(wv, fx, name)
    p = wv.analyze_2d(fx[f"{name}|x"], levels, kind)
    assert p.levels == levels
    assert np.array_equal(p.data, fx[f"{name}|analysis"])


def test_pyramid_validation():
    import paper_2208_10859_b200 as wv
    with pytest.raises(wv.DimensionError):
        wv.CoefficientPyramid(np.zeros((48, 40), np.float32), 4)
    assert wv.WaveletKind.CDF97.half_width == 4 and wv.WaveletKind.HAAR.half_width == 0


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_synthesize_2d_matches_reference(fx, name):
    import paper_2208_10859_b200 as wv
    from paper_2208_10859_b200 import build
    build.build()
    levels, kind = _kind(wv, fx, name)
    got = wv.synthesize_2d(wv.CoefficientPyramid(fx[f"{name}|pyramid"], levels), kind)
    want = fx[f"{name}|synthesis"]
    assert got.shape == want.shape and got.dtype == np.float32
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))

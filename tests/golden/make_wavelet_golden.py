"""Fixtures for the wavelet API (wavelets.py exports) from the REAL
reference: analyze_2d / synthesize_2d outputs for seeded inputs.
    python tests/golden/make_wavelet_golden.py"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
from wavevid.wavelets import CoefficientPyramid, WaveletKind, analyze_2d, synthesize_2d  # noqa: E402

out = {}
rng = np.random.default_rng(21)
cases = {"rgb_cdf97": ((64, 128, 3), 3, "CDF97"), "mono_cdf97": ((96, 64), 4, "CDF97"),
         "rgb_haar": ((32, 64, 3), 2, "HAAR"),
         # K3 edge shapes: subband widths that are not multiples of 4 floats
         # (plain-load boxes), partial 32x28 tiles, a 1x1 coarsest level
         "odd_cdf97": ((80, 40, 3), 3, "CDF97"), "tall_cdf97": ((144, 112), 4, "CDF97"),
         "tiny_cdf97": ((16, 16), 4, "CDF97"), "wide_cdf97": ((64, 232), 3, "CDF97")}
for name, (shape, levels, kind) in cases.items():
    x = rng.random(shape).astype(np.float32)
    p = analyze_2d(x, levels, WaveletKind[kind])
    # synthesis input: the analysis with a few coefficients perturbed
    q = p.data.copy()
    q.reshape(-1)[rng.integers(0, q.size, 50)] += rng.normal(0, 0.1, 50).astype(np.float32)
    out[f"{name}|x"] = x
    out[f"{name}|analysis"] = p.data
    out[f"{name}|pyramid"] = q
    out[f"{name}|synthesis"] = synthesize_2d(CoefficientPyramid(q, levels), WaveletKind[kind])
    out[f"{name}|meta"] = np.array([levels, 0 if kind == "CDF97" else 1])
np.savez_compressed(os.path.join(HERE, "wavelets.npz"), **out)
print(sorted(out))

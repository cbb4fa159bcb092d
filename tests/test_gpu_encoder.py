"""CUDA encoder (csrc/wv_encode.cu) against the
reference's bytes: every golden fixture re-encoded on the GPU must hash to
the manifest's sha256 (the first three are pkg/tests/data/golden.json's),
and an 8K stereo set must round-trip through the decoder like the torch
restatement's encode of the same clip."""
import hashlib

import numpy as np
import pytest

from test_host import _clip

pytestmark = pytest.mark.gpu

NAMES = ["golden_quantized.wvv", "golden_float.wvv", "golden_stereo.wvv", "smooth_hq.wvv",
         "smooth_lossless.wvv", "noise_bs16.wvv", "smooth_n8.wvv", "smooth_n1_mono.wvv",
         "wide_equirect.wvv"]


def _encode_bytes(name, manifest, tmp_path, backend):
    from paper_2208_10859_b200.encoding import EncodeParams, MappingKind, encode_video
    from paper_2208_10859_b200.fileio import write_video
    spec = dict(manifest[name]["params"])
    spec["mapping"] = MappingKind[spec.get("mapping", "EQUIRECTANGULAR")]
    out = tmp_path / f"{backend}.wvv"
    write_video(encode_video(_clip(name), EncodeParams(**spec), device="cuda", backend=backend), out)
    return out.read_bytes()


@pytest.mark.parametrize("name", NAMES)
def test_cuda_encoder_reproduces_reference_bytes(manifest, name, tmp_path):
    data = _encode_bytes(name, manifest, tmp_path, "native")
    assert hashlib.sha256(data).hexdigest() == manifest[name]["sha256"]


def test_cuda_encoder_record_arrays(manifest, tmp_path):
    """keep_arrays: the parallel record arrays rebuilt from the packed bytes
    equal the torch restatement's."""
    import torch
    from paper_2208_10859_b200.encoding import EncodeParams, MappingKind, encode_video
    spec = dict(manifest["golden_stereo.wvv"]["params"])
    spec["mapping"] = MappingKind[spec.get("mapping", "EQUIRECTANGULAR")]
    clip = _clip("golden_stereo.wvv")
    a = encode_video(clip, EncodeParams(**spec), device="cuda", backend="native")
    b = encode_video(clip, EncodeParams(**spec), device="cpu")
    for sa, sb in zip(a.sets, b.sets):
        ra, rb = sa.records, sb.records
        np.testing.assert_array_equal(ra.temporal, rb.temporal)
        np.testing.assert_array_equal(ra.block, rb.block)
        np.testing.assert_array_equal(ra.offset, rb.offset)
        np.testing.assert_array_equal(np.asarray(ra.values), np.asarray(rb.values))
        np.testing.assert_array_equal(sa.extrema, sb.extrema)
    assert torch.cuda.is_available()


def test_cuda_encoder_8k_set_matches_torch():
    """One 8K stereo set (the bench input's first set): native and torch
    restatement (both on the GPU) write identical bytes."""
    import io
    import torch
    from paper_2208_10859_b200.encoding import EncodeParams, MappingKind, encode_video
    from paper_2208_10859_b200.fileio import write_video
    from paper_2208_10859_b200.synthetic import make_synthetic_clip_torch
    clip = make_synthetic_clip_torch(4, 8192, 8192, 3, seed=7, device="cuda", first_frame=0,
                                     total_frames=4)
    p = EncodeParams(alpha=0.1, inter_threshold=0.005, inter_size=4, block_size=32,
                     mapping=MappingKind.EQUIRECTANGULAR, stereo=True, fps=120.0,
                     mask_w=256, mask_h=256)
    outs = []
    for backend in ("native", "torch"):
        v = encode_video(clip, p, device="cuda", keep_arrays=False, backend=backend)
        buf = io.BytesIO()
        write_video(v, buf)
        outs.append(hashlib.sha256(buf.getvalue()).hexdigest())
        del v
        torch.cuda.empty_cache()
    assert outs[0] == outs[1]


@pytest.mark.parametrize("shape,n,quant,mapping", [
    ((4, 64, 64, 4), 4, True, "EQUIRECTANGULAR"),     # 4 channels (generic point kernel)
    ((6, 128, 64, 2), 2, False, "NONE"),              # float records, n = 2, padded last set
    ((16, 64, 128, 1), 16, True, "EQUIRECTANGULAR"),  # n = 16 (run-time temporal depth)
])
def test_cuda_encoder_matches_restatement_other_shapes(shape, n, quant, mapping, tmp_path):
    """Shapes outside the golden fixtures: CUDA encoder bytes == the torch
    restatement's on CPU (itself pinned to the reference bytes)."""
    from paper_2208_10859_b200.encoding import EncodeParams, MappingKind, encode_video
    from paper_2208_10859_b200.fileio import write_video
    clip = np.random.default_rng(21).integers(0, 256, shape, dtype=np.uint8)
    p = EncodeParams(levels=3, inter_size=n, quantize=quant, mapping=MappingKind[mapping],
                     alpha=0.05, inter_threshold=0.002)
    outs = []
    for dev in ("cuda", "cpu"):
        f = tmp_path / f"{dev}.wvv"
        write_video(encode_video(clip, p, device=dev), f)
        outs.append(f.read_bytes())
    assert outs[0] == outs[1]

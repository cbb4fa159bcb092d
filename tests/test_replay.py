"""Trajectory replay harness against fixtures produced by
the reference's wavevid.bench (tests/golden/make_replay_golden.py)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN


@pytest.fixture(scope="module")
def fix():
    return json.load(open(os.path.join(GOLDEN, "replay.json")))


def _pairs():
    # tests/golden/make_replay_golden.py:pairs
    rng = np.random.default_rng(21)
    out = []
    for shape in [(32, 48, 3), (64, 64, 1), (17, 23)]:
        a = rng.integers(0, 256, shape, dtype=np.uint8)
        b = np.clip(a.astype(int) + rng.integers(-9, 10, shape), 0, 255).astype(np.uint8)
        out.append((a, b))
    a = rng.integers(0, 256, (20, 20, 3), dtype=np.uint8)
    out.append((a, a.copy()))
    return out


def test_host_metrics_match_reference(fix):
    from paper_2208_10859_b200.replay import psnr, ssim
    for (a, b), want in zip(_pairs(), fix["metrics"]):
        assert psnr(a, b) == want["psnr"]
        if want["ssim"] is not None:
            assert ssim(a, b) == want["ssim"]


def test_trajectory_roundtrip(tmp_path):
    from paper_2208_10859_b200.replay import BenchError, TrajectoryLog, circle_trajectory
    ref = TrajectoryLog.load(os.path.join(GOLDEN, "trajectory.csv"))
    mine = circle_trajectory(2000.0, 20)
    np.testing.assert_allclose(ref.samples, mine.samples, rtol=1e-9)
    mine.save(tmp_path / "t.csv")
    assert open(tmp_path / "t.csv").read() == open(os.path.join(GOLDEN, "trajectory.csv")).read()
    assert (ref.sample_at(-5.0) == ref.samples[0]).all()
    assert (ref.sample_at(1e9) == ref.samples[-1]).all()
    with pytest.raises(BenchError):
        TrajectoryLog(np.zeros((2, 6)))


@pytest.mark.gpu
@pytest.mark.parametrize("name,frames,size", [("smooth_hq.wvv", 8, 128), ("smooth_n8.wvv", 10, 64)])
@pytest.mark.parametrize("mode", ["full", "viewport", "foveated"])
def test_gpu_replay_matches_reference(fix, name, frames, size, mode):
    import torch
    from paper_2208_10859_b200 import build
    from paper_2208_10859_b200.replay import replay, TrajectoryLog
    from paper_2208_10859_b200.synthetic import make_synthetic_clip
    build.build()
    want = fix["replay"][f"{name}|{mode}"]
    traj = TrajectoryLog.load(os.path.join(GOLDEN, "trajectory.csv"))
    clip = torch.from_numpy(make_synthetic_clip(frames, size)).cuda()
    got = replay(os.path.join(GOLDEN, name), traj, mode=mode, reference=clip).to_dict()
    for k in ("frames", "total_bytes", "total_records", "frame_bytes", "frame_records",
              "compression_ratio"):
        assert got[k] == want[k], k
    for k in ("psnr_db", "ssim"):
        if want[k] is None:
            assert got[k] is None, k
        else:
            assert got[k] == pytest.approx(want[k], rel=1e-9), k

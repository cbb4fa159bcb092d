"""Replay/quality-metric fixtures from the REAL reference (wavevid.bench):

    python tests/golden/make_replay_golden.py      # build container only

Outputs (committed): ``replay.json`` -- psnr/ssim of seeded image pairs,
``replay`` reports (trajectory replay of smooth_hq.wvv and smooth_n8.wvv
against their source clips, timing fields dropped) and ``trajectory.csv``
(TrajectoryLog.save of circle_trajectory).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from wavevid.bench import (TrajectoryLog, circle_trajectory, make_synthetic_clip,  # noqa: E402
                           psnr, replay, ssim)


def pairs():
    rng = np.random.default_rng(21)
    out = []
    for shape in [(32, 48, 3), (64, 64, 1), (17, 23)]:
        a = rng.integers(0, 256, shape, dtype=np.uint8)
        b = np.clip(a.astype(int) + rng.integers(-9, 10, shape), 0, 255).astype(np.uint8)
        out.append((a, b))
    a = rng.integers(0, 256, (20, 20, 3), dtype=np.uint8)
    out.append((a, a.copy()))
    return out


def main():
    res = {"metrics": [], "replay": {}}
    for a, b in pairs():
        res["metrics"].append({"seed_shape": list(a.shape), "psnr": psnr(a, b),
                               "ssim": ssim(a, b) if min(a.shape[:2]) >= 8 else None})
    traj = circle_trajectory(duration_ms=2000.0, steps=20)
    traj.save(os.path.join(HERE, "trajectory.csv"))
    clips = {"smooth_hq.wvv": make_synthetic_clip(8, 128), "smooth_n8.wvv": make_synthetic_clip(10, 64)}
    for name, clip in clips.items():
        for mode in ("full", "viewport", "foveated"):
            d = replay(os.path.join(HERE, name), traj, mode=mode, reference=clip).to_dict()
            for k in ("fps", "mean_ms"):
                d.pop(k)
            res["replay"][f"{name}|{mode}"] = d
    with open(os.path.join(HERE, "replay.json"), "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res["replay"]["smooth_hq.wvv|viewport"], indent=1)[:600])


if __name__ == "__main__":
    main()

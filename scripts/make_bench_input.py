"""Generate the benchmark clips on the CPU (deterministic, no CUDA, no
native library): synthetic content (make_synthetic_clip restated for H x W,
float64 torch on the host) encoded with the package's torch restatement of
the reference encoder (byte-identical to the reference, tests/test_host.py;
set 0 of the 8K clip is pinned against the reference encoder itself by
tests/golden/bench_8k.json).

    python scripts/make_bench_input.py c3 OUT.wvv      # 8192x8192 stereo, 4 sets
    python scripts/make_bench_input.py c2 OUT.wvv      # 4096x2048 mono, 4 sets

bench.py runs this in a subprocess when the clip is not cached yet, so
neither arm's own process encodes anything.
"""
from __future__ import annotations

import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# config -> (width, height, stereo, sets, mask)
CONFIGS = {
    "c3": (8192, 8192, True, 4, 256),
    "c2": (4096, 2048, False, 4, 64),
}


def clip_frames(cfg: str, set_index: int):
    """u8 (4, H, W, 3) frames of one set, on the host."""
    from paper_2208_10859_b200.synthetic import make_synthetic_clip_torch
    w, h, _, n_sets, _ = CONFIGS[cfg]
    return make_synthetic_clip_torch(4, h, w, 3, seed=7, device="cpu",
                                     first_frame=4 * set_index, total_frames=4 * n_sets)


def params_for(cfg: str):
    from paper_2208_10859_b200.encoding import EncodeParams, MappingKind
    w, h, stereo, _, m = CONFIGS[cfg]
    return EncodeParams(alpha=0.1, inter_threshold=0.005, inter_size=4, block_size=32,
                        mapping=MappingKind.EQUIRECTANGULAR, stereo=stereo, fps=120.0,
                        mask_w=m, mask_h=m)


def make(cfg: str, path: str, sets: int | None = None) -> None:
    import torch
    from paper_2208_10859_b200.encoding import encode_video
    from paper_2208_10859_b200.fileio import write_video
    torch.set_num_threads(max(1, len(os.sched_getaffinity(0))))
    n_sets = CONFIGS[cfg][3] if sets is None else sets
    all_sets, video = [], None
    for si in range(n_sets):
        t0 = time.perf_counter()
        frames = clip_frames(cfg, si)
        v = encode_video(frames, params_for(cfg), device="cpu", keep_arrays=False)
        all_sets.extend(v.sets)
        video = v
        print(f"[make_bench_input] {cfg} set {si}: {time.perf_counter() - t0:.1f} s",
              file=sys.stderr, flush=True)
    video.sets = all_sets
    video.frame_count = 4 * n_sets
    video.pad_frames = 0
    os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
    tmp = path + f".tmp{os.getpid()}"
    write_video(video, tmp)
    os.replace(tmp, path)


# ------------------------------------------------------------ display schedule

TRAJ_MS, TRAJ_STEPS = 2000.0, 240


def trajectory_table():
    """circle_trajectory (bench.py:241-250) sampled finely enough that every
    120 Hz display step gets its own head pose."""
    from paper_2208_10859_b200.replay import circle_trajectory
    return circle_trajectory(TRAJ_MS, TRAJ_STEPS)


def display_step(step: int, frame_count: int, fps: float = 120.0, traj=None):
    """Display step -> (frame, yaw, pitch, roll, gaze_u, gaze_v): frames
    cycle through the clip while the head pose walks the trajectory (as
    bench.replay, bench.py:168-171, with time = step / fps)."""
    traj = traj or trajectory_table()
    t_ms = (step * 1000.0 / fps) % TRAJ_MS
    _, yaw, pitch, roll, gu, gv = traj.sample_at(t_ms)
    return step % frame_count, float(yaw), float(pitch), float(roll), float(gu), float(gv)


# ------------------------------------------------------------ committed clips

GOLDEN = os.path.join(ROOT, "tests", "golden")
CLIP_FILES = {"c3": "bench_c3_8k.wvv.xz", "c2": "bench_c2.wvv.xz"}


def ensure_clip(cfg: str, cache_dir: str) -> str:
    """The committed benchmark clip of ``cfg``, decompressed into
    ``cache_dir`` once and checked against the sha256 in
    tests/golden/bench_8k.json (no encoding, no CUDA)."""
    import hashlib
    import json
    import lzma
    with open(os.path.join(GOLDEN, "bench_8k.json")) as fh:
        want = json.load(fh)["clips"][cfg]["sha256"]
    path = os.path.join(cache_dir, f"{cfg}_{want[:16]}.wvv")
    if os.path.exists(path):
        return path
    with open(os.path.join(GOLDEN, CLIP_FILES[cfg]), "rb") as fh:
        data = lzma.decompress(fh.read())
    got = hashlib.sha256(data).hexdigest()
    if got != want:
        raise RuntimeError(f"{CLIP_FILES[cfg]}: sha256 {got} != bench_8k.json {want}")
    os.makedirs(cache_dir, exist_ok=True)
    tmp = path + f".tmp{os.getpid()}"
    with open(tmp, "wb") as fh:
        fh.write(data)
    os.replace(tmp, path)
    return path


if __name__ == "__main__":
    make(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else None)

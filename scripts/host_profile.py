"""Host-side cost of one decode_render_device call (the bench's headline
path): cProfile over N frames after warm-up.  Run on the GPU box:
    python scripts/host_profile.py [N]"""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
import torch  # noqa: E402

import paper_2208_10859_b200 as wv  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 400
    path = bench.input_path(type("A", (), {"cache_dir": "/tmp/wvb200_bench", "size": 8192})(), 2)
    import os
    if not os.path.exists(path):
        bench.make_input(path, 8192, 2, torch.device("cuda"))
    s = wv.DecodeSession(path)
    h = s.header
    frames = list(range(h.frame_count))
    pm = bench.poses_and_masks(h, frames)
    out = torch.empty((2, bench.OUT_H, bench.OUT_W, 3), dtype=torch.uint8, device="cuda")
    for i in range(20):
        f = frames[i % len(frames)]
        s.decode_render_device(f, "viewport", pm[f][1], pm[f][0], (bench.OUT_W, bench.OUT_H), out)
    torch.cuda.synchronize()
    t = time.perf_counter()
    pr = cProfile.Profile()
    pr.enable()
    for i in range(n):
        f = frames[i % len(frames)]
        s.decode_render_device(f, "viewport", pm[f][1], pm[f][0], (bench.OUT_W, bench.OUT_H), out)
    pr.disable()
    torch.cuda.synchronize()
    print(f"{(time.perf_counter() - t) / n * 1e6:.1f} us/frame wall (profiled)")
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()

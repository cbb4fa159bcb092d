"""K4 kernel time per call for viewport vs foveated decodes (events around
the launch only, GPU kept busy while the host enqueues)."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import torch  # noqa: E402

import paper_2208_10859_b200 as wv  # noqa: E402

path = bench.input_path(type("A", (), {"cache_dir": "/tmp/wvb200_bench", "size": 8192})(), 2)
s = wv.DecodeSession(path)
h = s.header
pm = bench.poses_and_masks(h, list(range(h.frame_count)))
out = torch.empty((2, 2000, 2000, 3), dtype=torch.uint8, device="cuda")
for mode, cov in (("viewport", False), ("foveated", True), ("foveated", False), ("viewport", True)):
    ts = []
    for f in range(8):
        pose, mask, gaze = pm[f]
        if mode == "viewport":
            s.decode_viewport_device(f, mask)
        else:
            s.decode_foveated_device(f, mask, wv.FoveationSchedule.default(h.levels, *gaze))
        with torch.cuda.stream(s.stream):
            torch.cuda._sleep(400000)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        s.render_views(pose, (2000, 2000), out=out, check=False, all_covered=cov, events=(e0, e1))
        torch.cuda.synchronize()
        ts.append(round(e0.elapsed_time(e1) * 1000, 1))
    print(mode, "all_covered" if cov else "footprint", ts, "uncovered", s.uncovered(reset=True))

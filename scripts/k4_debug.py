import sys, time
sys.path.insert(0, ".")
import bench, torch
import paper_2208_10859_b200 as wv
path = bench.input_path(type("A", (), {"cache_dir": "/tmp/wvb200_bench", "size": 8192})(), 2)
s = wv.DecodeSession(path)
h = s.header
pm = bench.poses_and_masks(h, list(range(h.frame_count)))
out = torch.empty((2, 2000, 2000, 3), dtype=torch.uint8, device="cuda")
for mode in ("viewport", "foveated", "foveated", "viewport"):
    for f in range(4):
        pose, mask, gaze = pm[f]
        if mode == "viewport":
            s.decode_viewport_device(f, mask)
        else:
            s.decode_foveated_device(f, mask, wv.FoveationSchedule.default(h.levels, *gaze))
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s.stream)
        s.render_views(pose, (2000, 2000), out=out, check=False, all_covered=(mode == "foveated"))
        e1.record(s.stream)
        torch.cuda.synchronize()
        print(mode, f, round(e0.elapsed_time(e1), 3), "uncovered", s.uncovered(reset=True))

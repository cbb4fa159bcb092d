"""Host cost per decode_render_device call on the 8K bench clip, per mode
(idle GPU, one frame repeated so the set cache never evicts), with a
per-function split."""
import cProfile, os, pstats, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch
import make_bench_input as mbi
import paper_2208_10859_b200 as wv

path = mbi.ensure_clip("c3", os.path.join(ROOT, "gpurun_out", "clip_cache"))
s = wv.DecodeSession(path)
s.time_stages = False
h = s.header
poses = [wv.CameraPose(yaw=-60 + 2 * i, pitch=10) for i in range(8)]
masks = [wv.stereo_mask(p, (h.mask_w, h.mask_h)) for p in poses]
out = torch.empty((2, 2000, 2000, 3), dtype=torch.uint8, device="cuda")
for mode in ("viewport", "foveated", "viewport"):
    sc = wv.FoveationSchedule.default(h.levels, 0.5, 0.5) if mode == "foveated" else None
    call = lambda i: s.decode_render_device(0, mode, masks[i % 8], poses[i % 8], (2000, 2000), out, schedule=sc)
    for i in range(16): call(i)
    torch.cuda.synchronize(); s._settle_until(None)
    ts = []
    for i in range(8):
        t = time.perf_counter(); call(i); ts.append((time.perf_counter() - t) * 1e6)
    torch.cuda.synchronize(); s._settle_until(None)
    print(mode, " ".join(f"{x:.0f}" for x in ts))
    pr = cProfile.Profile(); pr.enable()
    for i in range(8): call(i)
    pr.disable()
    torch.cuda.synchronize(); s._settle_until(None)
    pstats.Stats(pr).sort_stats("tottime").print_stats(8)

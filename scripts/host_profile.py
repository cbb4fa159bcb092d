"""Host-side cost of one decode_render_device call (the bench's headline
path), isolated from GPU time: a small stereo file (tests/golden/
golden_stereo.wvv, so the kernels are short), cProfile over N frames after
warm-up, plus the unprofiled wall time per frame.  Run on the GPU box:
    python scripts/host_profile.py [N] [viewport|foveated|full]"""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2208_10859_b200 as wv  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 400
    mode = sys.argv[2] if len(sys.argv) > 2 else "viewport"
    s = wv.DecodeSession(os.path.join(ROOT, "tests", "golden", "golden_stereo.wvv"))
    s.time_stages = False
    h = s.header
    poses = [wv.CameraPose(yaw=-60 + 0.5 * i, pitch=10) for i in range(64)]
    masks = [wv.stereo_mask(p, (h.mask_w, h.mask_h)) for p in poses]
    out = torch.empty((2, 256, 256, 3), dtype=torch.uint8, device="cuda")
    sc = wv.FoveationSchedule.default(h.levels, 0.5, 0.5) if mode == "foveated" else None

    def run(k):
        for i in range(k):
            if mode == "full":
                s.decode_full_device(i % h.frame_count)
            else:
                s.decode_render_device(i % h.frame_count, mode, masks[i % 64], poses[i % 64],
                                       (256, 256), out, schedule=sc)

    run(80)
    torch.cuda.synchronize()
    s._settle_until(None)
    # fewer frames than the session's result ring, GPU idle at the start:
    # nothing pushes back on the host, so this is the enqueue cost alone
    t = time.perf_counter()
    run(48)
    host = (time.perf_counter() - t) / 48 * 1e6
    torch.cuda.synchronize()
    s._settle_until(None)
    print(f"{host:.1f} us/frame host enqueue (unprofiled, no back-pressure)")
    pr = cProfile.Profile()
    pr.enable()
    run(n)
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(22)


if __name__ == "__main__":
    main()

"""Small decode workload for compute-sanitizer (memcheck / racecheck /
synccheck): every mode, device render path, span fetch, on golden files.
    compute-sanitizer --tool racecheck python scripts/sanitize.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_10859_b200 as wv  # noqa: E402

G = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def main():
    for name, residency in (("golden_stereo.wvv", "set"), ("smooth_hq.wvv", "spans"),
                            ("noise_bs16.wvv", "set"), ("wide_equirect.wvv", "set")):
        s = wv.DecodeSession(os.path.join(G, name), residency=residency)
        h = s.header
        s.use_graphs = False
        pose = wv.CameraPose(yaw=40, pitch=20)
        mask = (wv.stereo_mask if h.stereo else wv.viewport_to_mask)(pose, (h.mask_w, h.mask_h))
        s.decode_full(0)
        s.decode_viewport(min(1, h.frame_count - 1), mask)
        s.decode_foveated(0, mask, wv.FoveationSchedule.default(h.levels, 0.3, 0.6))
        nv = 2 if h.stereo else 1
        out = torch.empty((nv, 96, 128, h.channels), dtype=torch.uint8, device="cuda")
        s.decode_render_device(0, "viewport", mask, pose, (128, 96), out).result()
        s.render_views(pose, (64, 64), check=False)
        torch.cuda.synchronize()
        print(name, "ok")


if __name__ == "__main__":
    main()

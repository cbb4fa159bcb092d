"""Time the CUDA encoder on one 8K stereo set (device-resident input):
python scripts/encode_time.py [reps]"""
import sys
import time

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
from paper_2208_10859_b200.encoding import EncodeParams, MappingKind, encode_video  # noqa: E402
from paper_2208_10859_b200.synthetic import make_synthetic_clip_torch  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
clip = make_synthetic_clip_torch(4, 8192, 8192, 3, seed=7, device="cuda", first_frame=0,
                                 total_frames=4)
p = EncodeParams(alpha=0.1, inter_threshold=0.005, inter_size=4, block_size=32,
                 mapping=MappingKind.EQUIRECTANGULAR, stereo=True, fps=120.0, mask_w=256, mask_h=256)
for backend in ("native", "torch"):
    for i in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        v = encode_video(clip, p, device="cuda", keep_arrays=False, backend=backend)
        torch.cuda.synchronize()
        print(backend, i, f"{(time.perf_counter() - t0) * 1000:.1f} ms",
              len(v.sets[0].records.packed))
        del v

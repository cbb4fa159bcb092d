"""Encoder measurement: one 8K stereo set (4 frames,
8192x8192x3, the C3 bench input's first set) through the CUDA encoder.

    python scripts/bench_encode.py [--steps K] [--warmup W] [--no-cpu-baseline]

Prints one JSON line like bench.py's: `value` = sets/s with the frames
resident in HBM (CUDA events around wv_encode_set, the L2 is flushed between
steps by the 3.2 GB working set itself), `e2e` = the public call
encode_video() from pinned host frames to the host-side packed set (H2D of
the frames and D2H of records, counts and extrema inside the timed region),
`roofline` = algorithmic bytes of the whole encode / its time against the
measured HBM peak, `cpu_baseline` = the torch restatement (byte-identical to
the reference encoder) on host cores over a bounded 1024x1024 sample, scaled
to samples/s.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402  (ClockSampler, peaks)
from paper_2208_10859_b200 import _native as nat  # noqa: E402
from paper_2208_10859_b200.encoding import (EncodeParams, MappingKind, encode_video,  # noqa: E402
                                            equirect_mapping_factors, temporal_level_of,
                                            threshold_value)
from paper_2208_10859_b200.synthetic import make_synthetic_clip_torch  # noqa: E402

N, SIZE, C3 = 4, 8192, 3


def params():
    return EncodeParams(alpha=0.1, inter_threshold=0.005, inter_size=N, block_size=32,
                        mapping=MappingKind.EQUIRECTANGULAR, stereo=True, fps=120.0,
                        mask_w=256, mask_h=256)


def algorithmic_bytes(n, h, w, c, levels):
    """Bytes an encode must move: level-1 rows read u8 and write f32, every
    other lifting pass reads and writes its level region in f32, the point
    pass reads the pyramid once; records and tables are < 1%."""
    s = n * h * w * c
    total = s * 1 + s * 4            # level-1 rows: u8 in, f32 out
    total += 8 * s                   # level-1 columns
    for k in range(2, levels + 1):
        total += 2 * 8 * s / 4 ** (k - 1)
    total += 4 * s                   # point pass read (nonzero write-back is sparse)
    return total


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    p = params()
    levels = p.resolved_levels(SIZE, SIZE)
    clip = make_synthetic_clip_torch(N, SIZE, SIZE, C3, seed=7, device=dev, first_frame=0,
                                     total_frames=N)
    lib = nat.load()
    ep = nat.EncodeParams()
    ep.width = ep.height = SIZE
    ep.channels, ep.levels, ep.inter_size, ep.block_size, ep.quantize = C3, levels, N, 32, 1
    for k in range(1, levels + 1):
        ep.level_threshold[k - 1] = float(np.float32(threshold_value(p.alpha, k - 1, levels)))
    for ti in range(1, N):
        ep.temporal_threshold[ti] = float(np.float32(threshold_value(
            p.inter_threshold, temporal_level_of(ti, N) - 1, int(np.log2(N)))))
    ws_b, cap = C.c_uint64(), C.c_uint64()
    nat.check(lib.wv_encode_workspace_bytes(C.byref(ep), C.byref(ws_b)), "ws")
    nat.check(lib.wv_encode_payload_capacity(C.byref(ep), C.byref(cap)), "cap")
    ws = torch.empty(ws_b.value, dtype=torch.uint8, device=dev)
    payload = torch.empty(cap.value, dtype=torch.uint8, device=dev)
    rowf = torch.as_tensor(equirect_mapping_factors(SIZE), device=dev)
    nb = (SIZE // 32) ** 2
    ext = torch.empty((N, C3, 4), dtype=torch.float32, device=dev)
    counts = torch.empty((N, nb), dtype=torch.int32, device=dev)
    nrec = torch.zeros(1, dtype=torch.int64, device=dev)
    frames = clip.contiguous()
    stream = torch.cuda.current_stream(dev)

    def once():
        nat.check(lib.wv_encode_set(C.byref(ep), C.c_void_p(frames.data_ptr()),
                                    C.c_void_p(rowf.data_ptr()), C.c_void_p(ws.data_ptr()),
                                    C.c_uint64(ws_b.value), C.c_void_p(ext.data_ptr()),
                                    C.c_void_p(counts.data_ptr()), C.c_void_p(payload.data_ptr()),
                                    C.c_uint64(cap.value), C.c_void_p(nrec.data_ptr()),
                                    C.c_void_p(stream.cuda_stream)), "wv_encode_set")

    for _ in range(args.warmup):
        once()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with bench.ClockSampler(0) as clk:
        for a, b in evs:
            a.record(stream)
            once()
            b.record(stream)
        torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    n_records = int(nrec.item())

    # e2e: the public API from pinned host frames to host-side records
    host = clip.cpu().pin_memory()
    del ws, payload
    torch.cuda.empty_cache()
    e2e_ms = []
    for i in range(args.warmup + max(3, args.steps // 4)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        v = encode_video(host, p, device=dev, keep_arrays=False)
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e_ms.append((time.perf_counter() - t0) * 1000.0)
        payload_bytes = len(v.sets[0].records.packed)
        del v
    e2e = float(np.median(e2e_ms))

    peak, peak_kind = bench.peaks()
    alg = algorithmic_bytes(N, SIZE, SIZE, C3, levels)
    achieved = alg / (ms * 1e-3) / 1e9
    samples = N * SIZE * SIZE * C3
    cpu = None
    if not args.no_cpu_baseline:
        sub = clip[:, :1024, :1024].cpu()
        sp = EncodeParams(alpha=0.1, inter_threshold=0.005, inter_size=N, block_size=32,
                          mapping=MappingKind.EQUIRECTANGULAR, levels=3)
        t0 = time.perf_counter()
        encode_video(sub, sp, device="cpu", keep_arrays=False)
        el = time.perf_counter() - t0
        cpu = {"value": round(sub.numel() / el / 1e6, 3), "unit": "Msamples/s",
               "cores": torch.get_num_threads(), "kind": "port",
               "sample": f"one 4-frame 1024x1024x3 set (L3), torch CPU restatement of the "
                         f"reference encoder (byte-identical output), {el:.2f} s"}
    line = {
        "metric": "8K stereo sets encoded/s (4 frames, 8192x8192x3)",
        "value": round(1000.0 / ms, 2), "unit": "sets/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "Msamples_per_s": round(samples / (ms * 1e-3) / 1e6, 1),
        "dtype": "f32", "data": "synthetic (make_synthetic_clip, seed 7)",
        "config": {"workload": "encode one 4-frame 8192x8192x3 stereo set, L6, alpha 0.1, "
                               "inter 0.005, equirect, u8 records",
                   "records": n_records, "payload_bytes": payload_bytes,
                   "l2": "3.2 GB f32 working set per step (> L2)"},
        "roofline": {"bound": "hbm", "kernel": "whole encode (13 launches)",
                     "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "peak_kind": peak_kind,
                     "algorithmic_bytes": int(alg)},
        "e2e": {"value": round(1000.0 / e2e, 2), "unit": "sets/s",
                "h2d_bytes_per_step": samples, "d2h_bytes_per_step": payload_bytes + N * nb * 8},
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "gpu_launches": args.steps * (2 * levels + 7),
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()

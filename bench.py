#!/usr/bin/env python
"""Headline benchmark: 8192x8192 stereo 360-degree viewport decode on B200.

Workload (BASELINE.json configs[2]): a synthetic
8192x8192x3 top-bottom stereo clip of 4 inter-frame sets / 16 frames
(make_synthetic_clip restated for HxW, encoded with the reference
encoder's algorithm: alpha 0.1, beta 0.005, n 4, 32-px blocks, 6 levels,
256x256 mask grid, 120 fps header; committed as
tests/golden/bench_c3_8k.wvv.xz, set 0 pinned against the reference
encoder and 9 decodes pinned against the reference decoder in
tests/golden/bench_8k.json).  One step = one display frame: step i shows
frame i mod 16 under the head pose of the circle trajectory at time
i / 120 s (a new pose every step) -> stereo viewport mask (90x90 FOV) ->
K1 select -> K2 dequant+temporal -> K3 6-level synthesis into the u8
canvas -> K4 per-eye perspective writeout to 2000x2000.  Inputs are
resident in HBM for ``value``; ``e2e`` adds the host->device set payload
and the device->host result every step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--config c3|c2] [--mode viewport|foveated|full]

N>1 runs under torchrun: sets are sharded round-robin over ranks (weak
scaling), and every step gathers each rank's two eye images to rank 0 over
NCCL (the display GPU), the path's only exchange.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("decoded frames/s (Mpixel/s) for 8K×8K stereo 360° viewport decode "
          "at 1/2/4/8 B200")
OUT_W = OUT_H = 2000
FPS = 120.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=["c3", "c2"], default="c3",
                    help="c3: 8192x8192 stereo (configs 3-5); c2: 4096x2048 mono (config 2)")
    ap.add_argument("--mode", choices=["viewport", "foveated", "full"], default=None,
                    help="default: viewport for c3, full for c2")
    ap.add_argument("--clip", default=None, help="decode this .wvv instead of the config's clip")
    ap.add_argument("--tile-strips", type=int, choices=[1, 2], default=None,
                    help="K3 tile width in 28-column strips (default: 2 for full mode, else 1)")
    ap.add_argument("--cache-dir", default="/tmp/wvb200_bench")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--pipeline", type=int, default=8,
                    help="decode sessions (streams) per GPU; frames round-robin so one "
                         "frame's writeout overlaps the next frame's decode")
    ap.add_argument("--residency", choices=["set", "spans"], default="set",
                    help="spans: only BlockEnd tables are uploaded; the GPU fetches the record "
                         "spans of selected blocks from pinned host memory (load_blocks)")
    ap.add_argument("--split", choices=["sets", "eyes"], default="sets",
                    help="N>1: sets round-robin over ranks (both eyes each), or rank pairs "
                         "splitting the stereo eyes of each frame (sets round-robin over pairs)")
    ap.add_argument("--profile-only", action="store_true",
                    help="a few decodes for ncu; prints nothing")
    return ap.parse_args()


# ------------------------------------------------------------------ inputs

sys.path.insert(0, os.path.join(ROOT, "scripts"))
import make_bench_input as mbi  # noqa: E402  (stdlib-only at import)


def clip_for(args) -> str:
    """The committed benchmark clip (decompressed once into the cache dir),
    or --clip."""
    return args.clip or mbi.ensure_clip(args.config, args.cache_dir)


class Schedule:
    """Display step -> (frame, pose, mask, gaze): frames cycle through
    ``frames`` while the head walks the circle trajectory at 120 Hz
    (scripts/make_bench_input.display_step), so consecutive steps -- and
    the sessions they land on -- never repeat an input.  ``api`` supplies
    CameraPose / stereo_mask / viewport_to_mask (ours, or the reference's
    in the reference arm)."""

    def __init__(self, header, frames, CameraPose, stereo_mask, viewport_to_mask, traj):
        self.h, self.frames, self.traj = header, list(frames), traj
        self.CameraPose, self.stereo_mask, self.viewport_to_mask = (CameraPose, stereo_mask,
                                                                    viewport_to_mask)
        self._masks = {}

    def __call__(self, step: int):
        h = self.h
        _, yaw, pitch, roll, gu, gv = mbi.display_step(step, 1, h.fps or FPS, self.traj)
        frame = self.frames[step % len(self.frames)]
        pose = self.CameraPose(yaw=yaw, pitch=pitch, roll=roll, fov_h=90, fov_v=90)
        key = (yaw, pitch, roll)
        mask = self._masks.get(key)
        if mask is None:
            dims = (h.mask_w, h.mask_h)
            mask = self.stereo_mask(pose, dims) if h.stereo else self.viewport_to_mask(pose, dims)
            self._masks[key] = mask
        return frame, pose, mask, (gu, gv)


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]
        else:
            self.lines = []

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            parts = [p.strip() for p in l.split(",")]
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ ours

def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def launches_per_frame(L: int, mode: str, residency: str) -> int:
    """Kernels of one frame's graph (csrc launch sequence): K1 rows, one
    direct cascade launch (all levels), L-1 footprint steps, blocks, tile
    lists (2), finest footprint; K2; K3 L levels; K4 -- full frame: rows,
    footprint fill, blocks, tile lists, K2, K3 (no cascades, footprint chain
    or writeout)."""
    tiles = 1 + (1 if L >= 2 else 0)
    if mode == "full":
        n = 1 + 1 + 1 + tiles + 1 + L
    else:
        n = 1 + 1 + (L - 1) + 1 + tiles + 1 + 1 + L + 1
    return n + (1 if residency == "spans" else 0)


def ncu_traffic(mode: str):
    """DRAM bytes per launch of the K3 finest level from the latest committed
    `ncu --set full` capture of this mode (profiles/ncu_k3_final[_full]_<tag>.json)."""
    import glob
    pat = "ncu_k3_final_full_*.json" if mode == "full" else "ncu_k3_final_r*.json"
    found = sorted(glob.glob(os.path.join(ROOT, "profiles", pat)))
    if not found:
        return None, None
    p = found[-1]
    try:
        with open(p) as fh:
            d = json.load(fh)
        return d.get("dram_bytes_per_launch"), d.get("algorithmic_bytes_per_launch")
    except (OSError, ValueError):
        return None, None


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2208_10859_b200 as wv
    from paper_2208_10859_b200 import build
    from paper_2208_10859_b200.decoding import FoveationSchedule
    from paper_2208_10859_b200.projection import CameraPose, stereo_mask, viewport_to_mask
    from paper_2208_10859_b200.sharding import assign, gather_views
    from paper_2208_10859_b200.replay import circle_trajectory
    from paper_2208_10859_b200 import _native as N

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if rank == 0:
        build.build()
        path = clip_for(args)
    if world > 1:
        dist.barrier()
    if rank != 0:
        path = clip_for(args)
    mode = args.mode

    P = max(1, args.pipeline)
    # whole-frame decodes use the 56-column synthesis tiles (faster there;
    # the viewport headline keeps 28-column tiles)
    strips = args.tile_strips or (2 if mode == "full" else 1)
    sessions = [wv.DecodeSession(path, device=dev, max_resident_sets=8,
                                 residency=args.residency, tile_strips=strips)
                for _ in range(P)]
    for s_ in sessions:
        s_.time_stages = False
    sess = sessions[0]
    h = sess.header
    share = assign(h.num_sets, h.inter_size, h.frame_count, rank, world,
                   args.split if mode != "full" else "sets", h.stereo)
    my_sets, frames, eye = share.sets, share.frames, share.eye
    sched = Schedule(h, frames, CameraPose, stereo_mask, viewport_to_mask,
                     circle_trajectory(mbi.TRAJ_MS, mbi.TRAJ_STEPS))
    # every step's inputs are prepared before timing (host pose -> mask work
    # is the caller's, as in bench.replay)
    plan = []
    for i in range(args.warmup + args.steps):
        f, pose, mask, gaze = sched(i)
        sc = FoveationSchedule.default(h.levels, *gaze) if mode == "foveated" else None
        plan.append((f, pose, mask, sc))
    views = (2 if h.stereo else 1) if eye is None else 1
    outs = [torch.empty((views, OUT_H, OUT_W, h.channels), dtype=torch.uint8, device=dev)
            for _ in range(P)]
    out = outs[0]
    # the step's result: the eye images, or the whole decoded canvas in full mode
    results = [s_._canvas if mode == "full" else o for s_, o in zip(sessions, outs)]
    gather_buf = ([torch.empty_like(results[0]) for _ in range(world)]
                  if (world > 1 and rank == 0) else None)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = sess.stream

    def step(i, p_=0):
        ss = sessions[p_]
        f, pose, mask, sc = plan[i]
        if mode == "full":
            ss.decode_full_device(f)
        else:
            ss.decode_render_device(f, mode, mask, pose, (OUT_W, OUT_H), outs[p_], schedule=sc,
                                    eye=eye)

    def gather(p_=0):
        if world > 1:
            with torch.cuda.stream(sessions[p_].stream):
                gather_views(results[p_], rank, world, 0, gather_buf)

    # make every set resident and warm up
    for ss in sessions:
        for s in my_sets:
            ss._make_resident(s)
    for i in range(args.warmup):
        for p_ in range(P):
            step(i, p_)
            gather(p_)
    torch.cuda.synchronize()
    for ss in sessions:
        ss._settle_until(None)
    if args.profile_only:
        return

    # headline: P sessions (streams), steps round-robin, whole-job time from
    # one start event to the join of all streams (per-frame working set
    # ~300 MB of plane/level/canvas traffic > 126 MB L2; no flush needed)
    start_ev = torch.cuda.Event(enable_timing=True)
    end_ev = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        start_ev.record(stream)
        for ss in sessions[1:]:
            ss.stream.wait_event(start_ev)
        t_host = time.perf_counter()
        for i in range(args.steps):
            p_ = i % P
            step(args.warmup + i, p_)
            gather(p_)
        t_host = (time.perf_counter() - t_host) * 1000.0 / args.steps
        for ss in sessions[1:]:
            e = torch.cuda.Event()
            e.record(ss.stream)
            stream.wait_event(e)
        end_ev.record(stream)
        torch.cuda.synchronize()
    pipe_ms = start_ev.elapsed_time(end_ev)
    tp = torch.tensor([pipe_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.barrier()
        dist.all_reduce(tp, op=dist.ReduceOp.MAX)
    max_ms = float(tp.item())
    for ss in sessions:
        ss._settle_until(None)
    unc = sum(ss.uncovered() for ss in sessions)
    # host cost of one frame's enqueue (the public call), measured where the
    # GPU cannot push back: an idle GPU, fewer frames than the session ring
    # (one step's frame repeated: a frame of another set would make the call
    # settle the pending decodes first -- the reference's two-set cache can
    # evict, decoding.py:236-241 -- and time the GPU instead of the host)
    torch.cuda.synchronize()
    sess._settle_until(None)
    nh = min(args.steps, 8)   # few enough that no launch queue fills up
    th = time.perf_counter()
    for i in range(nh):
        step(args.warmup, 0)
    host_enqueue_us = (time.perf_counter() - th) * 1e6 / nh
    torch.cuda.synchronize()
    sess._settle_until(None)

    # serial latency view: one stream, L2 flushed (256 MiB write) before each
    # step, each step bracketed by events
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    torch.cuda.synchronize()
    for i in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        ev[i][0].record(stream)
        step(args.warmup + i)
        gather()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    serial_ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    sess._settle_until(None)

    # per-kernel timing pass (events on the launching stream), L2 flushed
    sess.kernel_timing = True
    sess.kernel_events = []
    frames_out = []
    R = max(5, min(20, args.steps))
    # a GPU-side sleep before each timed stage keeps the stream busy while the
    # host enqueues the stage, so the event intervals hold kernel time only
    busy = int(4e5)   # clock cycles (~0.2 ms)
    if mode != "full":
        # first use of the by-value K4 launch path loads its kernel (lazy module
        # loading): keep that out of the timed frames
        sess.render_views(plan[0][1], (OUT_W, OUT_H), out=out, check=False,
                          all_covered=mode == "foveated")
        torch.cuda.synchronize()
    for i in range(R):
        with torch.cuda.stream(stream):
            flush.zero_()
            torch.cuda._sleep(busy)
        f, pose, mask, sc = plan[i % len(plan)]
        if mode == "full":
            frames_out.append(sess.decode_full_device(f))
        elif mode == "foveated":
            frames_out.append(sess.decode_foveated_device(f, mask, sc))
        else:
            frames_out.append(sess.decode_viewport_device(f, mask))
        if mode != "full":
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                torch.cuda._sleep(busy)
            sess.render_views(pose, (OUT_W, OUT_H), out=out, check=False,
                              all_covered=mode == "foveated", events=(e0, e1))
            sess.kernel_events[-1].extend([e0, e1])
    torch.cuda.synchronize()
    sess.kernel_timing = False
    ks = sess.kernel_events
    mean = lambda xs: sum(xs) / len(xs)
    k1 = mean([e[0].elapsed_time(e[1]) for e in ks])
    k2 = mean([e[1].elapsed_time(e[2]) for e in ks])
    k3m = mean([e[2].elapsed_time(e[3]) for e in ks])
    k3f = mean([e[3].elapsed_time(e[4]) for e in ks])
    k4 = mean([e[5].elapsed_time(e[6]) for e in ks]) if mode != "full" else 0.0
    k2_items = int(len(sess.block_work()))   # last frame's K2 work list
    lvl_tiles = sess.tile_counts()             # last frame's synthesis tiles per level
    records = mean([fo.result().records for fo in frames_out])
    tiles = mean([fo.result().n_tiles for fo in frames_out])
    sel_blocks = mean([fo.result().n_selected for fo in frames_out])
    C = h.channels
    # K3 finest level, per launch: read 4 subband tiles (ty x tx f32 each per
    # channel, 32 x 28) and write a 2ty x 2tx u8 tile per channel (SURVEY §8d
    # K3+K4 terms)
    ty, tx = N.synthesis_tile(sess._lib)
    alg = tiles * (4 * ty * tx * 4 * C + 4 * ty * tx * C)
    peak, peak_kind = peaks()
    achieved = alg / (k3f * 1e-3) / 1e9
    # whole display frame, SURVEY §8(d) byte model over the work actually done:
    # K2 = BlockEnd spans (8 B x n) + records (2 + C B, u8) + dense f32 block
    # write; K3 level k >= 2 = 4 subband tiles read + 2ty x 2tx f32 written per
    # tile-channel; K3 level 1 = `alg`; K4 = C B canvas read + C B written
    # per output pixel.  K1's bit masks (~3 MB) are left out.
    out_px_frame = views * OUT_W * OUT_H if mode != "full" else 0
    frame_bytes = (k2_items * (8 * h.inter_size + 4 * C * h.block_size ** 2)
                   + records * (2 + C)
                   + sum(lvl_tiles[1:]) * (4 * ty * tx * 4 + 4 * ty * tx * 4) * C
                   + alg + 2 * C * out_px_frame)
    traffic, _ = ncu_traffic(mode)

    # end-to-end through the public API with host buffers: every step copies
    # its set payload + mask from pinned host memory and reads the step's
    # result (the two eye images; in full mode the decoded u8 canvas, as
    # decode_full returns it, decoding.py:328-331) back into pinned host
    # memory, with the same pipelining as the headline
    e2e = None
    if not args.no_e2e:
        pinned = {s: sess.pinned_payload(s) for s in my_sets}
        host_outs = [torch.empty(r.shape, dtype=torch.uint8).pin_memory() for r in results]
        bi = bo = 0
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e_start = torch.cuda.Event(enable_timing=True)
        e_end = torch.cuda.Event(enable_timing=True)
        e_start.record(stream)
        for ss in sessions[1:]:
            ss.stream.wait_event(e_start)
        fetched0 = sum(ss.bytes_fetched for ss in sessions)
        for i in range(args.steps):
            p_ = i % P
            ss = sessions[p_]
            s = plan[args.warmup + i][0] // h.inter_size
            # whole payload ("set") or BlockEnd table + spans fetched by the
            # decode ("spans", counted after the run)
            ss.upload_set(s, pinned[s])
            step(args.warmup + i, p_)
            gather(p_)
            with torch.cuda.stream(ss.stream):
                host_outs[p_].copy_(results[p_], non_blocking=True)
            bi += (pinned[s].numel() if args.residency == "set" else ss.table_upload_bytes)
            bi += h.mask_w * h.mask_h if mode != "full" else 0
            bo += host_outs[p_].numel()
        for ss in sessions[1:]:
            e = torch.cuda.Event()
            e.record(ss.stream)
            stream.wait_event(e)
        e_end.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([e_start.elapsed_time(e_end)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        for ss in sessions:
            ss._settle_until(None)
        bi += sum(ss.bytes_fetched for ss in sessions) - fetched0
        e2e = {"value": round(world * share.frames_per_step * args.steps /
                              (float(te.item()) / 1000.0), 2),
               "unit": "frames/s",
               "h2d_bytes_per_step": bi // args.steps, "d2h_bytes_per_step": bo // args.steps,
               "result": "decoded u8 canvas (C, H, W)" if mode == "full"
                         else "per-eye perspective images"}
        # the link the e2e rate is bound by: plain device->pinned-host copies of
        # the same result buffers, same streams, no decode
        r0 = torch.cuda.Event(enable_timing=True)
        r1 = torch.cuda.Event(enable_timing=True)
        nrep = min(args.steps, 64 if mode != "full" else 16)
        torch.cuda.synchronize()
        r0.record(stream)
        for ss in sessions[1:]:
            ss.stream.wait_event(r0)
        for i in range(nrep):
            p_ = i % P
            with torch.cuda.stream(sessions[p_].stream):
                host_outs[p_].copy_(results[p_], non_blocking=True)
        for ss in sessions[1:]:
            e = torch.cuda.Event()
            e.record(ss.stream)
            stream.wait_event(e)
        r1.record(stream)
        torch.cuda.synchronize()
        d2h_gbs = nrep * host_outs[0].numel() / (r0.elapsed_time(r1) * 1e-3) / 1e9
        e2e["d2h_link_gbs"] = round(d2h_gbs, 1)
        e2e["d2h_link_frac"] = round(e2e["value"] * (bo / args.steps) / (d2h_gbs * 1e9), 4)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(path, [plan[args.warmup + i] for i in range(3)], mode)

    if rank == 0:
        fps = world * share.frames_per_step * args.steps / (max_ms / 1000.0)
        out_px = ((2 if h.stereo else 1) * OUT_W * OUT_H if mode != "full"
                  else h.width * h.height)
        stereo = "stereo" if h.stereo else "mono"
        workload = (f"{args.config.upper()} {h.width}x{h.height} {stereo} 360 {mode} decode + "
                    f"per-eye {OUT_W}x{OUT_H} perspective writeout, 90x90 FOV, circle trajectory"
                    if mode != "full" else
                    f"{args.config.upper()} {h.width}x{h.height} {stereo} full-frame decode"
                    + (" (config 5 per GPU)" if args.config == "c3" else ""))
        metric = (METRIC if (args.config, mode) == ("c3", "viewport")
                  else f"decoded frames/s (Mpixel/s) for {workload}")
        line = {
            "metric": metric,
            "value": round(fps, 2),
            "unit": "frames/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(max_ms / args.steps, 4),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f32",
            "data": ("synthetic: make_synthetic_clip restated for HxW, encoded with the reference "
                     "encoder's algorithm (committed clip; set 0 byte-identical to the reference "
                     "encoder, decodes pinned to the reference, tests/golden/bench_8k.json)"),
            "serial_ms_per_frame": round(serial_ms, 4),
            "host_ms_per_step": round(t_host, 4),
            "host_enqueue_us": round(host_enqueue_us, 1),
            "config": {
                "workload": workload,
                "levels": h.levels, "inter_size": h.inter_size, "block_size": h.block_size,
                "mask": f"{h.mask_w}x{h.mask_h}", "alpha": 0.1, "inter_threshold": 0.005,
                "sets": h.num_sets, "frames": h.frame_count, "sets_per_rank": len(my_sets),
                "schedule": ("step i: frame i mod frames, head pose of circle_trajectory(2000 ms, "
                             "240 samples) at i/120 s"),
                "l2": ("headline: per-frame working set (~300 MB plane/level/canvas traffic) "
                       "exceeds the 126 MB L2; serial_ms_per_frame: L2 flushed (256 MiB write) "
                       "before every step"),
                "pipeline": f"{P} decode sessions (CUDA streams) per GPU, steps round-robin",
                "residency": args.residency,
                "synthesis_tile": f"{ty}x{tx} coefficients ({strips} warp strip(s))",
                "parallelism": ((f"sets round-robin over {world} GPU(s), "
                                 if eye is None else
                                 f"stereo eyes split over rank pairs, sets round-robin over "
                                 f"{world // 2} pair(s), ")
                                + ("decoded canvas" if mode == "full" else "eye images")
                                + " gathered to rank 0"),
            },
            "mpix_per_s": round(fps * out_px / 1e6, 1),
            "roofline": {"bound": "hbm", "kernel": "k_level<FINAL> (K3 finest level + u8 writeout)",
                         "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic, "algorithmic_bytes_per_launch": int(alg),
                         "launch_ms": round(k3f, 4)},
            "frame_roofline": {"bytes_per_frame": int(frame_bytes),
                               "fps_at_peak": round(peak * 1e9 / frame_bytes, 1),
                               "frac": round(fps * frame_bytes / (peak * 1e9), 4),
                               "tiles_per_level": lvl_tiles,
                               "model": "SURVEY 8(d) bytes over the work done (K2 spans+records+"
                                        "dense blocks, K3 tiles per level, K4 canvas read + "
                                        "output write; K1 masks excluded), whole job rate"},
            "stage_ms": {"k1_select": round(k1, 4), "k2_dequant_temporal": round(k2, 4),
                         "k3_levels_L_to_2": round(k3m, 4), "k3_level1_final": round(k3f, 4),
                         "k4_perspective": round(k4, 4)},
            "selected_blocks": sel_blocks, "k2_work_blocks": k2_items, "level1_tiles": tiles,
            "uncovered_pixels": unc,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk.summary(),
            "gpu_launches": args.steps * launches_per_frame(h.levels, mode, args.residency),
        }
        print(json.dumps(line), flush=True)
    for ss in sessions:
        ss.close()
    if world > 1:
        dist.destroy_process_group()


# ----------------------------------------------- CPU legs (no CUDA, no .so)

_W = {}


def _oracle_init(path):
    from oracle import wavevid_oracle as wo
    _W["wo"] = wo
    _W["path"] = path


def _oracle_frame(job):
    """One display frame through the CPU oracle (decode + per-eye render)."""
    import numpy as np
    wo = _W["wo"]
    frame, ypr, mask, fractions, gaze, mode = job
    sess = wo.OracleSession(_W["path"])
    h = sess.header
    t0 = time.perf_counter()
    if mode == "full":
        pix, fp, _ = sess.decode(frame, "full")
    elif mode == "foveated":
        pix, fp, _ = sess.decode(frame, "foveated", mask, fractions, gaze)
        fp = np.ones_like(fp)   # the reference's foveated callers (cli.py:177)
    else:
        pix, fp, _ = sess.decode(frame, "viewport", mask)
    if mode != "full":
        rot = wo.pose_rotation(*ypr)
        half = h.height // 2 if h.stereo else h.height
        for e in range(2 if h.stereo else 1):
            wo.perspective(pix[e * half:(e + 1) * half], fp[e * half:(e + 1) * half], rot,
                           90.0, 90.0, OUT_W, OUT_H)
    return time.perf_counter() - t0


def cpu_baseline_sample(path, plan_rows, mode):
    """The oracle port on the host cores: one worker process per sample,
    each warmed by one frame, then the samples timed in parallel."""
    import multiprocessing as mp
    jobs = []
    for f, pose, mask, sc in plan_rows:
        jobs.append((f, (pose.yaw, pose.pitch, pose.roll), mask,
                     sc.fractions if sc is not None else None,
                     (sc.gaze_u, sc.gaze_v) if sc is not None else None, mode))
    n = len(jobs)
    with mp.get_context("spawn").Pool(n, initializer=_oracle_init, initargs=(path,)) as pool:
        pool.map(_oracle_frame, jobs, chunksize=1)
        t0 = time.perf_counter()
        per = pool.map(_oracle_frame, jobs, chunksize=1)
        wall = time.perf_counter() - t0
    return {"value": round(n / wall, 4), "unit": "frames/s", "cores": n, "kind": "port",
            "sample": (f"{n} display frames ({mode} decode"
                       + ("" if mode == "full" else f" + per-eye {OUT_W}x{OUT_H} renders")
                       + f") of the timed schedule, numpy oracle, {n} processes in parallel "
                         f"after one warm-up frame each; per-frame s "
                       + ", ".join(f"{x:.1f}" for x in per))}


def _ref_path():
    return os.path.join(ROOT, "baseline", "_ref")


def _ref_init(path):
    sys.path.insert(0, _ref_path())
    import wavevid
    _W["wv"] = wavevid
    _W["sess"] = wavevid.DecodeSession(path)


def _ref_frame(job):
    """One display frame through the UNMODIFIED reference package
    (baseline/_ref): DecodeSession.decode_* then render_perspective per eye,
    timed with perf_counter as bench.replay does (bench.py:178-185)."""
    import numpy as np
    wv = _W["wv"]
    sess = _W["sess"]
    frame, ypr, mask, fractions, gaze, mode = job
    h = sess.header
    pose = wv.CameraPose(yaw=ypr[0], pitch=ypr[1], roll=ypr[2], fov_h=90, fov_v=90)
    t0 = time.perf_counter()
    if mode == "full":
        pix, fp, _ = sess.decode_full(frame)
    elif mode == "foveated":
        pix, fp, _ = sess.decode_foveated(frame, mask,
                                          wv.FoveationSchedule(tuple(fractions), *gaze))
        fp = np.ones_like(fp)   # cli.py:177, service.py:135
    else:
        pix, fp, _ = sess.decode_viewport(frame, mask)
    uncovered = 0
    if mode != "full":
        half = h.height // 2 if h.stereo else h.height
        for e in range(2 if h.stereo else 1):
            sl = slice(e * half, (e + 1) * half)
            try:
                wv.render_perspective(pix[sl], fp[sl], pose, (OUT_W, OUT_H))
            except wv.CoverageError:   # cli.py:242-245 reports it; count it here
                uncovered += 1
    return time.perf_counter() - t0, _native_of_ours(), uncovered


def _native_of_ours():
    """Shared objects of this repo's package mapped into this process."""
    try:
        with open("/proc/self/maps") as fh:
            return sorted({l.split()[-1] for l in fh
                           if "paper_2208_10859_b200" in l and ".so" in l})
    except OSError:
        return []


def run_reference(args):
    """--impl reference: the reference package itself (baseline/_ref, pure
    Python/numpy, unmodified) on the host cores, one DecodeSession per
    worker process, display frames of the same schedule in parallel.  No
    torch, no CUDA and nothing of paper_2208_10859_b200 is imported."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import multiprocessing as mp
    path = clip_for(args)
    mode = args.mode
    if not os.path.isdir(os.path.join(_ref_path(), "wavevid")):
        print(json.dumps({"impl": "reference",
                          "unavailable": "baseline/_ref missing (pip install --target "
                                         "baseline/_ref of /root/reference/pkg not done)"}))
        return
    sys.path.insert(0, _ref_path())
    import wavevid as rw
    with rw.VideoReader(path) as r:
        h = r.header
    sched = Schedule(h, range(h.frame_count), rw.CameraPose, _ref_stereo_mask(rw),
                     rw.viewport_to_mask, rw.circle_trajectory(mbi.TRAJ_MS, mbi.TRAJ_STEPS))
    cores = len(os.sched_getaffinity(0))
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError):
        avail = 16 << 30
    per = (7 << 30) if h.width * h.height >= (1 << 26) else (2 << 30)
    procs = max(1, min(cores, int(avail // per), args.steps))
    # bounded sample: at most two timed frames per worker (~30 s at 8K)
    n_timed = max(1, min(args.steps, 2 * procs))

    def job(i):
        f, pose, mask, gaze = sched(i)
        fr = None
        if mode == "foveated":
            fr = tuple(rw.FoveationSchedule.default(h.levels, *gaze).fractions)
        return (f, (pose.yaw, pose.pitch, pose.roll), mask, fr, gaze, mode)

    ctx = mp.get_context("spawn")
    with ctx.Pool(procs, initializer=_ref_init, initargs=(path,)) as pool:
        # warm every worker (imports, first set load, first-touch allocations)
        pool.map(_ref_frame, [job(i) for i in range(procs)], chunksize=1)
        t0 = time.perf_counter()
        res = pool.map(_ref_frame, [job(args.warmup + i) for i in range(n_timed)], chunksize=1)
        wall = time.perf_counter() - t0
    fps = n_timed / wall
    ours_loaded = sorted(set(_native_of_ours()).union(*[set(r[1]) for r in res]))
    stereo = "stereo" if h.stereo else "mono"
    workload = (f"{args.config.upper()} {h.width}x{h.height} {stereo} 360 {mode} decode + per-eye "
                f"{OUT_W}x{OUT_H} perspective writeout, 90x90 FOV, circle trajectory"
                if mode != "full" else f"{args.config.upper()} {h.width}x{h.height} {stereo} "
                                       f"full-frame decode")
    metric = (METRIC if (args.config, mode) == ("c3", "viewport")
              else f"decoded frames/s (Mpixel/s) for {workload}")
    sample = (f"{n_timed} display frames (steps {args.warmup}..{args.warmup + n_timed - 1} of the "
              f"schedule; bounded sample of the {args.steps} requested) over {procs} worker "
              f"processes, each with its own reference DecodeSession (wavevid "
              f"{getattr(rw, '__version__', '?')} from baseline/_ref, decode_{mode} + "
              f"render_perspective per eye), after one warm-up frame per worker; per-frame s "
              f"median {statistics.median(r[0] for r in res):.2f}")
    line = {
        "impl": "reference", "metric": metric, "value": round(fps, 4), "unit": "frames/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(wall * 1000.0 / n_timed, 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (the same committed clip as the GPU arm)",
        "config": {"workload": workload + " (reference CPU decoder)",
                   "frames": h.frame_count, "sets": h.num_sets},
        "cpu_baseline": {"value": round(fps, 4), "unit": "frames/s", "cores": procs,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": round(fps, 4), "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "repo_native_loaded": ours_loaded,
        "coverage_errors": sum(r[2] for r in res),
    }
    print(json.dumps(line), flush=True)


def _ref_stereo_mask(rw):
    from wavevid.projection import stereo_mask
    return stereo_mask


def main():
    args = parse()
    if args.mode is None:
        args.mode = "full" if args.config == "c2" else "viewport"
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

"""Multi-GPU layout on CPU (gloo, world size 2): set sharding is a
partition with no data-path collective, and the display gather delivers
every rank's rendered views to rank 0 (sharding.py; bench.py N>1)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2208_10859_b200.sharding import frames_for_sets, gather_views, sets_for_rank


def test_sets_partition_all_frames():
    for num_sets in (1, 2, 3, 8, 13):
        for world in (1, 2, 4, 8):
            owned = [sets_for_rank(num_sets, r, world) for r in range(world)]
            flat = sorted(s for o in owned for s in o)
            if num_sets >= world:
                assert flat == list(range(num_sets))       # a partition
            assert all(o for o in owned)                   # nobody idle
    assert frames_for_sets([0, 2], 4, 10) == [0, 1, 2, 3, 8, 9]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sets = sets_for_rank(4, rank, world)
        frames = frames_for_sets(sets, 4, 16)
        # stand-in for the two rendered eye images of this rank's frame
        views = torch.full((2, 6, 5, 3), rank + 1, dtype=torch.uint8)
        views[0, 0, 0, 0] = frames[0]
        got = gather_views(views, rank, world)
        if rank == 0:
            q.put([(int(t[1, 2, 3, 1]), int(t[0, 0, 0, 0])) for t in got])
        else:
            assert got is None
    finally:
        dist.destroy_process_group()


def test_gather_to_display_rank_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = q.get(timeout=10)
    # rank r contributes value r+1; its first frame is set r's first frame
    assert res == [(1, 0), (2, 4)]


def test_assign_splits():
    """bench.py's N>1 work assignment (sharding.assign): sets round-robin,
    or rank pairs splitting the stereo eyes with sets round-robin over the
    pairs; every (frame, eye) is produced exactly once per cycle."""
    from paper_2208_10859_b200.sharding import assign
    for world in (2, 4, 8):
        for split in ("sets", "eyes"):
            work = set()
            for r in range(world):
                a = assign(8, 4, 32, r, world, split, stereo=True)
                eyes = (0, 1) if a.eye is None else (a.eye,)
                for f in a.frames:
                    for e in eyes:
                        assert (f, e) not in work
                        work.add((f, e))
                assert a.frames_per_step == (1.0 if split == "sets" else 0.5)
            assert work == {(f, e) for f in range(32) for e in (0, 1)}
    assert assign(4, 4, 16, 1, 2, "eyes", stereo=False).eye is None   # mono: sets
    with pytest.raises(ValueError):
        assign(4, 4, 16, 0, 3, "eyes")


def _bench_worker(rank, world, port, q, split):
    """The N>1 step of bench.py on CPU stand-ins: the rank's share from
    sharding.assign, then the per-step gathers to rank 0 -- the decoded
    canvas (full-frame mode, 8192x8192x3 u8) and the eye images."""
    from paper_2208_10859_b200.sharding import assign
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = assign(4, 4, 16, rank, world, split, stereo=True)
        canvas = torch.full((3, 8192, 8192), rank + 1, dtype=torch.uint8)
        canvas[0, 0, :len(a.frames)] = torch.tensor(a.frames, dtype=torch.uint8)
        views = torch.full((2 if a.eye is None else 1, 200, 200, 3), 10 + rank, dtype=torch.uint8)
        bufs = [torch.empty_like(canvas) for _ in range(world)] if rank == 0 else None
        got_c = gather_views(canvas, rank, world, 0, bufs)
        got_v = gather_views(views, rank, world)
        if rank == 0:
            q.put(([(int(t[2, 8191, 8191]), t[0, 0, :4].tolist()) for t in got_c],
                   [(tuple(t.shape), int(t[-1, -1, -1, -1])) for t in got_v]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("split", ["sets", "eyes"])
def test_bench_multi_rank_path_gloo(split):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, q, split))
             for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    canv, views = res
    if split == "sets":
        assert canv == [(1, [0, 1, 2, 3]), (2, [4, 5, 6, 7])]
        assert views == [((2, 200, 200, 3), 10), ((2, 200, 200, 3), 11)]
    else:   # both ranks decode the same frames, one eye each
        assert canv == [(1, [0, 1, 2, 3]), (2, [0, 1, 2, 3])]
        assert views == [((1, 200, 200, 3), 10), ((1, 200, 200, 3), 11)]

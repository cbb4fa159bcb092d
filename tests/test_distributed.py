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

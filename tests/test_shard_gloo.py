"""Multi-process (gloo, world size 2, CPU) coverage of the sharding and the
cluster gather used by bench.py on multi-GPU boxes."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_2112_10603_b200.shard import frames_of_rank, gather_to_root, units_of_rank


def test_frame_and_unit_partitions_cover_everything_once():
    for world in (1, 2, 4, 8):
        frames = sorted(f for r in range(world) for f in frames_of_rank(10, r, world))
        assert frames == list(range(10))
        units = sorted(u for r in range(world) for u in units_of_rank(3, 7, r, world))
        assert units == [(t, g) for t in range(3) for g in range(7)]
        sizes = [len(units_of_rank(3, 7, r, world)) for r in range(world)]
        assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = torch.full((5, 7), rank + 1, dtype=torch.uint8)
        got = gather_to_root(t, rank, world)
        if rank == 0:
            q.put([int(x[0, 0]) for x in got])
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gather_to_root_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert q.get(timeout=10) == list(range(1, world + 1))

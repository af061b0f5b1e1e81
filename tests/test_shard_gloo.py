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


# ---------------------------------------------------------------------------
# gap-sharded rig frame (SURVEY.md sec. 8(e) option 2): plan, halo, gather
# ---------------------------------------------------------------------------
def test_gap_plan_covers_the_rig():
    from paper_2112_10603_b200.shard import gap_plan
    for ncams, stages, vps in [(8, 4, 16), (4, 4, 16), (5, 2, 3), (3, 1, 1), (16, 5, 32)]:
        step = 1 << stages
        for world in (1, 2, 3, 4, 7, 8, 16):
            plans = [gap_plan(ncams, stages, vps, r, world) for r in range(world)]
            gaps = [g for p in plans for g in p.gaps]
            assert gaps == list(range(ncams - 1))
            clusters = [c for p in plans for c in p.clusters]
            assert clusters == list(range(ncams))
            for p in plans:
                if not p.active:
                    assert not len(p.clusters) and p.halo_in is None and p.halo_out is None
                    continue
                local = range(p.view_base, p.view_base + p.n_views)
                halo = range(p.halo_in[1], p.halo_in[1] + p.halo_in[2]) if p.halo_in else range(0)
                for c in p.clusters:  # every tile of every owned cluster is local or halo
                    total = (ncams - 1) * step + 1
                    lo, hi = max(0, c * step - vps), min(total - 1, c * step + vps)
                    assert c * step in local
                    for v in range(lo, hi + 1):
                        assert v in local or v in halo, (world, p.rank, c, v)
                if p.halo_out:  # what a rank sends is local to it and is its neighbour's halo_in
                    dst = plans[p.halo_out[0]]
                    assert dst.halo_in == (p.rank, p.halo_out[1], p.halo_out[2])
                    assert all(v in local for v in range(p.halo_out[1], p.halo_out[1] + p.halo_out[2]))


def _gap_worker(rank, world, port, q, ncams, stages, vps):
    import numpy as np
    import torch.distributed as dist
    from oracle import oracle as O
    from bench import synth_rig
    from paper_2112_10603_b200.shard import exchange_halo, gap_plan, gather_var_to_root
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        O.set_threads(1)
        W, H, fmt = 64, 48, 1
        cams = synth_rig(W, H, fmt, ncams, seed=11)
        p = gap_plan(ncams, stages, vps, rank, world)
        qb = O.frame_bytes(W // 4, H // 4, fmt)
        sizes = []
        for r in range(world):
            pr = gap_plan(ncams, stages, vps, r, world)
            sizes.append(sum(int(O.frame_bytes(W + ((min((ncams - 1) * (1 << stages), c * (1 << stages) + vps)
                                                   - max(0, c * (1 << stages) - vps) + 3) // 4) * (W // 4),
                                                   H, fmt)) for c in pr.clusters))
        send = torch.zeros((p.halo_out[2] if p.halo_out else 1, qb), dtype=torch.uint8)
        recv = torch.zeros((p.halo_in[2] if p.halo_in else 1, qb), dtype=torch.uint8)
        local = None
        if p.active:
            local = O.rig_dense_views(cams[p.cams.start:p.cams.stop], W, H, fmt, stages)
            assert local.shape[0] == p.n_views
            if p.halo_out:
                lo = p.halo_out[1] - p.view_base
                for i in range(p.halo_out[2]):
                    send[i] = torch.from_numpy(O.downscale(local[lo + i], W, H, fmt, 4))
        exchange_halo(p, send, recv)
        parts = []
        step = 1 << stages
        total = (ncams - 1) * step + 1
        for c in p.clusters:
            a = c * step
            lo, hi = max(0, a - vps), min(total - 1, a + vps)
            smalls = []
            for v in range(lo, hi + 1):
                if v == a:
                    continue
                if p.halo_in and p.halo_in[1] <= v < p.halo_in[1] + p.halo_in[2]:
                    smalls.append(recv[v - p.halo_in[1]].numpy())
                else:
                    smalls.append(O.downscale(local[v - p.view_base], W, H, fmt, 4))
            st, _ = O.assemble_cluster(local[a - p.view_base], W, H, fmt, np.stack(smalls))
            parts.append(st)
        mine = torch.from_numpy(np.concatenate(parts)) if parts else torch.zeros(1, dtype=torch.uint8)
        assert (mine.numel() if parts else 0) == sizes[rank]
        got = gather_var_to_root(mine, sizes, rank, world)
        if rank == 0:
            views = O.rig_dense_views(cams, W, H, fmt, stages)
            ref = []
            for c in range(ncams):
                a = c * step
                lo, hi = max(0, a - vps), min(total - 1, a + vps)
                smalls = np.stack([O.downscale(views[v], W, H, fmt, 4) for v in range(lo, hi + 1) if v != a])
                ref.append(O.assemble_cluster(views[a], W, H, fmt, smalls)[0])
            q.put(bool(np.array_equal(got.numpy(), np.concatenate(ref))))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,ncams,stages,vps", [(2, 5, 2, 3), (3, 5, 2, 4), (5, 4, 1, 2)])
def test_gap_sharded_rig_gloo(world, ncams, stages, vps):
    """Each rank synthesises its gaps (oracle as the compute), sends its halo
    quarter tiles right, assembles its clusters, gathers them to rank 0: equal
    to the unsharded rig's clusters.  (5, 4, 1, 2): more ranks than gaps."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gap_worker, args=(r, world, port, q, ncams, stages, vps)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True

"""Multi-GPU layout of the dense view-synthesis path.

Units of work are (rig frame, camera gap) pairs; they are independent
(server/pipeline.py:264-268: a gap reads only its two cameras), so ranks
own whole rig frames and never exchange data while synthesising.  The one
exchange step is the gather of every rank's stitched cluster frames to the
encoder-feeding rank (rank 0) -- grouped point-to-point sends/receives
(NCCL over NVLink on the B200 box, gloo in the CPU tests).
"""
from __future__ import annotations


def frames_of_rank(n_frames: int, rank: int, world: int) -> list:
    """Rig frames (ticks) owned by `rank`: round-robin, t = rank, rank+world, ..."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return list(range(rank, n_frames, world))


def units_of_rank(n_frames: int, n_gaps: int, rank: int, world: int) -> list:
    """(frame, gap) units of `rank` when a single frame must be split (e.g. 7 gaps
    on 8 GPUs): units are dealt round-robin over the flattened (frame, gap) grid."""
    units = [(t, g) for t in range(n_frames) for g in range(n_gaps)]
    return units[rank::world]


def gather_to_root(tensor, rank: int, world: int, root: int = 0, out=None):
    """Gather each rank's `tensor` (same shape everywhere) to `root`.

    Returns a list of `world` tensors on the root (its own first) and None
    elsewhere.  One batched group of isend/irecv: NCCL has no gather
    primitive, this is its idiom.
    """
    import torch
    import torch.distributed as dist
    if world == 1:
        return [tensor]
    ops = []
    if rank == root:
        bufs = out if out is not None else [torch.empty_like(tensor) for _ in range(world - 1)]
        srcs = [r for r in range(world) if r != root]
        for src, b in zip(srcs, bufs):
            ops.append(dist.P2POp(dist.irecv, b, src))
    else:
        ops.append(dist.P2POp(dist.isend, tensor, root))
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    if rank == root:
        return [tensor] + list(bufs)
    return None

"""Multi-GPU layout of the dense view-synthesis path.

Units of work are (rig frame, camera gap) pairs; they are independent
(server/pipeline.py:264-268: a gap reads only its two cameras).  Two
partitions:

* frame sharding (throughput, cfg5's batched live stream): ranks own whole
  rig frames and never exchange data while synthesising;
* gap sharding (latency, cfg3/cfg4 "pairs sharded across B200s"): ranks own
  contiguous runs of camera gaps of ONE rig frame.  The one dependency is
  the tiling: cluster c holds views of gaps c-1 and c (cluster.py:58-74),
  so the rank owning gap c receives the top `views_per_side` views of gap
  c-1 from its left neighbour as a halo -- as quarter tiles (1/16 of the
  bytes), since that is all the cluster frame keeps of them.

The exchange steps are point-to-point (NCCL over NVLink on the B200 box,
gloo in the CPU tests): the halo, then the gather of every rank's cluster
frames to the encoder-feeding rank 0.
"""
from __future__ import annotations

from dataclasses import dataclass


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


def gaps_of_rank(n_gaps: int, rank: int, world: int) -> range:
    """Contiguous, balanced run of camera gaps owned by `rank` (ranks past
    n_gaps own none: a rig frame has only ncams-1 gaps)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    active = min(world, n_gaps)
    if rank >= active:
        return range(n_gaps, n_gaps)
    q, r = divmod(n_gaps, active)
    a = rank * q + min(rank, r)
    return range(a, a + q + (1 if rank < r else 0))


@dataclass(frozen=True)
class GapPlan:
    """What one rank of a gap-sharded rig frame holds, computes and exchanges.

    Global view indices follow ViewIndexModel (viewmodel.py:23-71): camera c
    at c * 2**stages, gap g's views between cameras g and g+1.
    """

    ncams: int
    stages: int
    views_per_side: int
    rank: int
    world: int
    gaps: range          # camera gaps synthesised here
    cams: range          # cameras resident here (both ends of every gap)
    view_base: int       # global index of local view slot 0
    n_views: int         # local views: every view of the gaps plus both end cameras
    clusters: range      # cluster frames assembled here
    halo_in: tuple | None   # (src rank, first global view, count) received as quarter tiles
    halo_out: tuple | None  # (dst rank, first global view, count) sent as quarter tiles

    @property
    def active(self) -> bool:
        return len(self.gaps) > 0


def owner_of_gap(n_gaps: int, gap: int, world: int) -> int:
    for r in range(min(world, n_gaps)):
        if gap in gaps_of_rank(n_gaps, r, world):
            return r
    raise ValueError(f"gap {gap} outside 0..{n_gaps - 1}")


def gap_plan(ncams: int, stages: int, views_per_side: int, rank: int, world: int) -> GapPlan:
    """The gap-sharded layout of one rig frame for `rank` (SURVEY.md sec. 8(e) option 2).

    Rank r owns gaps [a, b), cameras a..b, clusters a..b-1 (and the last
    camera's cluster when b is the last camera).  Cluster a (a > 0) spans
    views [a*2^S - vps, a*2^S + vps] (cluster.py:67-73); its lower half is the
    halo from the owner of gap a-1.
    """
    if ncams < 2:
        raise ValueError("need at least 2 cameras")
    if not 1 <= views_per_side <= (1 << stages):
        raise ValueError("views_per_side must be in 1..2**stages")
    n_gaps = ncams - 1
    g = gaps_of_rank(n_gaps, rank, world)
    if not len(g):
        return GapPlan(ncams, stages, views_per_side, rank, world, g, range(0), 0, 0, range(0), None, None)
    a, b = g.start, g.stop
    step = 1 << stages
    clusters = range(a, b + 1) if b == ncams - 1 else range(a, b)
    halo_in = None
    if a > 0:
        first = max(0, a * step - views_per_side)
        halo_in = (rank - 1, first, a * step - first)
    halo_out = None
    if b < ncams - 1:
        first = max(0, b * step - views_per_side)
        halo_out = (rank + 1, first, b * step - first)
    return GapPlan(ncams, stages, views_per_side, rank, world, g, range(a, b + 1), a * step,
                   (b - a) * step + 1, clusters, halo_in, halo_out)


def exchange_halo(plan: GapPlan, send_tiles, recv_tiles) -> None:
    """The one data-path exchange of the gap-sharded rig: quarter tiles of
    plan.halo_out to the right neighbour, plan.halo_in from the left one
    (grouped isend/irecv; no-op pieces are skipped)."""
    import torch.distributed as dist
    ops = []
    if plan.halo_in is not None:
        ops.append(dist.P2POp(dist.irecv, recv_tiles, plan.halo_in[0]))
    if plan.halo_out is not None:
        ops.append(dist.P2POp(dist.isend, send_tiles, plan.halo_out[0]))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def gather_var_to_root(tensor, sizes: list, rank: int, world: int, root: int = 0, out=None):
    """Gather 1-D uint8 buffers of per-rank `sizes` (bytes; 0 = nothing) to `root`.

    Returns the concatenation in rank order on the root, None elsewhere."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return tensor
    if rank == root:
        total = sum(sizes)
        if out is None:
            out = torch.empty(total, dtype=torch.uint8, device=tensor.device)
        offs = [sum(sizes[:r]) for r in range(world)]
        if sizes[root]:
            out[offs[root]:offs[root] + sizes[root]].copy_(tensor[:sizes[root]])
        ops = [dist.P2POp(dist.irecv, out[offs[r]:offs[r] + sizes[r]], r)
               for r in range(world) if r != root and sizes[r]]
    else:
        ops = [dist.P2POp(dist.isend, tensor[:sizes[rank]], root)] if sizes[rank] else []
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return out if rank == root else None


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


class GapShardedRig:
    """One rank's share of a gap-sharded rig frame on its B200.

    compute(): the dense views of the rank's gaps (fvv_rig_views over its
    cameras) and the quarter tiles of its outgoing halo (fvv_downscale);
    exchange(): the halo (NCCL P2P); stitch(): its cluster frames from local
    views + received halo tiles (fvv_rig_clusters_shard).  compute() and
    stitch() only enqueue on the current stream, so each can be captured as a
    CUDA graph; exchange() runs between them.
    """

    def __init__(self, width: int, height: int, fmt, ncams: int, stages: int, views_per_side: int,
                 rank: int, world: int, config=None, device=None):
        import torch
        from .frame import frame_nbytes
        from .interp import Interpolator
        from .cluster import rig_cluster_sizes
        self.plan = gap_plan(ncams, stages, views_per_side, rank, world)
        self.width, self.height, self.format = int(width), int(height), int(fmt)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        p = self.plan
        fb = frame_nbytes(width, height, fmt)
        qb = frame_nbytes(width // 4, height // 4, fmt)
        self.frame_bytes = fb
        all_sizes = rig_cluster_sizes(width, height, fmt, ncams, stages, views_per_side)
        self.cluster_sizes = [all_sizes[c] for c in p.clusters]
        self.sizes_by_rank = [sum(all_sizes[c] for c in gap_plan(ncams, stages, views_per_side, r, world).clusters)
                              for r in range(world)]
        self.engine = None
        if p.active:
            self.engine = Interpolator(width, height, fmt, config, max_pairs=len(p.gaps) << (stages - 1),
                                       device=self.device)
        self.cams = torch.empty((max(1, len(p.cams)), fb), dtype=torch.uint8, device=self.device)
        self.views = torch.empty((max(1, p.n_views), fb), dtype=torch.uint8, device=self.device)
        self.halo_send = torch.empty((p.halo_out[2] if p.halo_out else 1, qb), dtype=torch.uint8, device=self.device)
        self.halo_recv = torch.empty((p.halo_in[2] if p.halo_in else 1, qb), dtype=torch.uint8, device=self.device)
        self.clusters = torch.empty(max(1, sum(self.cluster_sizes)), dtype=torch.uint8, device=self.device)

    def compute(self):
        from .cluster import downscale_device
        p = self.plan
        if not p.active:
            return
        self.engine.rig(self.cams, p.stages, self.views)
        if p.halo_out is not None:
            lo = p.halo_out[1] - p.view_base
            downscale_device(self.views[lo:lo + p.halo_out[2]], self.width, self.height, self.format, 4,
                             out=self.halo_send)

    def exchange(self):
        exchange_halo(self.plan, self.halo_send, self.halo_recv)

    def stitch(self):
        from .cluster import rig_clusters_shard
        p = self.plan
        if not len(p.clusters):
            return
        hf, hc = (p.halo_in[1], p.halo_in[2]) if p.halo_in else (0, 0)
        rig_clusters_shard(self.views[:p.n_views], p.view_base, self.width, self.height, self.format, p.ncams,
                           p.stages, p.views_per_side, p.clusters.start, len(p.clusters),
                           halo=self.halo_recv if hc else None, halo_first=hf, halo_count=hc, out=self.clusters)

    def gather(self, out=None):
        """Every rank's cluster frames, in camera order, to rank 0."""
        return gather_var_to_root(self.clusters, self.sizes_by_rank, self.plan.rank, self.plan.world, out=out)

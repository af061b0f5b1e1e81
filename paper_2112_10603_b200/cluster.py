"""Dense-view tiling into multi-view cluster frames on the B200.

Mirror of the reference's tiling API (cluster.py:19-191): `build_layouts`,
`cluster_geometry`, `downscale`, `assemble_cluster_frame`, `crop_frame` and
the layout types, with identical geometry and errors (LayoutError /
ValueError).  Pixel work runs in csrc/tile_kernels.cu; `rig_clusters`
produces every cluster of a rig frame straight from the device views buffer
(server/pipeline.py:273-292 `_stitch`, downscale fused into the paste).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .frame import Frame, PixelFormat, frame_from_packed, frame_from_planes, frame_nbytes, packed
from .viewmodel import ViewIndexModel

TIER_FULL = "full"
TIER_QUARTER = "quarter"
SCALE_FACTOR = 4


class LayoutError(_lib.LayoutErrorBase):
    pass


@dataclass(frozen=True)
class TileRef:
    index: int
    tier: str


@dataclass(frozen=True)
class ClusterLayout:
    cluster_id: int
    anchor_index: int
    first_index: int
    last_index: int
    views_per_side: int
    tiles: tuple

    @property
    def tile_count(self) -> int:
        return len(self.tiles)

    def contains(self, view: int) -> bool:
        return self.first_index <= view <= self.last_index

    def clamp(self, view: int) -> int:
        return min(max(view, self.first_index), self.last_index)

    def tile_of(self, view: int) -> int:
        if not self.contains(view):
            raise LayoutError(f"view {view} outside cluster {self.cluster_id} "
                              f"range {self.first_index}..{self.last_index}")
        return view - self.first_index


def build_layouts(model: ViewIndexModel, views_per_side: int = 16) -> list:
    """cluster.py:58-74: one cluster per camera, 2*vps+1 consecutive views."""
    if views_per_side < 1:
        raise LayoutError("views_per_side must be >= 1")
    if views_per_side > (1 << model.stages):
        raise LayoutError(f"views_per_side {views_per_side} exceeds the {(1 << model.stages) - 1} "
                          f"interpolated views available per gap")
    layouts = []
    for cam in range(model.camera_count):
        anchor = model.view_index(cam)
        lo = max(0, anchor - views_per_side)
        hi = min(model.total_views - 1, anchor + views_per_side)
        tiles = tuple(TileRef(i, TIER_FULL if i == anchor else TIER_QUARTER) for i in range(lo, hi + 1))
        layouts.append(ClusterLayout(cam, anchor, lo, hi, views_per_side, tiles))
    return layouts


@dataclass(frozen=True)
class TileRect:
    index: int
    tier: str
    x: int
    y: int
    width: int
    height: int


@dataclass(frozen=True)
class ClusterFrame:
    cluster_id: int
    frame: Frame
    tile_map: tuple

    def crop(self, rect: TileRect) -> Frame:
        return crop_frame(self.frame, rect.x, rect.y, rect.width, rect.height)


def crop_frame(frame, x: int, y: int, w: int, h: int) -> Frame:
    """cluster.py:105-132 (host slicing of a downloaded cluster frame)."""
    if int(frame.format) == PixelFormat.YUV420 and (x % 2 or y % 2 or w % 2 or h % 2):
        raise ValueError("4:2:0 crops must be even-aligned")
    planes = [np.ascontiguousarray(frame.planes[0][y:y + h, x:x + w])]
    if int(frame.format) == PixelFormat.YUV420:
        planes.append(np.ascontiguousarray(frame.planes[1][y // 2:(y + h) // 2, x // 2:(x + w) // 2]))
        planes.append(np.ascontiguousarray(frame.planes[2][y // 2:(y + h) // 2, x // 2:(x + w) // 2]))
    return frame_from_planes(planes, frame.format, frame.timestamp)


def cluster_geometry(base_width: int, base_height: int, small_count: int) -> tuple:
    """cluster.py:135-140: (stitched width, stitched height, grid columns)."""
    cols = (small_count + SCALE_FACTOR - 1) // SCALE_FACTOR
    return base_width + cols * (base_width // SCALE_FACTOR), base_height, cols


def tile_rects(layout: ClusterLayout, width: int, height: int) -> tuple:
    """Tile map of a stitched cluster (cluster.py:171-190; server/pipeline.py:374-393)."""
    cell_w, cell_h = width // SCALE_FACTOR, height // SCALE_FACTOR
    rects, small_i = [], 0
    for ref in layout.tiles:
        if ref.tier == TIER_FULL:
            rects.append(TileRect(ref.index, TIER_FULL, 0, 0, width, height))
        else:
            col, row = divmod(small_i, SCALE_FACTOR)
            rects.append(TileRect(ref.index, TIER_QUARTER, width + col * cell_w, row * cell_h,
                                  cell_w, cell_h))
            small_i += 1
    return tuple(rects)


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def downscale_device(frames, width: int, height: int, fmt, factor: int, out=None):
    """Batched cluster.py:77-89 on packed device frames (n, frame_bytes)."""
    import torch
    L = _lib.require_cuda()
    frames = frames.reshape(-1, frame_nbytes(width, height, fmt))
    n = frames.shape[0]
    qb = frame_nbytes(width // factor, height // factor, fmt) if width % factor == 0 and height % factor == 0 else 0
    if out is None:
        out = torch.empty((n, max(qb, 1)), dtype=torch.uint8, device=frames.device)
    d = _lib.desc(width, height, int(fmt))
    _lib.check(L.fvv_downscale(ctypes.byref(d), ctypes.c_void_p(frames.data_ptr()), n, factor,
                               ctypes.c_void_p(out.data_ptr()), _stream()))
    return out


def downscale(frame, factor: int) -> Frame:
    """cluster.py:77-89: box-filter reduction by an integer factor per dimension."""
    import torch
    if frame.width % factor or frame.height % factor:
        raise ValueError(f"{frame.width}x{frame.height} not divisible by {factor}")
    _lib.require_cuda()
    dev = torch.from_numpy(packed(frame)).cuda()
    out = downscale_device(dev, frame.width, frame.height, frame.format, factor)
    return frame_from_packed(out[0].cpu().numpy(), frame.width // factor, frame.height // factor,
                             frame.format, frame.timestamp)


def assemble_cluster_frame(anchor_frame, interp_frames: list, layout: ClusterLayout) -> ClusterFrame:
    """cluster.py:143-191: anchor at full resolution on the left, 1/4-scale tiles
    in a column-major grid of 4 rows to its right; absent cells stay black."""
    import torch
    small_refs = [t for t in layout.tiles if t.tier == TIER_QUARTER]
    if len(interp_frames) != len(small_refs):
        raise LayoutError(f"layout wants {len(small_refs)} interpolated views, got {len(interp_frames)}")
    w, h = anchor_frame.width, anchor_frame.height
    if w % (2 * SCALE_FACTOR) or h % (2 * SCALE_FACTOR):
        raise LayoutError("anchor dimensions must be divisible by 8")
    fmt = int(anchor_frame.format)
    if fmt == PixelFormat.RGB8:
        raise LayoutError("cluster frames are gray or 4:2:0")
    cell_w, cell_h = w // SCALE_FACTOR, h // SCALE_FACTOR
    for ref, small in zip(small_refs, interp_frames):
        if (small.width, small.height) != (cell_w, cell_h):
            raise LayoutError(f"tile {ref.index} is {small.width}x{small.height}, cell is {cell_w}x{cell_h}")
    L = _lib.require_cuda()
    from .interp import _pinned, _to_host
    sw, sh, _ = cluster_geometry(w, h, len(small_refs))
    # anchor and every tile in one pinned staging buffer, one H2D copy
    fa, fs = frame_nbytes(w, h, fmt), frame_nbytes(cell_w, cell_h, fmt)
    host = _pinned("cluster_in", fa + fs * len(interp_frames))
    hn = host.numpy()
    hn[:fa] = packed(anchor_frame)
    for i, f in enumerate(interp_frames):
        hn[fa + i * fs:fa + (i + 1) * fs] = packed(f)
    dev = host.to("cuda", non_blocking=True)
    base = dev.data_ptr()
    out = torch.empty(frame_nbytes(sw, sh, fmt), dtype=torch.uint8, device="cuda")
    d = _lib.desc(w, h, fmt)
    _lib.check(L.fvv_assemble_cluster(ctypes.byref(d), ctypes.c_void_p(base),
                                      _lib.ptr_array([base + fa + i * fs for i in range(len(interp_frames))]),
                                      len(interp_frames), ctypes.c_void_p(out.data_ptr()), _stream()))
    stitched = frame_from_packed(_to_host(out, "cluster_out"), sw, sh, fmt, anchor_frame.timestamp)
    return ClusterFrame(layout.cluster_id, stitched, tile_rects(layout, w, h))


def rig_cluster_sizes(width: int, height: int, fmt, camera_count: int, stages: int,
                      views_per_side: int) -> list:
    L = _lib.load()
    d = _lib.desc(width, height, int(fmt))
    return [int(L.fvv_rig_cluster_bytes(ctypes.byref(d), camera_count, stages, views_per_side, c))
            for c in range(camera_count)]


def rig_clusters(views, width: int, height: int, fmt, camera_count: int, stages: int,
                 views_per_side: int = 16, out=None):
    """server/pipeline.py:273-292 on device: global views (T, fb) -> all cluster
    frames packed back to back (camera order).  Returns (out, sizes)."""
    import torch
    L = _lib.require_cuda()
    sizes = rig_cluster_sizes(width, height, fmt, camera_count, stages, views_per_side)
    if out is None:
        out = torch.empty(sum(sizes), dtype=torch.uint8, device=views.device)
    d = _lib.desc(width, height, int(fmt))
    _lib.check(L.fvv_rig_clusters(ctypes.byref(d), camera_count, stages, views_per_side,
                                  ctypes.c_void_p(views.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                  _stream()))
    return out, sizes


def rig_clusters_shard(views, view_base: int, width: int, height: int, fmt, camera_count: int,
                       stages: int, views_per_side: int, first_cluster: int, ncluster: int,
                       halo=None, halo_first: int = 0, halo_count: int = 0, out=None):
    """Clusters [first_cluster, first_cluster + ncluster) of a rig frame from a
    rank's local views (global indices view_base..) plus halo quarter tiles
    (fvv_rig_clusters_shard; the gap-sharded rig of shard.GapShardedRig).
    Returns (out, sizes)."""
    import torch
    L = _lib.require_cuda()
    sizes = rig_cluster_sizes(width, height, fmt, camera_count, stages,
                              views_per_side)[first_cluster:first_cluster + ncluster]
    if out is None:
        out = torch.empty(max(1, sum(sizes)), dtype=torch.uint8, device=views.device)
    d = _lib.desc(width, height, int(fmt))
    _lib.check(L.fvv_rig_clusters_shard(
        ctypes.byref(d), camera_count, stages, views_per_side, first_cluster, ncluster,
        ctypes.c_void_p(views.data_ptr()), view_base, views.shape[0],
        ctypes.c_void_p(halo.data_ptr() if halo is not None else 0), halo_first, halo_count,
        ctypes.c_void_p(out.data_ptr()), _stream()))
    return out, sizes

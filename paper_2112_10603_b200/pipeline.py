"""Device-resident rig stages: the reference's `PipelineHandle._interp` and
`_stitch` (server/pipeline.py:254-292) without byte bundling.

The reference moves every rig frame through its stage threads as serialized
bytes (server/pipeline.py:145-163) -- at 1080p the host (de)serialisation
costs as much as the synthesis itself.  Here a
rig frame stays in HBM from camera upload to cluster frames: one C-ABI call
per stage (`fvv_rig_views`, `fvv_rig_clusters`), captured once as a CUDA
graph and replayed per tick; host I/O goes through pinned staging buffers on
the pipeline's own stream.
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .cluster import ClusterFrame, build_layouts, rig_cluster_sizes, rig_clusters, tile_rects
from .frame import PixelFormat, frame_from_packed, frame_nbytes, packed
from .interp import InterpConfig, Interpolator
from .viewmodel import ViewIndexModel


class RigPipeline:
    """Camera frames of one tick -> every dense view and every cluster frame.

    `process()` works on device tensors; `process_frames()` is the host-facing
    form (reference Frames in, `ClusterFrame`s out).  Reentrant per instance;
    use one instance per stream.
    """

    def __init__(self, width: int, height: int, fmt, camera_count: int, stages: int = 4,
                 views_per_side: int = 16, config: InterpConfig | None = None, graph: bool = True,
                 device=None):
        import torch
        _lib.require_cuda()
        self.model = ViewIndexModel(camera_count, stages)
        self.width, self.height, self.format = int(width), int(height), PixelFormat(int(fmt))
        self.views_per_side = int(views_per_side)
        self.layouts = build_layouts(self.model, self.views_per_side) if self.views_per_side else []
        self.engine = Interpolator(width, height, fmt, config,
                                   max_pairs=(camera_count - 1) << (stages - 1), device=device)
        dev = self.engine.device
        fb = self.engine.frame_bytes
        self.cams = torch.empty((camera_count, fb), dtype=torch.uint8, device=dev)
        self.views = torch.empty((self.model.total_views, fb), dtype=torch.uint8, device=dev)
        tiled = self.views_per_side > 0 and int(fmt) != PixelFormat.RGB8
        self.sizes = rig_cluster_sizes(width, height, fmt, camera_count, stages,
                                       self.views_per_side) if tiled else []
        self.clusters = torch.empty(max(1, sum(self.sizes)), dtype=torch.uint8, device=dev)
        self.stream = torch.cuda.Stream(device=dev)
        self._host_in = torch.empty((camera_count, fb), dtype=torch.uint8).pin_memory()
        self._host_out = torch.empty(self.clusters.numel(), dtype=torch.uint8).pin_memory()
        self._tiled = tiled
        self._graph = None
        if graph:
            with torch.cuda.stream(self.stream):
                self._compute()  # warm: lazy attributes, allocator
            self.stream.synchronize()
            self._graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self._graph, stream=self.stream):
                self._compute()
            self.stream.synchronize()

    def _compute(self):
        self.engine.rig(self.cams, self.model.stages, self.views)
        if self._tiled:
            rig_clusters(self.views, self.width, self.height, self.format, self.model.camera_count,
                         self.model.stages, self.views_per_side, out=self.clusters)

    def process(self, cams=None):
        """Run one tick on the pipeline stream.  `cams` (C, frame_bytes) device or
        host tensor; None means `self.cams` was filled by the caller.  Returns
        (views, clusters) device tensors (valid once the stream reaches them)."""
        import torch
        with torch.cuda.stream(self.stream):
            if cams is not None:
                self.cams.copy_(cams, non_blocking=True)
            if self._graph is not None:
                self._graph.replay()
            else:
                self._compute()
        return self.views, self.clusters

    def process_frames(self, frames) -> list:
        """Reference-facing form: C camera Frames -> C `ClusterFrame`s (host)."""
        import torch
        if len(frames) != self.model.camera_count:
            raise ValueError(f"rig has {self.model.camera_count} cameras, got {len(frames)} frames")
        for i, f in enumerate(frames):
            if (f.width, f.height, int(f.format)) != (self.width, self.height, int(self.format)):
                raise ValueError("camera frames must share the pipeline's size and format")
            self._host_in[i].copy_(torch.from_numpy(packed(f)))
        self.process(self._host_in)
        if not self._tiled:
            raise ValueError("pipeline built without tiling (RGB8 or views_per_side = 0)")
        with torch.cuda.stream(self.stream):
            self._host_out.copy_(self.clusters, non_blocking=True)
        self.stream.synchronize()
        host = self._host_out.numpy()
        out, off = [], 0
        for lay, size in zip(self.layouts, self.sizes):
            sw = (size * 2) // (3 * self.height) if int(self.format) == PixelFormat.YUV420 \
                else size // self.height
            fr = frame_from_packed(host[off:off + size].copy(), sw, self.height, self.format,
                                   frames[0].timestamp)
            out.append(ClusterFrame(lay.cluster_id, fr, tile_rects(lay, self.width, self.height)))
            off += size
        return out

    def stream_ticks(self, host_cams, host_out, slots: int = 2):
        """Throughput form for a live stream: process len(host_cams) ticks with
        the host->device copy of tick t+1 and the device->host copy of tick t-1
        overlapping the synthesis of tick t.

        host_cams: list of pinned uint8 tensors (C, frame_bytes); host_out: list
        of pinned uint8 tensors (cluster bytes), same length.  Uses `slots`
        device buffer sets, each with its own CUDA graph and compute stream, so
        the synthesis of consecutive ticks overlaps as well (one tick's small
        stage-1 launches run beside another's large ones).  Returns when all
        copies are enqueued; synchronise on `self.stream` (or the device) before
        reading.
        """
        import torch
        if not self._tiled:
            raise ValueError("stream_ticks needs a tiling pipeline")
        if not hasattr(self, "_slots") or len(self._slots) != slots:
            self._make_slots(slots)
        h2d = torch.cuda.Stream(device=self.engine.device)
        d2h = torch.cuda.Stream(device=self.engine.device)
        done_in = [torch.cuda.Event() for _ in range(slots)]
        done_cmp = [torch.cuda.Event() for _ in range(slots)]
        done_out = [torch.cuda.Event() for _ in range(slots)]
        for t, (hin, hout) in enumerate(zip(host_cams, host_out)):
            k = t % slots
            cams, clusters, graph = self._slots[k][:3]
            if t >= slots:
                h2d.wait_event(done_cmp[k])          # the slot's previous tick has been consumed
            with torch.cuda.stream(h2d):
                cams.copy_(hin, non_blocking=True)
                done_in[k].record(h2d)
            cs = self._cstreams[k]
            cs.wait_event(done_in[k])
            if t >= slots:
                cs.wait_event(done_out[k])  # its clusters have left the device
            with torch.cuda.stream(cs):
                graph.replay()
                done_cmp[k].record(cs)
            d2h.wait_event(done_cmp[k])
            with torch.cuda.stream(d2h):
                hout.copy_(clusters, non_blocking=True)
                done_out[k].record(d2h)
        self.stream.wait_stream(d2h)

    def _make_slots(self, slots: int):
        import torch
        self._slots = []
        self._cstreams = [self.stream] + [torch.cuda.Stream(device=self.engine.device) for _ in range(slots - 1)]
        for k in range(slots):
            if k == 0:
                eng, cams, views, clusters = self.engine, self.cams, self.views, self.clusters
            else:
                eng = Interpolator(self.width, self.height, self.format, self.engine.config,
                                   max_pairs=self.engine.max_pairs, device=self.engine.device)
                cams = torch.empty_like(self.cams)
                views = torch.empty_like(self.views)
                clusters = torch.empty_like(self.clusters)

            def run(eng=eng, cams=cams, views=views, clusters=clusters):
                eng.rig(cams, self.model.stages, views)
                rig_clusters(views, self.width, self.height, self.format, self.model.camera_count,
                             self.model.stages, self.views_per_side, out=clusters)
            with torch.cuda.stream(self.stream):
                run()
            self.stream.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=self.stream):
                run()
            self.stream.synchronize()
            # the graph replays into this slot's engine workspace and views: keep
            # them alive with it (a collected engine's memory would be reused)
            self._slots.append((cams, clusters, graph, eng, views))

    def views_host(self) -> np.ndarray:
        self.stream.synchronize()
        return self.views.cpu().numpy()

    @property
    def views_per_tick(self) -> int:
        return (self.model.camera_count - 1) * self.model.views_per_gap

    @property
    def frame_bytes(self) -> int:
        return frame_nbytes(self.width, self.height, self.format)


class DeviceRigStages:
    """Device-resident state behind the reference pipeline's `_interp` and
    `_stitch` stage workers (server/pipeline.py:254-292), installed by
    `plugin.install(fvv, pipeline=True)`.

    `interp(cams)` uploads one tick's camera Frames and synthesises every dense
    view into a device slot (fvv_rig_views), returning the slot number -- the
    only thing the views channel then carries (no byte bundling of 45-105
    frames).  `stitch(slot)` builds every cluster frame of that slot on the
    device (fvv_rig_clusters) and downloads them for the host encoder stage.
    The two run on their own threads and CUDA streams; events order a slot's
    views before its stitch and its stitch before the slot's reuse.  `slots`
    must exceed the views channel's capacity + 1 (the pipeline's back-pressure
    then guarantees a slot is stitched before it is rewritten).
    """

    def __init__(self, width: int, height: int, fmt, camera_count: int, stages: int, views_per_side: int,
                 config: InterpConfig | None = None, slots: int = 6, device=None):
        import torch
        _lib.require_cuda()
        self.model = ViewIndexModel(camera_count, stages)
        self.width, self.height, self.format = int(width), int(height), PixelFormat(int(fmt))
        self.views_per_side = int(views_per_side)
        self.layouts = build_layouts(self.model, self.views_per_side)
        self.engine = Interpolator(width, height, fmt, config, max_pairs=(camera_count - 1) << (stages - 1),
                                   device=device)
        dev = self.engine.device
        fb = self.engine.frame_bytes
        self.slots = int(slots)
        self.cams = [torch.empty((camera_count, fb), dtype=torch.uint8, device=dev) for _ in range(self.slots)]
        self.views = [torch.empty((self.model.total_views, fb), dtype=torch.uint8, device=dev)
                      for _ in range(self.slots)]
        self.tiled = int(fmt) != PixelFormat.RGB8
        self.sizes = rig_cluster_sizes(width, height, fmt, camera_count, stages, self.views_per_side) \
            if self.tiled else []
        # one cluster buffer per slot: with the encoder hand-off the clusters stay on
        # the device until the encode stage has read them
        self.clusters = [torch.empty(max(1, sum(self.sizes)), dtype=torch.uint8, device=dev)
                         for _ in range(self.slots)]
        self._host_in = torch.empty((camera_count, fb), dtype=torch.uint8).pin_memory()
        self._host_out = torch.empty(self.clusters[0].numel(), dtype=torch.uint8).pin_memory()
        self.s_interp = torch.cuda.Stream(device=dev)
        self.s_stitch = torch.cuda.Stream(device=dev)
        self.s_encode = torch.cuda.Stream(device=dev)
        self._ev_views = [torch.cuda.Event() for _ in range(self.slots)]
        self._ev_clusters = [torch.cuda.Event() for _ in range(self.slots)]
        self._ev_free = [None] * self.slots
        self._encoder = None
        self._stamps = [None] * self.slots
        self._next = 0

    def interp(self, frames) -> int:
        """One tick's camera Frames -> every global view in a device slot."""
        import torch
        if len(frames) != self.model.camera_count:
            raise ValueError(f"rig has {self.model.camera_count} cameras, got {len(frames)} frames")
        for i, f in enumerate(frames):
            if (f.width, f.height, int(f.format)) != (self.width, self.height, int(self.format)):
                raise ValueError("interpolation inputs must share size and format")
            self._host_in[i].copy_(torch.from_numpy(packed(f)))
        k = self._next
        self._next = (k + 1) % self.slots
        with torch.cuda.stream(self.s_interp):
            if self._ev_free[k] is not None:
                self.s_interp.wait_event(self._ev_free[k])  # the slot's previous tick is stitched
            self.cams[k].copy_(self._host_in, non_blocking=True)
            self.engine.rig(self.cams[k], self.model.stages, self.views[k])
            self._ev_views[k].record(self.s_interp)
        self._stamps[k] = [f.timestamp for f in frames]
        self.s_interp.synchronize()  # the stage's latency is real; the pinned input is free again
        return k

    def stitch_device(self, slot: int) -> None:
        """Every cluster frame of the tick in `slot`, left on the device (clusters[slot])."""
        import torch
        from .cluster import LayoutError
        if not self.tiled:
            raise LayoutError("cluster frames are gray or 4:2:0")
        with torch.cuda.stream(self.s_stitch):
            self.s_stitch.wait_event(self._ev_views[slot])
            rig_clusters(self.views[slot], self.width, self.height, self.format, self.model.camera_count,
                         self.model.stages, self.views_per_side, out=self.clusters[slot])
            ev = torch.cuda.Event()
            ev.record(self.s_stitch)
            self._ev_free[slot] = ev
            self._ev_clusters[slot].record(self.s_stitch)
        self.s_stitch.synchronize()  # the stage's latency is real

    def encode(self, slot: int, quality: int, gop: int, encoder_factory=None) -> list:
        """FVT1 records of every tile of every cluster frame of `slot`
        (PipelineHandle._encode, server/pipeline.py:294-318): per cluster, the
        record bytes of its tiles in tile-map order.  The transform stage runs on
        the device (encoder.RigEncoder); one encoder per pipeline keeps every
        tile's closed-loop reconstruction."""
        import torch
        if self._encoder is None:
            if encoder_factory is None:
                from .encoder import RigEncoder as encoder_factory  # noqa: N813
            self._encoder = encoder_factory(self.layouts, self.width, self.height, self.format, quality, gop,
                                            self.engine.device)
        with torch.cuda.stream(self.s_encode):
            self.s_encode.wait_event(self._ev_clusters[slot])
            return self._encoder.encode(self.clusters[slot])

    def stitch(self, slot: int) -> list:
        """Every cluster frame of the tick in `slot` (host ClusterFrames)."""
        import torch
        self.stitch_device(slot)
        with torch.cuda.stream(self.s_stitch):
            self._host_out.copy_(self.clusters[slot], non_blocking=True)
        self.s_stitch.synchronize()
        host = self._host_out.numpy()
        stamps = self._stamps[slot]
        out, off = [], 0
        for lay, size in zip(self.layouts, self.sizes):
            sw = (size * 2) // (3 * self.height) if int(self.format) == PixelFormat.YUV420 \
                else size // self.height
            fr = frame_from_packed(host[off:off + size].copy(), sw, self.height, self.format,
                                   stamps[lay.anchor_index >> self.model.stages])
            out.append(ClusterFrame(lay.cluster_id, fr, tile_rects(lay, self.width, self.height)))
            off += size
        return out

    def views_host(self, slot: int) -> np.ndarray:
        self.s_interp.synchronize()
        return self.views[slot].cpu().numpy()

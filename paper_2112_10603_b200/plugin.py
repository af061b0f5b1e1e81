"""Drop-in installation into the reference package (`fvv`).

The reference's seams for this path are plain Python names (SURVEY.md
sec. 8(b)): `fvv.interp.interpolate` / `dense_views`, `fvv.cluster.downscale`
/ `assemble_cluster_frame`, and the copies of those names bound at import
time in `fvv.server.pipeline` (server/pipeline.py:17-21) and `fvv.report`
(report.py:69-105).  `install(fvv)` rebinds every one of them to the B200
implementations of this package, so the reference's pipeline, reports and
CLI run the CUDA path unchanged:

    import fvv, paper_2112_10603_b200.plugin as p
    p.install(fvv)           # fvv.interp.interpolate is now the B200 path

Frames flow in and out as the reference's own `fvv.frame.Frame` objects.
`uninstall(fvv)` restores the originals.

`install(fvv, pipeline=True)` additionally replaces the two GPU stage
workers of the reference's live pipeline, `PipelineHandle._interp` and
`PipelineHandle._stitch` (server/pipeline.py:254-292), with device-resident
ones: the views of a tick stay in HBM between
the two stages (pipeline.DeviceRigStages) and the views channel carries a
slot number instead of a byte bundle of every view.  The channels, the
stage-latency report, the trace stamps and the host stages around them
(capture, encode, segment) are the reference's own.
"""
from __future__ import annotations

import importlib
import struct
import threading
import time

from . import cluster as _cluster
from . import interp as _interp
from .frame import packed

_SAVED: dict = {}


def _ref_frame(fvv_frame_mod, ours, template):
    """This package's Frame -> the reference's Frame class (same planes)."""
    return fvv_frame_mod.Frame(ours.width, ours.height, template.format.__class__(int(ours.format)),
                               tuple(ours.planes), ours.timestamp)


def install(fvv, pipeline: bool = False, stages_factory=None, encoder: bool = False, encoder_factory=None,
            segment: bool = False, names: bool = True) -> None:
    """Rebind the reference's path names (and, with `pipeline`, its stage
    workers).  `stages_factory(width, height, fmt, cams, stages, vps, config,
    slots)` builds the device stage state; default pipeline.DeviceRigStages.
    With `encoder` the encode stage's transform runs on the device too: the
    cluster frames stay in HBM from _stitch to _encode (encoder.RigEncoder,
    or `encoder_factory(layouts, width, height, fmt, quality, gop, device)`).
    With `segment` the TS stage (_segment) muxes every cluster of a segment
    boundary concurrently with the native muxer (segmenter.py); host code,
    independent of the other hooks.  names=False leaves the path's function
    names alone (e.g. only the TS stage on a host without a GPU)."""
    frame_mod = importlib.import_module(fvv.__name__ + ".frame")
    interp_mod = importlib.import_module(fvv.__name__ + ".interp")
    cluster_mod = importlib.import_module(fvv.__name__ + ".cluster")

    def interpolate(left, right, config=None, diagnostics=False):
        cfg = _interp.InterpConfig(config.block_size, config.search_radius, config.mask_epsilon,
                                   config.border_band, None) if config is not None else None
        res = _interp.interpolate(left, right, cfg, diagnostics=diagnostics or
                                  (config is not None and config.refine is not None))
        out, diag = (res if isinstance(res, tuple) else (res, None))
        out = _ref_frame(frame_mod, out, left)
        if config is not None and config.refine is not None:
            out = config.refine(out, diag)
        return (out, diag) if diagnostics else out

    def dense_views(left, right, stages, config=None):
        if config is not None and config.refine is not None:
            seq = [left, right]
            for _ in range(stages):
                nxt = []
                for a, b in zip(seq, seq[1:]):
                    nxt += [a, interpolate(a, b, config)]
                seq = nxt + [seq[-1]]
            return seq[1:-1]
        cfg = _interp.InterpConfig(config.block_size, config.search_radius, config.mask_epsilon) \
            if config is not None else None
        return [_ref_frame(frame_mod, v, left) for v in _interp.dense_views(left, right, stages, cfg)]

    def downscale(frame, factor):
        return _ref_frame(frame_mod, _cluster.downscale(frame, factor), frame)

    def assemble_cluster_frame(anchor_frame, interp_frames, layout):
        try:
            cf = _cluster.assemble_cluster_frame(anchor_frame, interp_frames, layout)
        except _cluster.LayoutError as e:
            raise cluster_mod.LayoutError(str(e)) from None
        rects = tuple(cluster_mod.TileRect(r.index, r.tier, r.x, r.y, r.width, r.height)
                      for r in cf.tile_map)
        return cluster_mod.ClusterFrame(cf.cluster_id, _ref_frame(frame_mod, cf.frame, anchor_frame),
                                        rects)

    repl = {} if not names else {(interp_mod, "interpolate"): interpolate, (interp_mod, "dense_views"): dense_views,
            (cluster_mod, "downscale"): downscale,
            (cluster_mod, "assemble_cluster_frame"): assemble_cluster_frame}
    for modname, seams in ((".server.pipeline", ("dense_views", "downscale", "assemble_cluster_frame")),
                           (".report", ("dense_views",))):
        if not names:
            break
        try:
            m = importlib.import_module(fvv.__name__ + modname)
        except ImportError:
            continue
        for n in seams:
            if hasattr(m, n):
                src = interp_mod if n in ("interpolate", "dense_views") else cluster_mod
                repl[(m, n)] = repl[(src, n)]
    if pipeline:
        pl = importlib.import_module(fvv.__name__ + ".server.pipeline")
        hooks = _pipeline_hooks(pl, frame_mod, stages_factory, encoder, encoder_factory)
        for n, f in hooks.items():
            repl[(pl.PipelineHandle, n)] = f
    if segment:
        pl = importlib.import_module(fvv.__name__ + ".server.pipeline")
        ts = importlib.import_module(fvv.__name__ + ".mpegts")
        repl[(pl.PipelineHandle, "_segment")] = _segment_hook(pl, ts)
    for (m, n), f in repl.items():
        _SAVED.setdefault((m, n), getattr(m, n))
        setattr(m, n, f)


def _segment_hook(pl, ts):
    """server/pipeline.py:320-338 with the clusters of a segment boundary muxed
    concurrently by the native muxer (byte-identical to mpegts.mux_segment)."""
    from .segmenter import GopAlignmentError, SegmentMuxer

    def _segment(self) -> None:
        cfg = self.config
        fper = cfg.frames_per_segment
        muxer = SegmentMuxer(threads=max(1, len(self.layouts)))
        pending = [[] for _ in self.layouts]
        sequence = 0
        for pack in self._subs["segment"]:
            per_cluster = pl._unbundle_records(pack.payload)
            for c, records in enumerate(per_cluster):
                pending[c].append(records)
            self.ticks_done += 1
            if len(pending[0]) == fper:
                start_pts = sequence * fper * round(pl.PTS_CLOCK / cfg.fps)
                try:
                    bodies = muxer.mux_clusters(pending, cfg.fps, start_pts)
                except GopAlignmentError as e:
                    raise ts.GopAlignmentError(str(e)) from None
                for c, body in enumerate(bodies):
                    self._on_segment(c, sequence, body, cfg.segment_duration)
                    self.segments_published += 1
                pending = [[] for _ in self.layouts]
                sequence += 1
        self._on_end()
    return _segment


_TOKEN = struct.Struct("<4sI")  # views-channel payload: magic + device slot


def _pipeline_hooks(pl, frame_mod, stages_factory, encoder=False, encoder_factory=None):
    """Device-resident replacements of PipelineHandle._interp / _stitch (/ _encode)."""
    if stages_factory is None:
        from .pipeline import DeviceRigStages as stages_factory  # noqa: N813
    from .interp import InterpConfig
    lock = threading.Lock()

    def stages_of(self, cams):
        with lock:
            st = getattr(self, "_b200_stages", None)
            if st is None:
                cfg = self.config
                ic = cfg.interp
                our_cfg = InterpConfig(ic.block_size, ic.search_radius, ic.mask_epsilon, ic.border_band) \
                    if ic is not None else None
                f0 = cams[0]
                st = stages_factory(f0.width, f0.height, int(f0.format), len(cams), cfg.stages,
                                    cfg.views_per_side, our_cfg, max(2, cfg.channel_capacity) + 2)
                self._b200_stages = st
            return st

    def _interp(self) -> None:
        """server/pipeline.py:254-271 with the views left on the device."""
        if self.config.interp is not None and self.config.interp.refine is not None:
            return _SAVED[(pl.PipelineHandle, "_interp")](self)  # per-view host hook: reference flow
        for pack in self._subs["interp"]:
            t0 = time.perf_counter()
            cams = pl._unbundle_frames(pack.payload)
            slot = stages_of(self, cams).interp(cams)
            self.report.add(pl.STAGE_INTERP, time.perf_counter() - t0)
            out = pl.UnifiedDataPack(pl.PackType.FRAME_RAW, _TOKEN.pack(b"B200", slot))
            self.ch_views.put(out.stamped("interp-out"))

    def _stitch(self) -> None:
        """server/pipeline.py:273-292 on the device slot of the tick."""
        if self.config.interp is not None and self.config.interp.refine is not None:
            return _SAVED[(pl.PipelineHandle, "_stitch")](self)
        for pack in self._subs["stitch"]:
            t0 = time.perf_counter()
            magic, slot = _TOKEN.unpack(pack.payload)
            if magic != b"B200":
                raise ValueError("views channel pack is not a device-slot token")
            clusters = self._b200_stages.stitch(slot)
            frames = []
            for c in clusters:
                f = c.frame
                frames.append(frame_mod.Frame(f.width, f.height, frame_mod.PixelFormat(int(f.format)),
                                              tuple(f.planes), f.timestamp))
            self.report.add(pl.STAGE_STITCH, time.perf_counter() - t0)
            out = pl.UnifiedDataPack(pl.PackType.FRAME_RAW, pl._bundle_frames(frames))
            self.ch_clusters.put(out.stamped("stitch-out", time.perf_counter()))

    def _stitch_to_encoder(self) -> None:
        """server/pipeline.py:273-292 with the cluster frames left on the device."""
        if self.config.interp is not None and self.config.interp.refine is not None:
            return _SAVED[(pl.PipelineHandle, "_stitch")](self)
        for pack in self._subs["stitch"]:
            t0 = time.perf_counter()
            magic, slot = _TOKEN.unpack(pack.payload)
            if magic != b"B200":
                raise ValueError("views channel pack is not a device-slot token")
            self._b200_stages.stitch_device(slot)
            self.report.add(pl.STAGE_STITCH, time.perf_counter() - t0)
            out = pl.UnifiedDataPack(pl.PackType.FRAME_RAW, _TOKEN.pack(b"B2CL", slot))
            self.ch_clusters.put(out.stamped("stitch-out", time.perf_counter()))

    def _encode(self) -> None:
        """server/pipeline.py:294-318: every tile's FVT1 record, transform on the device."""
        if self.config.interp is not None and self.config.interp.refine is not None:
            return _SAVED[(pl.PipelineHandle, "_encode")](self)
        cfg = self.config
        for pack in self._subs["encode"]:
            t0 = time.perf_counter()
            self.report.add(pl.STAGE_SCHEDULE, t0 - pack.trace_time("stitch-out"))
            magic, slot = _TOKEN.unpack(pack.payload)
            if magic != b"B2CL":
                raise ValueError("clusters channel pack is not a device-slot token")
            per_cluster = self._b200_stages.encode(slot, cfg.quality, cfg.gop, encoder_factory)
            self.report.add(pl.STAGE_ENCODE, time.perf_counter() - t0)
            out = pl.UnifiedDataPack(pl.PackType.TILE_BITSTREAM, pl._bundle_records(per_cluster))
            self.ch_encoded.put(out.stamped("encode-out"))

    if encoder:
        return {"_interp": _interp, "_stitch": _stitch_to_encoder, "_encode": _encode}
    return {"_interp": _interp, "_stitch": _stitch}


def uninstall(fvv=None) -> None:
    for (m, n), f in _SAVED.items():
        setattr(m, n, f)
    _SAVED.clear()


__all__ = ["install", "uninstall", "packed"]

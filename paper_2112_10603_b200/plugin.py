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
"""
from __future__ import annotations

import importlib

from . import cluster as _cluster
from . import interp as _interp
from .frame import packed

_SAVED: dict = {}


def _ref_frame(fvv_frame_mod, ours, template):
    """This package's Frame -> the reference's Frame class (same planes)."""
    return fvv_frame_mod.Frame(ours.width, ours.height, template.format.__class__(int(ours.format)),
                               tuple(ours.planes), ours.timestamp)


def install(fvv) -> None:
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

    repl = {(interp_mod, "interpolate"): interpolate, (interp_mod, "dense_views"): dense_views,
            (cluster_mod, "downscale"): downscale,
            (cluster_mod, "assemble_cluster_frame"): assemble_cluster_frame}
    for modname, names in ((".server.pipeline", ("dense_views", "downscale", "assemble_cluster_frame")),
                           (".report", ("dense_views",))):
        try:
            m = importlib.import_module(fvv.__name__ + modname)
        except ImportError:
            continue
        for n in names:
            if hasattr(m, n):
                src = interp_mod if n in ("interpolate", "dense_views") else cluster_mod
                repl[(m, n)] = repl[(src, n)]
    for (m, n), f in repl.items():
        _SAVED.setdefault((m, n), getattr(m, n))
        setattr(m, n, f)


def uninstall(fvv=None) -> None:
    for (m, n), f in _SAVED.items():
        setattr(m, n, f)
    _SAVED.clear()


__all__ = ["install", "uninstall", "packed"]

"""plugin.install against the REAL reference package (/root/reference, build
container only; skipped elsewhere).

* every seam SURVEY.md sec. 8(b) names is rebound in the real module layout
  (fvv.interp, fvv.cluster, the copies imported into fvv.server.pipeline and
  fvv.report) and restored by uninstall;
* with pipeline=True the reference's own `run_pipeline` (reader -> _interp ->
  _stitch -> encoder -> TS segments, server/pipeline.py:193-406) runs through
  the device-resident stage hooks and publishes byte-identical TS segments
  to the unmodified reference pipeline.  This container has no GPU, so the
  stage state is an oracle-backed stand-in with DeviceRigStages' interface
  (interp(cams) -> slot, stitch(slot) -> ClusterFrames); the hook code, the
  token channel, the report/trace stamps and the reference's host stages are
  the real ones.  The device side of DeviceRigStages is checked against the
  same goldens on the GPU (tests/test_gpu_parity.py).
"""
import importlib
import sys

import numpy as np
import pytest

import refimpl
from oracle import oracle as O

pytestmark = [pytest.mark.reference,
              pytest.mark.skipif(not refimpl.available(), reason="/root/reference not present")]


@pytest.fixture()
def fvv():
    for m in [m for m in sys.modules if m == "fvv" or m.startswith("fvv.")]:
        del sys.modules[m]
    if refimpl.REF_SRC not in sys.path:
        sys.path.insert(0, refimpl.REF_SRC)
    mod = importlib.import_module("fvv")
    for sub in ("frame", "interp", "cluster", "server.pipeline", "report"):
        importlib.import_module("fvv." + sub)
    yield mod
    from paper_2112_10603_b200 import plugin
    plugin.uninstall()


SEAMS = [("interp", "interpolate"), ("interp", "dense_views"), ("cluster", "downscale"),
         ("cluster", "assemble_cluster_frame"), ("server.pipeline", "dense_views"),
         ("server.pipeline", "downscale"), ("server.pipeline", "assemble_cluster_frame"),
         ("report", "dense_views")]


def test_install_rebinds_the_real_package(fvv):
    from paper_2112_10603_b200 import plugin
    mods = {m: importlib.import_module("fvv." + m) for m, _ in SEAMS}
    before = {(m, n): getattr(mods[m], n) for m, n in SEAMS}
    h = mods["server.pipeline"].PipelineHandle
    hooks_before = (h._interp, h._stitch)
    plugin.install(fvv, pipeline=True)
    for (m, n), f in before.items():
        assert getattr(mods[m], n) is not f, f"fvv.{m}.{n} not rebound"
        assert getattr(mods[m], n).__module__.startswith("paper_2112_10603_b200")
    assert mods["server.pipeline"].dense_views is mods["interp"].dense_views
    assert (h._interp, h._stitch) != hooks_before
    plugin.uninstall()
    for (m, n), f in before.items():
        assert getattr(mods[m], n) is f
    assert (h._interp, h._stitch) == hooks_before


class OracleStages:
    """Test stand-in with DeviceRigStages' interface, computing with the oracle."""

    calls = []

    def __init__(self, width, height, fmt, cams, stages, vps, config, slots):
        from paper_2112_10603_b200.cluster import build_layouts, tile_rects
        from paper_2112_10603_b200.viewmodel import ViewIndexModel
        self.w, self.h, self.fmt, self.C, self.S, self.vps = width, height, fmt, cams, stages, vps
        self.cfg = config
        self.layouts = build_layouts(ViewIndexModel(cams, stages), vps)
        self.tile_rects = tile_rects
        self.slots = [None] * slots
        self.next = 0
        OracleStages.calls.append(("init", slots))

    def interp(self, frames):
        from paper_2112_10603_b200.frame import packed
        cams = np.stack([packed(f) for f in frames])
        kw = dict(block_size=self.cfg.block_size, search_radius=self.cfg.search_radius, eps=self.cfg.mask_epsilon)
        views = O.rig_dense_views(cams, self.w, self.h, self.fmt, self.S, **kw)
        k = self.next
        self.next = (k + 1) % len(self.slots)
        self.slots[k] = (views, [f.timestamp for f in frames])
        OracleStages.calls.append(("interp", k))
        return k

    def stitch(self, slot):
        from paper_2112_10603_b200.cluster import ClusterFrame
        from paper_2112_10603_b200.frame import frame_from_packed
        views, stamps = self.slots[slot]
        out = []
        for lay in self.layouts:
            smalls = np.stack([O.downscale(views[t.index], self.w, self.h, self.fmt, 4)
                               for t in lay.tiles if t.tier == "quarter"])
            st, sw = O.assemble_cluster(views[lay.anchor_index], self.w, self.h, self.fmt, smalls)
            fr = frame_from_packed(st, sw, self.h, self.fmt, stamps[lay.anchor_index >> self.S])
            out.append(ClusterFrame(lay.cluster_id, fr, self.tile_rects(lay, self.w, self.h)))
        OracleStages.calls.append(("stitch", slot))
        return out

    # encoder hand-off interface (DeviceRigStages.stitch_device / .encode)
    def stitch_device(self, slot):
        self.slots[slot] = self.slots[slot] + (self.stitch(slot),)

    def encode(self, slot, quality, gop, encoder_factory=None):
        from fvv.codec import TileEncoder
        from fvv.frame import PixelFormat, frame_from_planes
        encs = self.__dict__.setdefault("encs", {})
        per_cluster = []
        for cf in self.slots[slot][2]:
            recs = []
            for rect in cf.tile_map:
                tile = cf.crop(rect)
                ref = frame_from_planes(list(tile.planes), PixelFormat(int(tile.format)), tile.timestamp)
                enc = encs.setdefault((cf.cluster_id, rect.index), TileEncoder(quality, gop))
                recs.append(enc.encode(ref).to_bytes())
            per_cluster.append(recs)
        OracleStages.calls.append(("encode", slot))
        return per_cluster


def _run(fvv, ticks):
    from fvv.interp import InterpConfig
    from fvv.server.pipeline import PipelineConfig, PrerenderedSource, run_pipeline
    cfg = PipelineConfig(scene_dir=None, stages=2, views_per_side=3, fps=30, segment_duration=0.2, gop=6,
                         quality=75, port=0, interp=InterpConfig(search_radius=(4, 2, 1)))
    segs = {}
    h = run_pipeline(cfg, PrerenderedSource(ticks, iterations=6),
                     on_segment=lambda c, seq, body, dur: segs.__setitem__((c, seq), bytes(body)))
    h.wait(timeout=600)
    return segs, h


def test_pipeline_hooks_publish_reference_identical_segments(fvv):
    from fvv.scene import SceneSpec, SyntheticScene, default_sprites_for
    from paper_2112_10603_b200 import plugin
    spec = SceneSpec(seed=42, camera_count=3, width=64, height=48, format="yuv420",
                     sprites=default_sprites_for(64, 48))
    scene = SyntheticScene(spec)
    ticks = [[scene.render_view(float(c), t) for c in range(3)] for t in range(3)]
    ref_segs, _ = _run(fvv, ticks)
    assert len(ref_segs) == 3  # one 6-frame segment per cluster
    OracleStages.calls = []
    plugin.install(fvv, pipeline=True, stages_factory=OracleStages)
    got_segs, handle = _run(fvv, ticks)
    plugin.uninstall()
    assert [c for c, _ in OracleStages.calls].count("interp") == 6
    assert [c for c, _ in OracleStages.calls].count("stitch") == 6
    assert set(got_segs) == set(ref_segs)
    for k in ref_segs:
        assert got_segs[k] == ref_segs[k], f"segment {k} differs"
    stats = handle.report.stats()
    assert stats["view interpolation"]["count"] == 6 and stats["adaptive stitch"]["count"] == 6


def test_pipeline_hooks_with_encoder_hand_off(fvv):
    """install(fvv, pipeline=True, encoder=True): _stitch leaves the cluster
    frames on the device and _encode reads them there; the clusters channel
    carries slot tokens.  Segments equal the unmodified reference pipeline's."""
    from fvv.scene import SceneSpec, SyntheticScene, default_sprites_for
    from paper_2112_10603_b200 import plugin
    spec = SceneSpec(seed=7, camera_count=3, width=64, height=48, format="yuv420",
                     sprites=default_sprites_for(64, 48))
    scene = SyntheticScene(spec)
    ticks = [[scene.render_view(float(c), t) for c in range(3)] for t in range(3)]
    ref_segs, _ = _run(fvv, ticks)
    OracleStages.calls = []
    plugin.install(fvv, pipeline=True, stages_factory=OracleStages, encoder=True)
    got_segs, handle = _run(fvv, ticks)
    plugin.uninstall()
    kinds = [c for c, _ in OracleStages.calls]
    assert kinds.count("interp") == 6 and kinds.count("encode") == 6
    assert got_segs == ref_segs
    assert handle.report.stats()["encoder"]["count"] == 6


def test_segment_hook_on_the_real_pipeline(fvv):
    """install(fvv, segment=True, names=False) (host code, runs here): the reference's
    own pipeline with the native concurrent TS muxer publishes the same bytes."""
    from fvv.scene import SceneSpec, SyntheticScene, default_sprites_for
    from paper_2112_10603_b200 import plugin
    spec = SceneSpec(seed=3, camera_count=3, width=64, height=48, format="yuv420",
                     sprites=default_sprites_for(64, 48))
    scene = SyntheticScene(spec)
    ticks = [[scene.render_view(float(c), t) for c in range(3)] for t in range(2)]
    ref_segs, _ = _run(fvv, ticks)
    plugin.install(fvv, segment=True, names=False)
    h = importlib.import_module("fvv.server.pipeline").PipelineHandle
    assert h._segment.__module__.startswith("paper_2112_10603_b200")
    got_segs, handle = _run(fvv, ticks)
    plugin.uninstall()
    assert got_segs == ref_segs and handle.segments_published == 3

"""The CPU oracle (oracle/fvv_oracle.c) against the LIVE reference
(/root/reference, imported through tests/refimpl.py) -- build container
only; skipped where the reference is absent (the GPU box).

Byte-equality at the sizes the golden fixtures do not reach: a 1080p YUV420
scene pair at a realistic 1080p disparity (gain 36), BASELINE config 1 (RGB8
448x256, seed 42) with flows and mask, ragged sizes, and a 4-camera rig with
every cluster frame (cluster.py:58-191).
"""
import numpy as np
import pytest

import refimpl
from oracle import oracle as O

pytestmark = [pytest.mark.reference,
              pytest.mark.skipif(not refimpl.available(), reason="/root/reference not present")]


def _check_pair(L, R, fmt, diag=True):
    interp = refimpl.load()
    w, h = L.width, L.height
    if diag:
        mid, d = interp.interpolate(L, R, diagnostics=True)
        out, od = O.interpolate(refimpl.packed(L), refimpl.packed(R), w, h, fmt, with_diag=True)
        assert np.array_equal(od["flow_lr"], d.scales[-1].flow_lr.vectors)
        assert np.array_equal(od["flow_rl"], d.scales[-1].flow_rl.vectors)
        assert np.array_equal(od["mask"], d.mask)
    else:
        mid = interp.interpolate(L, R)
        out = O.interpolate(refimpl.packed(L), refimpl.packed(R), w, h, fmt)
    assert np.array_equal(out, refimpl.packed(mid))


def test_1080p_yuv420_scene_gain36():
    L, R = refimpl.scene_pair(1920, 1080, "yuv420", gain=36.0)
    _check_pair(L, R, 1)


def test_cfg1_rgb8_448x256():
    L, R = refimpl.scene_pair(448, 256, "rgb8")
    _check_pair(L, R, 2)


@pytest.mark.parametrize("w,h,fmt", [(328, 200, "gray8"), (1000, 604, "yuv420")])
def test_ragged_noise(w, h, fmt):
    refimpl.load()
    from fvv.frame import PixelFormat, frame_from_planes, plane_shapes
    pf = {"gray8": PixelFormat.GRAY8, "yuv420": PixelFormat.YUV420}[fmt]
    rng = np.random.default_rng(w + h)
    L, R = (frame_from_planes([rng.integers(0, 256, s, dtype=np.uint8) for s in plane_shapes(w, h, pf)], pf)
            for _ in range(2))
    _check_pair(L, R, int(pf), diag=False)


def test_4_camera_rig_with_clusters():
    interp = refimpl.load()
    from fvv.cluster import assemble_cluster_frame, build_layouts, downscale
    from fvv.viewmodel import ViewIndexModel
    w, h, C, S, vps = 320, 192, 4, 2, 4
    cams = refimpl.scene_pair(w, h, "yuv420", cams=C, positions=tuple(float(c) for c in range(C)))
    model = ViewIndexModel(C, S)
    step = 1 << S
    allv = [None] * model.total_views
    for c, fr in enumerate(cams):
        allv[c * step] = fr
    for c in range(C - 1):
        allv[c * step + 1:(c + 1) * step] = interp.dense_views(cams[c], cams[c + 1], S)
    views = O.rig_dense_views(np.stack([refimpl.packed(c) for c in cams]), w, h, 1, S)
    assert np.array_equal(views, np.stack([refimpl.packed(v) for v in allv]))
    for lay in build_layouts(model, vps):
        smalls = [downscale(allv[t.index], 4) for t in lay.tiles if t.tier == "quarter"]
        cf = assemble_cluster_frame(allv[lay.anchor_index], smalls, lay)
        a = lay.anchor_index
        osm = np.stack([O.downscale(views[t.index], w, h, 1, 4) for t in lay.tiles if t.tier == "quarter"])
        ref, sw = O.assemble_cluster(views[a], w, h, 1, osm)
        assert sw == cf.frame.width
        assert np.array_equal(ref, refimpl.packed(cf.frame))

"""Generate the golden fixtures from the REFERENCE itself (run in the build
container, where /root/reference exists):

    PYTHONPATH=/root/repo python tests/golden/make_golden.py

Each case stores packed input frames, the reference's packed output(s) and,
for single interpolations, the final full-resolution flows and the mask.
The reference is imported through tests/refimpl.py (two documented RGB8
overrides).  Versions are stamped into every file.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import refimpl  # noqa: E402

FMT = {"gray8": 0, "yuv420": 1, "rgb8": 2}


def versions():
    import numba
    import scipy
    return f"numpy {np.__version__}; scipy {scipy.__version__}; numba {numba.__version__}"


def rand_frame(rng, w, h, fmt):
    from fvv.frame import frame_from_planes, PixelFormat, plane_shapes
    pf = {"gray8": PixelFormat.GRAY8, "yuv420": PixelFormat.YUV420, "rgb8": PixelFormat.RGB8}[fmt]
    planes = [rng.integers(0, 256, s, dtype=np.uint8) for s in plane_shapes(w, h, pf)]
    return frame_from_planes(planes, pf)


def shifted(rng, w, h, shift):
    """Smooth texture shifted by `shift` px: a realistic flow target."""
    from fvv.frame import gray
    from fvv.scene import _value_noise
    tex = np.rint(28 + 190 * _value_noise(rng, h, w + abs(shift), (13, 5), (0.6, 0.4))).astype(np.uint8)
    return gray(tex[:, shift:shift + w].copy()), gray(tex[:, :w].copy())


def main():
    interp = refimpl.load()
    from fvv.cluster import downscale, assemble_cluster_frame, build_layouts
    from fvv.viewmodel import ViewIndexModel
    rng = np.random.default_rng(20261018)
    ver = versions()
    out = {}

    def single(name, L, R, fmt):
        d = dict(kind="interp", w=L.width, h=L.height, fmt=FMT[fmt], left=refimpl.packed(L),
                 right=refimpl.packed(R))
        try:
            mid, diag = interp.interpolate(L, R, diagnostics=True)
            d.update(flow_lr=diag.scales[-1].flow_lr.vectors, flow_rl=diag.scales[-1].flow_rl.vectors,
                     mask=diag.mask)
            if L.width * L.height <= 96 * 72:  # per-level ScaleDiagnostics (interp.py:114-128)
                for s, sd in enumerate(diag.scales):
                    d[f"lv{s}_flow_lr"] = sd.flow_lr.vectors
                    d[f"lv{s}_flow_rl"] = sd.flow_rl.vectors
                    d[f"lv{s}_err_lr"] = sd.match_error_lr
                    d[f"lv{s}_err_rl"] = sd.match_error_rl
                    if s < 2:  # coarse-scale mask and blend (interp.py:119-127)
                        d[f"lv{s}_mask"] = sd.mask
                        d[f"lv{s}_blend"] = sd.blend_luma
        except ValueError:  # per-level diagnostics need >= 2 px per axis at 1/4 scale
            mid = interp.interpolate(L, R)
        d["out"] = refimpl.packed(mid)
        out[name] = d

    # scenes (reference SyntheticScene, seed 42)
    for (w, h, fmt) in [(64, 48, "gray8"), (96, 72, "yuv420"), (448, 256, "rgb8")]:
        L, R = refimpl.scene_pair(w, h, fmt)
        single(f"scene_{fmt}_{w}x{h}", L, R, fmt)
    # random noise, ragged block grids and degenerate sizes
    for (w, h, fmt) in [(36, 20, "gray8"), (4, 4, "gray8"), (8, 12, "yuv420"), (44, 28, "rgb8"),
                        (40, 24, "yuv420")]:
        single(f"noise_{fmt}_{w}x{h}", rand_frame(rng, w, h, fmt), rand_frame(rng, w, h, fmt), fmt)
    L, R = shifted(rng, 96, 64, 6)
    single("shift6_gray8_96x64", L, R, "gray8")
    # identity (test_interp.py:14-21)
    f = rand_frame(rng, 48, 32, "gray8")
    single("identity_gray8_48x32", f, f, "gray8")
    # recursive dense views (interp.py:151-170)
    L, R = refimpl.scene_pair(64, 48, "yuv420")
    views = interp.dense_views(L, R, 3)
    out["dense3_yuv420_64x48"] = dict(kind="dense", w=64, h=48, fmt=1, stages=3, left=refimpl.packed(L),
                                      right=refimpl.packed(R),
                                      out=np.stack([refimpl.packed(v) for v in views]))
    # tiling (cluster.py:58-191): 3 cameras, 2 stages, vps 2
    model = ViewIndexModel(3, 2)
    layouts = build_layouts(model, 2)
    cams = refimpl.scene_pair(64, 48, "yuv420", cams=3, positions=(0.0, 1.0, 2.0))
    allv = [None] * model.total_views
    step = 1 << model.stages
    for c, fr in enumerate(cams):
        allv[c * step] = fr
    for c in range(2):
        allv[c * step + 1:(c + 1) * step] = interp.dense_views(cams[c], cams[c + 1], model.stages)
    clusters = []
    for lay in layouts:
        smalls = [downscale(allv[t.index], 4) for t in lay.tiles if t.tier == "quarter"]
        cf = assemble_cluster_frame(allv[lay.anchor_index], smalls, lay)
        clusters.append(dict(w=cf.frame.width, frame=refimpl.packed(cf.frame),
                             rects=np.array([[r.index, r.tier == "full", r.x, r.y, r.width, r.height]
                                             for r in cf.tile_map], np.int32)))
    out["rig3_s2_vps2_yuv420_64x48"] = dict(
        kind="rig", w=64, h=48, fmt=1, stages=2, vps=2,
        cams=np.stack([refimpl.packed(c) for c in cams]),
        views=np.stack([refimpl.packed(v) for v in allv]),
        quarters=np.stack([refimpl.packed(downscale(v, 4)) for v in allv]),
        cluster_w=np.array([c["w"] for c in clusters]),
        clusters=np.concatenate([c["frame"] for c in clusters]),
        cluster_sizes=np.array([c["frame"].size for c in clusters]),
        rects=np.concatenate([c["rects"] for c in clusters]),
        rect_counts=np.array([len(c["rects"]) for c in clusters]))
    for name, d in out.items():
        d = dict(d)
        d["versions"] = np.array(ver)
        d["kind"] = np.array(d["kind"])
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
        print(name)


if __name__ == "__main__":
    main()

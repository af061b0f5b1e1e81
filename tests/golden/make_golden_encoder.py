"""Encoder goldens from the REFERENCE (build container only):

    PYTHONPATH=/root/repo python tests/golden/make_golden_encoder.py

A 3-camera 64x48 YUV420 rig (reference SyntheticScene, sprites move with t),
stages 2, views_per_side 3: for each of 4 ticks the reference's cluster frames
(dense_views + downscale + assemble_cluster_frame, server/pipeline.py:254-292)
and the FVT1 records its encoder stage writes for them
(server/pipeline.py:294-318: one codec.TileEncoder per (cluster, tile),
records of cf.crop(rect) in tile-map order).  Two settings: quality 75 / gop 2
(I and P records, lossy DCT path) and quality 100 / gop 3 (lossless lifting).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import refimpl  # noqa: E402


def main():
    from make_golden import versions
    interp = refimpl.load()
    from fvv.cluster import assemble_cluster_frame, build_layouts, downscale
    from fvv.codec import TileEncoder
    from fvv.scene import SceneSpec, SyntheticScene, default_sprites_for
    from fvv.viewmodel import ViewIndexModel
    W, H, C, S, vps, T = 64, 48, 3, 2, 3, 4
    spec = SceneSpec(seed=42, camera_count=C, width=W, height=H, format="yuv420", sprites=default_sprites_for(W, H))
    scene = SyntheticScene(spec)
    model = ViewIndexModel(C, S)
    layouts = build_layouts(model, vps)
    step = 1 << S
    ticks = []
    for t in range(T):
        cams = [scene.render_view(float(c), t) for c in range(C)]
        allv = [None] * model.total_views
        for c, fr in enumerate(cams):
            allv[c * step] = fr
        for c in range(C - 1):
            allv[c * step + 1:(c + 1) * step] = interp.dense_views(cams[c], cams[c + 1], S)
        cfs = []
        for lay in layouts:
            smalls = [downscale(allv[x.index], 4) for x in lay.tiles if x.tier == "quarter"]
            cfs.append(assemble_cluster_frame(allv[lay.anchor_index], smalls, lay))
        ticks.append(cfs)
    out = dict(kind=np.array("encoder"), w=W, h=H, cams=C, stages=S, vps=vps, ticks=T, versions=np.array(versions()),
               clusters=np.stack([np.concatenate([refimpl.packed(cf.frame) for cf in cfs]) for cfs in ticks]))
    for name, q, gop in (("q75", 75, 2), ("q100", 100, 3)):
        encs = {}
        recs = []
        for cfs in ticks:
            for cf in cfs:
                for rect in cf.tile_map:
                    enc = encs.setdefault((cf.cluster_id, rect.index), TileEncoder(q, gop))
                    recs.append(enc.encode(cf.crop(rect)).to_bytes())
        out[f"{name}_records"] = np.frombuffer(b"".join(recs), np.uint8)
        out[f"{name}_lengths"] = np.array([len(r) for r in recs], np.int64)
    np.savez_compressed(os.path.join(HERE, "encoder_rig3_yuv420_64x48.npz"), **out)
    print("encoder_rig3_yuv420_64x48", {k: v.shape for k, v in out.items() if hasattr(v, "shape")})


if __name__ == "__main__":
    main()

"""1080p golden fixtures from the REFERENCE itself (build container only):

    PYTHONPATH=/root/repo python tests/golden/make_golden_1080p.py

The inputs are NOT stored: they are `bench.synth_rig(W, H, fmt, cams, seed)`
frames (numpy + scipy, deterministic), which the GPU box regenerates from the
stored parameters.  What is stored is what the reference computed on them:

* ref1080_pair: one 1920x1080 YUV420 `interpolate()` (interp.py:97-148) --
  the full output frame, its final f32 flows' SHA-256 and the f64 mask's.
* ref1080_cfg3: BASELINE config 3 -- a 4-camera 1080p YUV420 rig,
  `dense_views(n=4)` per gap (interp.py:151-170, server/pipeline.py:254-271)
  and the 4 cluster frames (views_per_side 16; cluster.py:58-191,
  server/pipeline.py:273-292) -- SHA-256 of every global view and every
  cluster frame (45 + 4 + 4 frames; storing them would be ~170 MB).

The reference is imported through tests/refimpl.py; versions are stamped.
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, ROOT)
import refimpl  # noqa: E402
from bench import synth_rig  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_frames(packed_frames, w, h):
    from fvv.frame import PixelFormat
    from paper_2112_10603_b200.frame import plane_shapes
    from fvv.frame import frame_from_planes
    out = []
    for p in packed_frames:
        planes, off = [], 0
        for shape in plane_shapes(w, h, 1):
            n = int(np.prod(shape))
            planes.append(p[off:off + n].reshape(shape).copy())
            off += n
        out.append(frame_from_planes(planes, PixelFormat.YUV420))
    return out


def main():
    from make_golden import versions
    interp = refimpl.load()
    from fvv.cluster import assemble_cluster_frame, build_layouts, downscale
    from fvv.viewmodel import ViewIndexModel
    ver = versions()
    W, H = 1920, 1080

    t0 = time.time()
    cams = synth_rig(W, H, 1, 2, seed=1080)
    L, R = ref_frames(cams, W, H)
    mid, diag = interp.interpolate(L, R, diagnostics=True)
    np.savez_compressed(os.path.join(HERE, "ref1080_pair.npz"), kind=np.array("ref1080"), w=W, h=H, fmt=1,
                        cams=2, seed=1080, left=0, right=1, out=refimpl.packed(mid),
                        flow_lr_sha=np.array(sha(diag.scales[-1].flow_lr.vectors)),
                        flow_rl_sha=np.array(sha(diag.scales[-1].flow_rl.vectors)),
                        mask_sha=np.array(sha(diag.mask)), versions=np.array(ver))
    print(f"ref1080_pair {time.time() - t0:.1f}s")

    t0 = time.time()
    C, stages, vps = 4, 4, 16
    cams = synth_rig(W, H, 1, C, seed=42)
    frames = ref_frames(cams, W, H)
    model = ViewIndexModel(C, stages)
    step = 1 << stages
    allv = [None] * model.total_views
    for c, fr in enumerate(frames):
        allv[c * step] = fr
    for c in range(C - 1):
        allv[c * step + 1:(c + 1) * step] = interp.dense_views(frames[c], frames[c + 1], stages)
    view_sha = [sha(refimpl.packed(v)) for v in allv]
    cl_sha, cl_w, rects = [], [], []
    for lay in build_layouts(model, vps):
        smalls = [downscale(allv[t.index], 4) for t in lay.tiles if t.tier == "quarter"]
        cf = assemble_cluster_frame(allv[lay.anchor_index], smalls, lay)
        cl_sha.append(sha(refimpl.packed(cf.frame)))
        cl_w.append(cf.frame.width)
        rects.append(np.array([[r.index, r.tier == "full", r.x, r.y, r.width, r.height] for r in cf.tile_map],
                              np.int32))
    np.savez_compressed(os.path.join(HERE, "ref1080_cfg3.npz"), kind=np.array("ref1080_rig"), w=W, h=H, fmt=1,
                        cams=C, seed=42, stages=stages, vps=vps, view_sha=np.array(view_sha),
                        cluster_sha=np.array(cl_sha), cluster_w=np.array(cl_w),
                        rects=np.concatenate(rects), rect_counts=np.array([len(r) for r in rects]),
                        versions=np.array(ver))
    print(f"ref1080_cfg3 {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()

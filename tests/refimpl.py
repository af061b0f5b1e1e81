"""Adapter that imports the read-only reference (only present in the build
container, never on the GPU box) with the two RGB8 overrides SURVEY.md
sec. 0.4 / 8(c) documents:

1. ``backward_warp``: for RGB8 skip ``warp.py:37`` (warp_plane on the (h,w,3)
   plane raises) and run only the per-channel branch ``warp.py:42-45``.
2. ``estimate_mask``: compare ``planes[0].shape[:2]`` (``warp.py:58-61``).

Everything else is the reference's own code.  Used only to pin the oracle
and to generate tests/golden/ fixtures.
"""
from __future__ import annotations

import os
import sys

REF_SRC = "/root/reference/pkg/src"


def available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "fvv"))


def load():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import numpy as np
    import fvv.interp as interp
    import fvv.warp as warp
    from fvv.frame import PixelFormat, frame_from_planes
    from fvv.imageops import to_uint8, warp_plane

    if getattr(warp, "_b200_overrides", False):
        return interp
    orig_bw = warp.backward_warp
    orig_em = warp.estimate_mask

    def backward_warp(image, flow):
        if image.format != PixelFormat.RGB8:
            return orig_bw(image, flow)
        if (flow.width, flow.height) != (image.width, image.height):
            raise ValueError("flow does not match frame")
        rgb = image.planes[0]
        planes = [to_uint8(np.stack([warp_plane(rgb[..., c], flow.vectors) for c in range(3)],
                                    axis=-1))]
        return frame_from_planes(planes, image.format, image.timestamp)

    def estimate_mask(warped_left, warped_right, error_left, error_right, epsilon=1e-3):
        shapes = {warped_left.planes[0].shape[:2], warped_right.planes[0].shape[:2],
                  error_left.shape, error_right.shape}
        if len(shapes) != 1:
            raise ValueError(f"mask inputs disagree on shape: {sorted(shapes)}")
        m = (error_right + epsilon) / (error_left + error_right + 2.0 * epsilon)
        return warp.OcclusionMask(np.clip(m, 0.0, 1.0))

    warp.backward_warp = backward_warp
    warp.estimate_mask = estimate_mask
    interp.backward_warp = backward_warp
    interp.estimate_mask = estimate_mask
    warp._b200_overrides = True
    return interp


def packed(frame):
    """Frame -> packed plane bytes (frame.py:99-101 raw_planes order)."""
    import numpy as np
    return np.frombuffer(frame.raw_planes(), np.uint8).copy()


def scene_pair(w, h, fmt="yuv420", seed=42, cams=2, positions=(0.0, 1.0), t=0, gain=None):
    """Two (or more) views of the reference SyntheticScene (scene.py:204-231)."""
    load()
    from fvv.scene import SceneSpec, SyntheticScene, default_sprites_for
    kw = {}
    if gain is not None:
        kw["gain"] = gain
    spec = SceneSpec(seed=seed, camera_count=cams, width=w, height=h,
                     format="yuv420" if fmt == "rgb8" else fmt,
                     sprites=default_sprites_for(w, h), **kw)
    sc = SyntheticScene(spec)
    frames = [sc.render_view(p, t) for p in positions]
    if fmt == "rgb8":
        from fvv.frame import frame_from_planes, PixelFormat
        frames = [frame_from_planes([frame_to_rgb(f)], PixelFormat.RGB8, f.timestamp) for f in frames]
    return frames


def frame_to_rgb(frame):
    """YUV420/gray -> RGB8 exactly as client/ui.py:17-30 does (restated here
    because that module imports PIL, which this image lacks)."""
    import numpy as np
    from fvv.frame import PixelFormat
    if frame.format == PixelFormat.RGB8:
        return frame.planes[0]
    y = frame.planes[0].astype(np.float64)
    if frame.format == PixelFormat.GRAY8:
        return np.repeat(y[..., None], 3, axis=2).astype(np.uint8)
    u = np.repeat(np.repeat(frame.planes[1].astype(np.float64) - 128, 2, 0), 2, 1)
    v = np.repeat(np.repeat(frame.planes[2].astype(np.float64) - 128, 2, 0), 2, 1)
    u = u[:frame.height, :frame.width]
    v = v[:frame.height, :frame.width]
    rgb = np.stack([y + 1.402 * v, y - 0.344136 * u - 0.714136 * v, y + 1.772 * u], axis=-1)
    return np.clip(np.rint(rgb), 0, 255).astype(np.uint8)

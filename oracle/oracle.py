"""ctypes front-end of the CPU oracle (oracle/fvv_oracle.c).

TEST INFRASTRUCTURE ONLY.  Importable from tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / ``--impl reference`` leg -- never from the
product package ``paper_2112_10603_b200``.  It restates the reference path
(/root/reference/pkg/src/fvv: interp.py:67-170, flow.py:40-131,
warp.py:27-88, imageops.py:10-56, _kernels.py:28-193, cluster.py:77-191)
literally in C; tests/test_oracle_vs_reference.py pins it against the live
reference itself, and tests/golden/ holds vectors the reference produced.

Frames cross this boundary as packed plane bytes in the reference's
``Frame.raw_planes()`` order (frame.py:99-101): Y then U then V, or one
interleaved RGB plane.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

GRAY8, YUV420, RGB8 = 0, 1, 2
_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "libfvv_oracle.so"
_lib = None


def build(force: bool = False) -> Path:
    """Compile the oracle with the committed Makefile (gcc, -ffp-contract=off)."""
    if force or not _LIB_PATH.exists() or \
            _LIB_PATH.stat().st_mtime < (_HERE / "fvv_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB_PATH))
        P = ctypes.c_void_p
        i = ctypes.c_int
        L.fvvo_frame_bytes.restype = ctypes.c_long
        L.fvvo_frame_bytes.argtypes = [i, i, i]
        L.fvvo_interpolate.argtypes = [P, P, i, i, i, P, P, ctypes.c_double, P, P, P, P]
        L.fvvo_dense_views.argtypes = [P, P, i, i, i, i, P, P, ctypes.c_double, P]
        L.fvvo_downscale.argtypes = [P, i, i, i, i, P]
        L.fvvo_assemble_cluster.argtypes = [P, i, i, i, P, i, i, P, P]
        L.fvvo_estimate_flow_level.argtypes = [P, P, i, i, P, P, i, i, i, i, P, P, P, P, P, P]
        L.fvvo_candidate_order.argtypes = [i, P, P, P]
        L.fvvo_sad_search.argtypes = [P, i, i, P, i, i, P]
        L.fvvo_level_mask.argtypes = [P, P, i, i, P, P, ctypes.c_double, P, P]
        L.fvvo_num_threads.restype = i
        L.fvvo_set_threads.argtypes = [i]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def frame_bytes(w: int, h: int, fmt: int) -> int:
    return int(lib().fvvo_frame_bytes(w, h, fmt))


def set_threads(n: int) -> None:
    lib().fvvo_set_threads(int(n))


def num_threads() -> int:
    return int(lib().fvvo_num_threads())


def _cfg(block_size=(8, 8, 8), search_radius=(12, 4, 2)):
    return (np.ascontiguousarray(block_size, dtype=np.int32),
            np.ascontiguousarray(search_radius, dtype=np.int32))


def interpolate(left: np.ndarray, right: np.ndarray, w: int, h: int, fmt: int,
                block_size=(8, 8, 8), search_radius=(12, 4, 2), eps: float = 1e-3,
                with_diag: bool = False):
    """interp.py:97-148 on packed frames; returns packed output (and diag)."""
    fb = frame_bytes(w, h, fmt)
    left = np.ascontiguousarray(left, dtype=np.uint8).reshape(-1)
    right = np.ascontiguousarray(right, dtype=np.uint8).reshape(-1)
    assert left.size == fb and right.size == fb
    out = np.empty(fb, np.uint8)
    bs, rr = _cfg(block_size, search_radius)
    if with_diag:
        flr = np.empty((h, w, 2), np.float32)
        frl = np.empty((h, w, 2), np.float32)
        m = np.empty((h, w), np.float64)
        rc = lib().fvvo_interpolate(_p(left), _p(right), w, h, fmt, _p(bs), _p(rr), eps, _p(out),
                                    _p(flr), _p(frl), _p(m))
    else:
        rc = lib().fvvo_interpolate(_p(left), _p(right), w, h, fmt, _p(bs), _p(rr), eps, _p(out),
                                    None, None, None)
    if rc:
        raise ValueError(f"oracle interpolate failed ({rc})")
    if with_diag:
        return out, {"flow_lr": flr, "flow_rl": frl, "mask": m}
    return out


def dense_views(left, right, w, h, fmt, stages, block_size=(8, 8, 8),
                search_radius=(12, 4, 2), eps=1e-3) -> np.ndarray:
    """interp.py:151-170; returns (2**stages - 1, frame_bytes) uint8."""
    fb = frame_bytes(w, h, fmt)
    n = (1 << stages) - 1
    out = np.empty((n, fb), np.uint8)
    bs, rr = _cfg(block_size, search_radius)
    left = np.ascontiguousarray(left, dtype=np.uint8).reshape(-1)
    right = np.ascontiguousarray(right, dtype=np.uint8).reshape(-1)
    rc = lib().fvvo_dense_views(_p(left), _p(right), w, h, fmt, stages, _p(bs), _p(rr), eps, _p(out))
    if rc:
        raise ValueError(f"oracle dense_views failed ({rc})")
    return out


def downscale(frame, w, h, fmt, factor=4) -> np.ndarray:
    """cluster.py:77-89."""
    out = np.empty(frame_bytes(w // factor, h // factor, fmt), np.uint8)
    frame = np.ascontiguousarray(frame, dtype=np.uint8).reshape(-1)
    rc = lib().fvvo_downscale(_p(frame), w, h, fmt, factor, _p(out))
    if rc:
        raise ValueError("oracle downscale: dimensions not divisible")
    return out


def assemble_cluster(anchor, w, h, fmt, smalls) -> tuple[np.ndarray, int]:
    """cluster.py:143-191 geometry: returns (packed stitched frame, stitched width)."""
    smalls = np.ascontiguousarray(smalls, dtype=np.uint8)
    nsmall = smalls.shape[0] if smalls.ndim == 2 else 0
    cols = (nsmall + 3) // 4
    sw = w + cols * (w // 4)
    out = np.empty(frame_bytes(sw, h, fmt), np.uint8)
    ow = ctypes.c_int(0)
    anchor = np.ascontiguousarray(anchor, dtype=np.uint8).reshape(-1)
    rc = lib().fvvo_assemble_cluster(_p(anchor), w, h, fmt, _p(smalls) if nsmall else None,
                                     nsmall, 0, _p(out), ctypes.byref(ow))
    if rc:
        raise ValueError("oracle assemble: layout error")
    return out, ow.value


def estimate_flow_level(left32, right32, prev, radius, block):
    """flow.py:101-131: returns ((flow_lr, flow_rl), (off_lr, off_rl), (err_lr, err_rl))."""
    h, w = left32.shape
    left32 = np.ascontiguousarray(left32, np.float32)
    right32 = np.ascontiguousarray(right32, np.float32)
    nby, nbx = (h + block - 1) // block, (w + block - 1) // block
    flr = np.empty((h, w, 2), np.float32)
    frl = np.empty((h, w, 2), np.float32)
    olr = np.empty((nby, nbx, 2), np.float32)
    orl = np.empty((nby, nbx, 2), np.float32)
    elr = np.empty((h, w), np.float64)
    erl = np.empty((h, w), np.float64)
    if prev is None:
        plr = prl = None
        ph = pw = 0
    else:
        plr = np.ascontiguousarray(prev[0], np.float32)
        prl = np.ascontiguousarray(prev[1], np.float32)
        ph, pw = plr.shape[:2]
    lib().fvvo_estimate_flow_level(_p(left32), _p(right32), h, w,
                                   _p(plr) if plr is not None else None,
                                   _p(prl) if prl is not None else None, ph, pw, radius, block,
                                   _p(flr), _p(frl), _p(olr), _p(orl), _p(elr), _p(erl))
    return (flr, frl), (olr, orl), (elr, erl)


def level_mask(yl, yr, flow_lr, flow_rl, eps: float = 1e-3):
    """interp.py:119-127 (coarse-scale diagnostics): (mask, blend_luma) f64 of one level."""
    h, w = yl.shape
    yl = np.ascontiguousarray(yl, np.float32)
    yr = np.ascontiguousarray(yr, np.float32)
    flr = np.ascontiguousarray(flow_lr, np.float32)
    frl = np.ascontiguousarray(flow_rl, np.float32)
    m = np.empty((h, w), np.float64)
    b = np.empty((h, w), np.float64)
    lib().fvvo_level_mask(_p(yl), _p(yr), h, w, _p(flr), _p(frl), float(eps), _p(m), _p(b))
    return m, b


def luma_pyramid(frame, w: int, h: int, fmt: int):
    """interp.py:67-71 on a packed frame: [quarter, half, full] f32 planes."""
    frame = np.ascontiguousarray(frame, np.uint8).reshape(-1)
    if fmt == RGB8:
        rgb = frame[:w * h * 3].reshape(h, w, 3).astype(np.float64)
        y = np.rint(0.299 * rgb[..., 0] + 0.587 * rgb[..., 1] + 0.114 * rgb[..., 2]).astype(np.uint8)
    else:
        y = frame[:w * h].reshape(h, w)
    full = y.astype(np.float32)
    half = ((full[0::2, 0::2] + full[0::2, 1::2]) + (full[1::2, 0::2] + full[1::2, 1::2])) / np.float32(4)
    quarter = ((half[0::2, 0::2] + half[0::2, 1::2]) + (half[1::2, 0::2] + half[1::2, 1::2])) / np.float32(4)
    return [quarter.astype(np.float32), half.astype(np.float32), full]


def candidate_order(radius: int):
    side = 2 * radius + 1
    dx = np.empty(side * side, np.int32)
    dy = np.empty(side * side, np.int32)
    idx = np.empty(side * side, np.int32)
    lib().fvvo_candidate_order(radius, _p(dx), _p(dy), _p(idx))
    return dx, dy, idx


def rig_dense_views(cams: np.ndarray, w, h, fmt, stages, **kw) -> np.ndarray:
    """server/pipeline.py:254-271 ``_interp``: all global views of one rig frame.

    cams: (C, frame_bytes).  Returns (total_views, frame_bytes) in global view order.
    """
    C = cams.shape[0]
    step = 1 << stages
    total = (C - 1) * step + 1
    out = np.empty((total, cams.shape[1]), np.uint8)
    for c in range(C):
        out[c * step] = cams[c]
    for c in range(C - 1):
        out[c * step + 1:(c + 1) * step] = dense_views(cams[c], cams[c + 1], w, h, fmt, stages, **kw)
    return out


def available() -> bool:
    try:
        lib()
        return True
    except Exception:  # noqa: BLE001
        return False


if __name__ == "__main__":  # pragma: no cover
    print(build(), num_threads(), os.cpu_count())

"""ctypes binding of include/fvv_b200.h (the C ABI of libfvv_b200.so).

The library is mandatory: there is no CPU or eager-torch fallback anywhere
in this package.  Import works without a GPU (the CPU test suite checks the
exported symbols); every compute entry point calls :func:`require_cuda`
first and raises if the CUDA device or the library is missing.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

from ._build import LIB

FVV_OK, FVV_EINVAL, FVV_ELAYOUT, FVV_ECUDA, FVV_EUNSUPPORTED = 0, -1, -2, -3, -4
FVV_TUNE_SCAN_COOP_MIN, FVV_TUNE_SADW_RB_MIN_CTAS, FVV_TUNE_MASK_COLS2, FVV_TUNE_PDL = 0, 1, 2, 3
FVV_DENSE_RECURSIVE, FVV_DENSE_DIRECT = 0, 1

# every symbol include/fvv_b200.h declares (tests/test_abi.py checks both ways)
EXPORTS = (
    "fvv_last_error", "fvv_build_info", "fvv_frame_bytes", "fvv_validate_params",
    "fvv_engine_workspace_size", "fvv_engine_create", "fvv_engine_destroy",
    "fvv_engine_max_pairs", "fvv_engine_set_tuning", "fvv_interpolate_pairs", "fvv_interp_diagnostics",
    "fvv_dense_views", "fvv_dense_views_scratch", "fvv_rig_views", "fvv_rig_views_scratch",
    "fvv_rig_views_mode", "fvv_downscale", "fvv_cluster_width",
    "fvv_assemble_cluster", "fvv_rig_cluster_bytes", "fvv_rig_clusters", "fvv_rig_clusters_shard",
    "fvv_profile_enable", "fvv_profile_read", "fvv_kernel_class_name",
    "fvv_interp_level_diagnostics", "fvv_interp_level_mask_scratch", "fvv_interp_level_mask", "fvv_conv2d_bf16", "fvv_vinet_workspace_size", "fvv_vinet_flow",
    "fvv_vinet_synth", "fvv_vinet_rig", "fvv_vinet_rig_clusters",
    "fvv_refine_image", "fvv_refine_inputs", "fvv_refine_flow_pool", "fvv_refine_warp_features",
    "fvv_nhwc_copy", "fvv_refine_output",
    "fvv_encode_set_tables", "fvv_encode_blocks", "fvv_encode_tokens", "fvv_deflate_scratch_bytes", "fvv_deflate",
    "fvv_ts_segment_bytes", "fvv_ts_mux_segment",
)


class FrameDesc(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32), ("format", ctypes.c_int32)]


class InterpParams(ctypes.Structure):
    _fields_ = [("block_size", ctypes.c_int32 * 3), ("search_radius", ctypes.c_int32 * 3),
                ("mask_epsilon", ctypes.c_double)]


class ConvDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "batch", "in_h", "in_w", "in_cpad", "out_h", "out_w", "out_cstride", "out_coff", "out_channels",
        "kernel", "stride", "pad", "transposed", "relu", "out_f32", "ntile")]


class LayoutErrorBase(Exception):
    """Mirrors fvv.cluster.LayoutError (cluster.py:22-23)."""


_lib = None


def lib_path() -> Path:
    return LIB


def load():
    """Load (building first if stale) the shared library and declare signatures."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB.exists():
        from ._build import build
        build()
    L = ctypes.CDLL(str(LIB))
    P, I, Z = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    PP = ctypes.POINTER(ctypes.c_void_p)
    pd, pp = ctypes.POINTER(FrameDesc), ctypes.POINTER(InterpParams)
    sig = {
        "fvv_last_error": (ctypes.c_char_p, []),
        "fvv_build_info": (ctypes.c_char_p, []),
        "fvv_frame_bytes": (Z, [pd]),
        "fvv_validate_params": (I, [pp]),
        "fvv_engine_workspace_size": (Z, [pd, pp, I]),
        "fvv_engine_create": (I, [pd, pp, I, P, Z, ctypes.POINTER(P)]),
        "fvv_engine_destroy": (None, [P]),
        "fvv_engine_max_pairs": (I, [P]),
        "fvv_engine_set_tuning": (I, [P, I, I]),
        "fvv_interpolate_pairs": (I, [P, PP, PP, PP, I, P]),
        "fvv_interp_diagnostics": (I, [P, I, P, P, P, P]),
        "fvv_interp_level_diagnostics": (I, [P, I, I, P, P, P, P, P]),
        "fvv_interp_level_mask_scratch": (Z, [P, I]),
        "fvv_interp_level_mask": (I, [P, I, I, P, Z, P, P, P]),
        "fvv_dense_views": (I, [P, P, P, I, I, P, P, Z, P]),
        "fvv_dense_views_scratch": (Z, [P, I]),
        "fvv_rig_views_scratch": (Z, [P, I, I]),
        "fvv_rig_views_mode": (I, [P, P, I, I, I, P, P, Z, P]),
        "fvv_rig_views": (I, [P, P, I, I, P, P]),
        "fvv_downscale": (I, [pd, P, I, I, P, P]),
        "fvv_cluster_width": (I, [I, I]),
        "fvv_assemble_cluster": (I, [pd, P, PP, I, P, P]),
        "fvv_rig_cluster_bytes": (Z, [pd, I, I, I, I]),
        "fvv_rig_clusters": (I, [pd, I, I, I, P, P, P]),
        "fvv_rig_clusters_shard": (I, [pd, I, I, I, I, I, P, I, I, P, I, I, P, P]),
        "fvv_profile_enable": (I, [P, I]),
        "fvv_profile_read": (I, [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I), I]),
        "fvv_kernel_class_name": (ctypes.c_char_p, [I]),
        "fvv_conv2d_bf16": (I, [ctypes.POINTER(ConvDesc), P, P, P, P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(rc: int) -> None:
    """Map a C status to the reference's exception classes."""
    if rc == FVV_OK:
        return
    msg = load().fvv_last_error().decode()
    if rc == FVV_EINVAL:
        raise ValueError(msg)
    if rc == FVV_ELAYOUT:
        from .cluster import LayoutError
        raise LayoutError(msg)
    if rc == FVV_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"CUDA failure: {msg}")


def require_cuda():
    """The product path needs a CUDA device and the in-tree library: fail loudly."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2112_10603_b200 needs a CUDA device (B200); there is no CPU path")
    return load()


def desc(width: int, height: int, fmt: int) -> FrameDesc:
    return FrameDesc(int(width), int(height), int(fmt))


def params(cfg) -> InterpParams:
    p = InterpParams()
    for i in range(3):
        p.block_size[i] = int(cfg.block_size[i])
        p.search_radius[i] = int(cfg.search_radius[i])
    p.mask_epsilon = float(cfg.mask_epsilon)
    return p


def ptr_array(ptrs):
    arr = (ctypes.c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = int(p)
    return arr

"""CPU-side checks of the C ABI: the library loads, exports exactly what
include/fvv_b200.h declares, and its host-only entry points behave like the
reference's validation (no GPU needed)."""
import ctypes
import os
import re

import pytest

from paper_2112_10603_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "fvv_b200.h")).read()
    return set(re.findall(r"\b(fvv_[a-z_0-9]+)\s*\(", src))


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    declared = header_symbols()
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name


def test_frame_bytes_and_geometry():
    L = _lib.load()
    for w, h, fmt, n in [(1920, 1080, 1, 1920 * 1080 * 3 // 2), (448, 256, 2, 448 * 256 * 3),
                         (64, 48, 0, 64 * 48), (5, 3, 1, 15 + 2 * 3 * 2)]:
        d = _lib.desc(w, h, fmt)
        assert L.fvv_frame_bytes(ctypes.byref(d)) == n
    assert L.fvv_cluster_width(1920, 32) == 1920 + 8 * 480
    d = _lib.desc(1920, 1080, 1)
    # cfg3: 4 cameras, 4 stages, vps 16 -> tiles [17, 33, 33, 17]
    widths = [L.fvv_rig_cluster_bytes(ctypes.byref(d), 4, 4, 16, c) for c in range(4)]
    assert widths[0] == widths[3] and widths[1] == widths[2]
    assert widths[1] == 5760 * 1080 * 3 // 2


def test_validate_params_matches_reference_errors():
    from paper_2112_10603_b200.interp import InterpConfig
    L = _lib.load()
    assert L.fvv_validate_params(ctypes.byref(_lib.params(InterpConfig()))) == 0
    bad = _lib.InterpParams()
    for i in range(3):
        bad.block_size[i] = 8
        bad.search_radius[i] = 0
    bad.mask_epsilon = 1e-3
    assert L.fvv_validate_params(ctypes.byref(bad)) == _lib.FVV_EINVAL
    assert b"degenerate" in L.fvv_last_error()
    with pytest.raises(ValueError):
        InterpConfig(block_size=(8, 1, 8))
    # every block size / radius the reference accepts is valid (non power-of-two blocks and
    # max_span > 120 run the literal path); only a non-positive epsilon is outside the path
    odd = _lib.params(InterpConfig(block_size=(8, 6, 8)))
    assert L.fvv_validate_params(ctypes.byref(odd)) == 0
    wide = _lib.params(InterpConfig(search_radius=(30, 4, 2)))
    assert L.fvv_validate_params(ctypes.byref(wide)) == 0
    d = _lib.desc(64, 48, 1)
    assert L.fvv_engine_workspace_size(ctypes.byref(d), ctypes.byref(odd), 4) > 0
    zero = _lib.params(InterpConfig(mask_epsilon=0.0))
    assert L.fvv_validate_params(ctypes.byref(zero)) == _lib.FVV_EUNSUPPORTED


def test_workspace_size_and_interp_dims():
    from paper_2112_10603_b200.interp import InterpConfig
    L = _lib.load()
    p = _lib.params(InterpConfig())
    d = _lib.desc(1920, 1080, 1)
    s1 = L.fvv_engine_workspace_size(ctypes.byref(d), ctypes.byref(p), 1)
    s4 = L.fvv_engine_workspace_size(ctypes.byref(d), ctypes.byref(p), 4)
    assert s1 > 0 and s4 > 3 * s1
    bad = _lib.desc(1922, 1080, 1)  # not divisible by 4
    assert L.fvv_engine_workspace_size(ctypes.byref(bad), ctypes.byref(p), 1) == 0


def test_product_path_refuses_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2112_10603_b200 as fv
    import numpy as np
    img = fv.gray(np.zeros((8, 8), np.uint8))
    with pytest.raises(RuntimeError, match="CUDA"):
        fv.interpolate(img, img)


def test_vinet_entry_points_validate_on_the_host():
    """The CNN-path entry points reject bad arguments before touching the device."""
    L = _lib.load()
    from paper_2112_10603_b200 import vinet  # declares the VINet signatures
    vinet._sig(L)
    d = _lib.desc(1920, 1080, 1)
    s1 = L.fvv_vinet_workspace_size(ctypes.byref(d), 1)
    s2 = L.fvv_vinet_workspace_size(ctypes.byref(d), 2)
    assert s1 > 0 and s2 > 1.9 * s1
    small = _lib.desc(32, 32, 1)  # below the 64-px minimum of the 64-aligned canvas
    assert L.fvv_vinet_workspace_size(ctypes.byref(small), 1) == 0
    conv = _lib.ConvDesc(1, 8, 8, 24, 8, 8, 128, 0, 128, 3, 1, 1, 0, 1, 0, 128)  # in_cpad 24: unsupported
    assert L.fvv_conv2d_bf16(ctypes.byref(conv), 1, 1, 1, 1, None) == _lib.FVV_EUNSUPPORTED
    conv = _lib.ConvDesc(1, 8, 8, 64, 8, 8, 128, 0, 128, 3, 1, 1, 0, 1, 0, 48)   # ntile 48: invalid
    assert L.fvv_conv2d_bf16(ctypes.byref(conv), 1, 1, 1, 1, None) == _lib.FVV_EINVAL
    conv = _lib.ConvDesc(1, 8, 8, 64, 5, 5, 128, 0, 128, 3, 1, 1, 0, 1, 0, 128)  # wrong output size
    assert L.fvv_conv2d_bf16(ctypes.byref(conv), 1, 1, 1, 1, None) == _lib.FVV_EINVAL
    conv = _lib.ConvDesc(1, 8, 8, 64, 16, 16, 128, 0, 128, 3, 2, 1, 1, 1, 0, 128)  # transposed must be k4 s2 p1
    assert L.fvv_conv2d_bf16(ctypes.byref(conv), 1, 1, 1, 1, None) == _lib.FVV_EUNSUPPORTED


def test_vinet_rig_clusters_validates_on_the_host():
    """fvv_vinet_rig_clusters applies fvv_rig_clusters' layout rules (cluster.py:148-183,
    server/pipeline.py:273-292) before any device work; pointers are never dereferenced."""
    L = _lib.load()
    from paper_2112_10603_b200 import vinet
    vinet._sig(L)
    w = vinet._Weights()
    fake = 16  # a non-null address: validation fails before anything is read

    def call(d, ncams=8, stages=4, vps=16):
        return L.fvv_vinet_rig_clusters(ctypes.byref(d), ctypes.byref(w), fake, ncams, stages, vps, fake, fake,
                                        fake, 1 << 30, None)
    rgb = _lib.desc(1920, 1080, 2)
    assert call(rgb) == _lib.FVV_ELAYOUT                      # cluster frames are gray or 4:2:0
    d = _lib.desc(1920, 1080, 1)
    assert call(d, vps=17) == _lib.FVV_ELAYOUT                # more than 2^stages views per side
    assert call(d, vps=0) == _lib.FVV_ELAYOUT
    assert call(d, ncams=1) == _lib.FVV_EINVAL
    assert call(d, stages=7) == _lib.FVV_EINVAL
    odd = _lib.desc(1916, 1080, 1)                            # VINet takes W % 4 == 0, clusters need W % 8
    assert call(odd) == _lib.FVV_ELAYOUT
    assert call(d, ncams=600, stages=4) == _lib.FVV_EINVAL     # > 8192 global views for the tile table
    assert "8192" in L.fvv_last_error().decode()


def test_deflate_sizes_and_offset_validation():
    """fvv_deflate_scratch_bytes is host-only: output capacity is zlib's
    compressBound summed over the streams; offsets must ascend."""
    from paper_2112_10603_b200.deflate import _sig
    L = _lib.load()
    _sig(L)
    offs = [0, 0, 1, 100, 70000]
    arr = (ctypes.c_longlong * len(offs))(*offs)
    sb, cap = ctypes.c_size_t(), ctypes.c_size_t()
    assert L.fvv_deflate_scratch_bytes(arr, len(offs) - 1, ctypes.byref(sb), ctypes.byref(cap)) == 0
    bound = lambda n: n + (n >> 12) + (n >> 14) + (n >> 25) + 13  # noqa: E731  zlib compressBound
    assert cap.value >= sum(bound(b - a) for a, b in zip(offs, offs[1:]))
    assert sb.value > 10 * 70000  # links, records, symbols per position
    bad = (ctypes.c_longlong * 3)(0, 10, 5)
    assert L.fvv_deflate_scratch_bytes(bad, 2, ctypes.byref(sb), ctypes.byref(cap)) != 0
    assert b"ascend" in L.fvv_last_error()

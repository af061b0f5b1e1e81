"""DEFLATE of many byte streams on the B200, byte-identical to
zlib.compress(stream, 6)[2:-4] (the raw data codec.py:148 keeps for each
plane's token stream).  The algorithm (zlib 1.3's level-6 deflate_slow and
trees.c, restated as parallel steps) is in csrc/zdeflate_core.h, the kernels
in csrc/deflate_kernels.cu.

    out, offs = deflate_streams(tokens_u8_cuda, [0, n0, n0 + n1, ...])
    raw = deflate_bytes(tokens_u8_cuda, offsets)   # list of bytes per stream
"""
from __future__ import annotations

import ctypes
import threading

from . import _lib

_tls = threading.local()


def _sig(L):
    P, I, LLP, SZP = ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(ctypes.c_size_t)
    L.fvv_deflate_scratch_bytes.restype = I
    L.fvv_deflate_scratch_bytes.argtypes = [LLP, I, SZP, SZP]
    L.fvv_deflate.restype = I
    L.fvv_deflate.argtypes = [P, LLP, I, P, P, P, ctypes.c_size_t, P]


def _buffer(name: str, nbytes: int, device):
    """Grow-only per-thread device buffer (a stream-ordered call per thread)."""
    import torch
    key = (name, str(device))
    cache = getattr(_tls, "bufs", None)
    if cache is None:
        cache = _tls.bufs = {}
    t = cache.get(key)
    if t is None or t.numel() < nbytes:
        t = cache[key] = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
    return t


def deflate_streams(data, offsets, stream=None):
    """data: uint8 CUDA tensor; offsets: host ints (nstreams + 1, ascending).
    Returns (out, out_offsets): uint8 CUDA buffer with the compressed streams
    back to back and their int64 CUDA offsets (nstreams + 1).  Stream-ordered
    on `stream` (default: the current stream)."""
    import torch
    L = _lib.require_cuda()
    _sig(L)
    if data.dtype != torch.uint8 or not data.is_cuda:
        raise TypeError("data must be a uint8 CUDA tensor")
    offs = [int(o) for o in offsets]
    if len(offs) < 2:
        raise ValueError("need at least one stream")
    if offs[-1] > data.numel():
        raise ValueError("offsets beyond the data")
    S = len(offs) - 1
    arr = (ctypes.c_longlong * (S + 1))(*offs)
    sb, cap = ctypes.c_size_t(), ctypes.c_size_t()
    _lib.check(L.fvv_deflate_scratch_bytes(arr, S, ctypes.byref(sb), ctypes.byref(cap)))
    scratch = _buffer("scratch", sb.value, data.device)
    out = torch.empty(cap.value, dtype=torch.uint8, device=data.device)
    out_off = torch.empty(S + 1, dtype=torch.int64, device=data.device)
    st = stream if stream is not None else torch.cuda.current_stream(data.device)
    _lib.check(L.fvv_deflate(ctypes.c_void_p(data.data_ptr()), arr, S, ctypes.c_void_p(out.data_ptr()),
                             ctypes.c_void_p(out_off.data_ptr()), ctypes.c_void_p(scratch.data_ptr()),
                             ctypes.c_size_t(scratch.numel()), ctypes.c_void_p(st.cuda_stream)))
    return out, out_off


def deflate_bytes(data, offsets) -> list:
    """deflate_streams, copied back: one bytes object per stream."""
    out, out_off = deflate_streams(data, offsets)
    offs = out_off.cpu().numpy()
    raw = out[:int(offs[-1])].cpu().numpy().tobytes()
    return [raw[offs[i]:offs[i + 1]] for i in range(len(offs) - 1)]

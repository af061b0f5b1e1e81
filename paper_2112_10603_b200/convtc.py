"""Convolution layers on the tcgen05 tensor cores (C ABI `fvv_conv2d_bf16`).

Activations are NHWC bf16 with the channel count padded (16, 32 or a multiple
of 64; padding channels zero); weights are packed once into the K-major GEMM
layouts the kernel's TMA maps read (include/fvv_b200.h).  There is no CPU or
torch fallback: these wrappers fail loudly without the CUDA library.
"""
from __future__ import annotations

import ctypes

from . import _lib


def cpad_of(c: int) -> int:
    """Padded channel count of an NHWC activation feeding the tensor-core conv."""
    if c <= 16:
        return 16
    if c <= 32:
        return 32
    return (c + 63) // 64 * 64


def ntile_of(n: int) -> int:
    for t in (16, 32, 64, 128, 256):
        if n <= t:
            return t
    return 256


def pack_conv(weight, cpad: int, ntile: int):
    """torch Conv2d weight [Cout][Cin][k][k] -> bf16 [npad][k*k*cpad], K = (ky*k+kx)*cpad + c."""
    import torch
    cout, cin, k, _ = weight.shape
    npad = (cout + ntile - 1) // ntile * ntile
    w = torch.zeros((npad, k * k, cpad), dtype=torch.float32, device=weight.device)
    w[:cout, :, :cin] = weight.detach().float().permute(0, 2, 3, 1).reshape(cout, k * k, cin)
    return w.reshape(npad, k * k * cpad).to(torch.bfloat16).contiguous()


# ConvTranspose2d(k4, s2, p1) as 4 phase convolutions: output parity -> kernel rows/cols of its 2 taps
_PHASE_K = {0: (1, 3), 1: (0, 2)}


def pack_convT(weight, cpad: int, ntile: int):
    """torch ConvTranspose2d weight [Cin][Cout][4][4] -> bf16 [4][npad][4*cpad] (include/fvv_b200.h)."""
    import torch
    cin, cout, k, _ = weight.shape
    assert k == 4
    npad = (cout + ntile - 1) // ntile * ntile
    w = torch.zeros((4, npad, 4, cpad), dtype=torch.float32, device=weight.device)
    wf = weight.detach().float()
    for ph in range(4):
        a, b = ph >> 1, ph & 1
        for t in range(4):
            ky, kx = _PHASE_K[a][t >> 1], _PHASE_K[b][t & 1]
            w[ph, :cout, t, :cin] = wf[:, :, ky, kx].t()
    return w.reshape(4, npad, 4 * cpad).to(torch.bfloat16).contiguous()


def pack_convT_subpixel(weight, cpad: int, ntile: int = 32):
    """ConvTranspose2d(k4 s2 p1) [Cin][Cout][4][4] as ONE 3x3 stride-1 convolution with 4*Cout
    outputs (sub-pixel form): row n = phase*Cout + c, phase = (oy&1)*2 + (ox&1); tap (ty, tx) reads
    input offset (ty-1, tx-1).  -> bf16 [npad][9*cpad]."""
    import torch
    cin, cout, k, _ = weight.shape
    assert k == 4
    n = 4 * cout
    npad = (n + ntile - 1) // ntile * ntile
    w = torch.zeros((npad, 9, cpad), dtype=torch.float32, device=weight.device)
    wf = weight.detach().float()
    kof = {0: {0: 1, -1: 3}, 1: {1: 0, 0: 2}}  # parity -> input offset -> kernel index
    for ph in range(4):
        a, b = ph >> 1, ph & 1
        for t in range(9):
            dy, dx = t // 3 - 1, t % 3 - 1
            if dy in kof[a] and dx in kof[b]:
                w[ph * cout:(ph + 1) * cout, t, :cin] = wf[:, :, kof[a][dy], kof[b][dx]].t()
    return w.reshape(npad, 9 * cpad).to(torch.bfloat16).contiguous()


def conv2d(x, w_packed, bias, cout: int, kernel: int, stride: int, pad: int, *, transposed: bool = False,
           relu: bool = True, out=None, out_coff: int = 0, out_f32: bool = False, ntile: int | None = None,
           stream=None, subpixel: bool = False):
    """One conv layer.  x: NHWC bf16 [B][H][W][cpad] (cuda); returns NHWC out.
    subpixel (with transposed): the ConvTranspose2d runs as one 3x3 GEMM with 4*cout
    outputs (weights from pack_convT_subpixel, bias repeated 4 times)."""
    import torch
    L = _lib.require_cuda()
    B, H, W, cpad = x.shape
    if transposed:
        Ho, Wo = 2 * H, 2 * W
    else:
        Ho, Wo = (H + 2 * pad - kernel) // stride + 1, (W + 2 * pad - kernel) // stride + 1
    nt = ntile or ntile_of(4 * cout if subpixel else cout)
    if out is None:
        out = torch.empty((B, Ho, Wo, cout if out_f32 else cpad_of(cout)),
                          dtype=torch.float32 if out_f32 else torch.bfloat16, device=x.device)
        if not out_f32 and out.shape[-1] != cout:
            out.zero_()
    d = _lib.ConvDesc(B, H, W, cpad, Ho, Wo, out.shape[-1], out_coff, cout, kernel, stride, pad,
                      (2 if subpixel else 1) if transposed else 0, int(relu), int(out_f32), nt)
    st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    _lib.check(L.fvv_conv2d_bf16(ctypes.byref(d), ctypes.c_void_p(x.data_ptr()),
                                 ctypes.c_void_p(w_packed.data_ptr()), ctypes.c_void_p(bias.data_ptr()),
                                 ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st)))
    return out

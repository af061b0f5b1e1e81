"""VINet on B200: the CNN flow / fusion estimator of the paper's hot path
 with the direct-t synthesis of N views per pair.

    net = VINet(1920, 1080, PixelFormat.YUV420, seed=0)
    flows = net.flows(left, right)           # (pairs, 5, H, W) f32: F_m->l, F_m->r, mask logit
    views = net.synth(left, right, flows, 15) # (pairs, 15, frame_bytes) u8, t = j/16

Every convolution runs on the tcgen05 tensor cores (csrc/conv_tc.cu, bf16
operands, fp32 TMEM accumulation); pyramid, block inputs, residual updates
and synthesis are CUDA kernels (csrc/vinet_kernels.cu).  Parity: against the
fp32 torch oracle oracle/vinet_ref.py (tests/test_gpu_vinet.py).  No CPU
fallback.
"""
from __future__ import annotations

import ctypes

from . import _lib
from .convtc import cpad_of, pack_conv, pack_convT, pack_convT_subpixel
from .frame import PixelFormat, frame_nbytes
from .vinet_params import BLOCK_IN, LAYERS, make_params

NTILE = {"c0": 128, "c1": 256, "u0": 128, "u1": 16}


class _Weights(ctypes.Structure):
    _fields_ = [("w", (ctypes.c_void_p * 10) * 3), ("b", (ctypes.c_void_p * 10) * 3)]


def _sig(L):
    P, I, Z = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    pd = ctypes.POINTER(_lib.FrameDesc)
    PP = ctypes.POINTER(ctypes.c_void_p)
    L.fvv_vinet_workspace_size.restype = Z
    L.fvv_vinet_workspace_size.argtypes = [pd, I]
    L.fvv_vinet_flow.restype = I
    L.fvv_vinet_flow.argtypes = [pd, ctypes.POINTER(_Weights), PP, PP, I, P, P, Z, P]
    L.fvv_vinet_synth.restype = I
    L.fvv_vinet_synth.argtypes = [pd, PP, PP, P, I, I, P, P]
    L.fvv_vinet_rig.restype = I
    L.fvv_vinet_rig.argtypes = [pd, ctypes.POINTER(_Weights), P, I, I, P, P, Z, P]
    L.fvv_vinet_rig_clusters.restype = I
    L.fvv_vinet_rig_clusters.argtypes = [pd, ctypes.POINTER(_Weights), P, I, I, I, P, P, P, Z, P]


class VINet:
    """Device-resident VINet for one frame size / format (reentrant per stream)."""

    def __init__(self, width: int, height: int, fmt, params=None, seed: int = 0, max_pairs: int = 8,
                 device=None):
        import torch
        self._L = _lib.require_cuda()
        _sig(self._L)
        self.width, self.height, self.format = int(width), int(height), PixelFormat(int(fmt))
        self.device = torch.device(device or "cuda")
        self._desc = _lib.desc(self.width, self.height, int(self.format))
        self.frame_bytes = frame_nbytes(self.width, self.height, self.format)
        params = params if params is not None else make_params(seed)
        self._keep = []
        self._w = _Weights()
        for i in range(3):
            for k, (name, kind, cin, cout) in enumerate(LAYERS):
                w, b = params[i][k]
                cin = BLOCK_IN[i] if cin is None else cin
                nt = NTILE.get(name, 256)
                wd = w.to(self.device)
                if name == "u1":  # the head: one sub-pixel 3x3 GEMM for all 4 output phases
                    packed = pack_convT_subpixel(wd, cpad_of(cin), 32)
                    bias = b.to(self.device, torch.float32).repeat(4).contiguous()
                elif kind == "convT":
                    packed = pack_convT(wd, cpad_of(cin), nt)
                    bias = b.to(self.device, torch.float32).contiguous()
                else:
                    packed = pack_conv(wd, cpad_of(cin), nt)
                    bias = b.to(self.device, torch.float32).contiguous()
                self._keep += [packed, bias]
                self._w.w[i][k] = packed.data_ptr()
                self._w.b[i][k] = bias.data_ptr()
        self.max_pairs = int(max_pairs)
        nbytes = self._L.fvv_vinet_workspace_size(ctypes.byref(self._desc), self.max_pairs)
        if nbytes == 0:
            raise ValueError("VINet needs width, height >= 64 and multiples of 4")
        self._ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)

    def _stream(self):
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _ptrs(self, frames):
        if frames.dim() != 2 or frames.shape[1] != self.frame_bytes or frames.dtype.itemsize != 1:
            raise ValueError(f"frames must be (pairs, {self.frame_bytes}) uint8")
        return _lib.ptr_array([frames[i].data_ptr() for i in range(frames.shape[0])])

    def flows(self, left, right, out=None):
        import torch
        n = left.shape[0]
        if right.shape != left.shape:
            raise ValueError("left and right batches differ")
        if out is None:
            out = torch.empty((n, 5, self.height, self.width), dtype=torch.float32, device=self.device)
        _lib.check(self._L.fvv_vinet_flow(ctypes.byref(self._desc), ctypes.byref(self._w), self._ptrs(left),
                                          self._ptrs(right), n, ctypes.c_void_p(out.data_ptr()),
                                          ctypes.c_void_p(self._ws.data_ptr()), self._ws.numel(), self._stream()))
        return out

    def synth(self, left, right, flows, nviews: int, out=None):
        import torch
        n = left.shape[0]
        if out is None:
            out = torch.empty((n, nviews, self.frame_bytes), dtype=torch.uint8, device=self.device)
        _lib.check(self._L.fvv_vinet_synth(ctypes.byref(self._desc), self._ptrs(left), self._ptrs(right),
                                           ctypes.c_void_p(flows.data_ptr()), n, int(nviews),
                                           ctypes.c_void_p(out.data_ptr()), self._stream()))
        return out

    def dense_views(self, left, right, nviews: int):
        """flows + synth: the nviews direct-t views of every pair."""
        return self.synth(left, right, self.flows(left, right), nviews)

    def rig(self, cams, stages: int, views=None):
        """Rig frame: cams (C, frame_bytes) -> global views ((C-1)*2^stages + 1, frame_bytes) in the
        fvv_rig_views layout (anchors + direct-t views per gap), ready for cluster.rig_clusters."""
        import torch
        C = cams.shape[0]
        if cams.shape[1] != self.frame_bytes:
            raise ValueError(f"cams must be (C, {self.frame_bytes}) uint8")
        if views is None:
            views = torch.empty((((C - 1) << stages) + 1, self.frame_bytes), dtype=torch.uint8, device=self.device)
        _lib.check(self._L.fvv_vinet_rig(ctypes.byref(self._desc), ctypes.byref(self._w),
                                         ctypes.c_void_p(cams.data_ptr()), C, int(stages),
                                         ctypes.c_void_p(views.data_ptr()), ctypes.c_void_p(self._ws.data_ptr()),
                                         self._ws.numel(), self._stream()))
        return views


    def rig_clusters(self, cams, stages: int, views_per_side: int = 16, views=None, out=None):
        """rig + cluster.rig_clusters in one call with the tiling fused into the synthesis
        (fvv_vinet_rig_clusters).  Returns (views, clusters, sizes); both buffers are
        byte-identical to rig() followed by cluster.rig_clusters()."""
        import torch
        from .cluster import rig_cluster_sizes
        C = cams.shape[0]
        if cams.shape[1] != self.frame_bytes:
            raise ValueError(f"cams must be (C, {self.frame_bytes}) uint8")
        sizes = rig_cluster_sizes(self.width, self.height, self.format, C, stages, views_per_side)
        if views is None:
            views = torch.empty((((C - 1) << stages) + 1, self.frame_bytes), dtype=torch.uint8, device=self.device)
        if out is None:
            out = torch.empty(sum(sizes), dtype=torch.uint8, device=self.device)
        _lib.check(self._L.fvv_vinet_rig_clusters(
            ctypes.byref(self._desc), ctypes.byref(self._w), ctypes.c_void_p(cams.data_ptr()), C, int(stages),
            int(views_per_side), ctypes.c_void_p(views.data_ptr()), ctypes.c_void_p(out.data_ptr()),
            ctypes.c_void_p(self._ws.data_ptr()), self._ws.numel(), self._stream()))
        return views, out, sizes

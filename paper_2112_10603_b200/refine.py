"""RefineNet + ContextNet on B200: the paper's refinement stage after the
VIBlocks ("Refinement Network", layer table PAPER.md:340-365;
architecture and seeded weights in vinet_params.py).

    net = VINet(W, H, fmt)
    ref = RefineNet(W, H, fmt)
    state = net.flows(left, right)                 # (pairs, 5, H, W)
    views = ref.views(left, right, state, 15)      # (pairs, 15, frame_bytes), refined direct-t views

ContextNet extracts 4 feature levels of each source image once per pair;
for every view t they are warped with the view's flow pyramid straight into
the U-Net's concatenation buffers (fvv_refine_warp_features), and the U-Net
(8 encoder convs, 4 transposed convs, 3-channel sigmoid head) predicts the
residual of the blended view.  All 21 convolutions run on the tcgen05 kernel
(fvv_conv2d_bf16, bf16 operands, fp32 accumulation); the glue kernels are
csrc/refine_kernels.cu.  Parity: the fp32 torch oracle oracle/vinet_ref.py
refine_view (tests/test_gpu_refine.py, >= 50 dB).

`hook()` returns a callable for the reference's one plugin seam,
InterpConfig.refine (interp.py:30, 144-145): it refines the interpolated
midpoint from the interpolation's own diagnostics (mid flows and mask).
"""
from __future__ import annotations

import ctypes

from . import _lib
from .convtc import conv2d, cpad_of, ntile_of, pack_conv, pack_convT, pack_convT_subpixel
from .frame import PixelFormat, frame_nbytes
from .vinet_params import CONTEXT_CH, CONTEXT_LAYERS, REFINE_LAYERS, make_refine_params


def _sig(L):
    P, I, LL = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong
    pd = ctypes.POINTER(_lib.FrameDesc)
    PP = ctypes.POINTER(ctypes.c_void_p)
    L.fvv_refine_image.restype = I
    L.fvv_refine_image.argtypes = [pd, PP, I, P, P]
    L.fvv_refine_inputs.restype = I
    L.fvv_refine_inputs.argtypes = [pd, PP, PP, PP, ctypes.POINTER(ctypes.c_float), I, P, P, P, P]
    L.fvv_refine_flow_pool.restype = I
    L.fvv_refine_flow_pool.argtypes = [P, P, I, I, I, P]
    L.fvv_refine_warp_features.restype = I
    L.fvv_refine_warp_features.argtypes = [P, I, I, I, I, P, I, I, I, P, I, I, I, P]
    L.fvv_nhwc_copy.restype = I
    L.fvv_nhwc_copy.argtypes = [P, I, I, P, I, I, LL, P]
    L.fvv_refine_output.restype = I
    L.fvv_refine_output.argtypes = [pd, PP, I, P, I, P, P]


SUBPIXEL_MAX_COUT = 32  # decoder layers up to this width run as sub-pixel 3x3 GEMMs (u2, u3)


class RefineNet:
    """Device-resident RefineNet + ContextNet for one frame size / format."""

    def __init__(self, width: int, height: int, fmt, params=None, seed: int = 1, max_views: int = 8, device=None):
        import torch
        self._L = _lib.require_cuda()
        _sig(self._L)
        self.width, self.height, self.format = int(width), int(height), PixelFormat(int(fmt))
        if self.width < 64 or self.height < 64 or self.width % 4 or self.height % 4:
            raise ValueError("RefineNet frames need width, height >= 64 and multiples of 4")
        self.device = torch.device(device or "cuda")
        self.Wp, self.Hp = (self.width + 63) // 64 * 64, (self.height + 63) // 64 * 64
        self.frame_bytes = frame_nbytes(self.width, self.height, self.format)
        self._desc = _lib.desc(self.width, self.height, int(self.format))
        self.max_views = int(max_views)
        params = params if params is not None else make_refine_params(seed)
        self.ctx = []
        for (name, stride, cin, cout), (w, b) in zip(CONTEXT_LAYERS, params["context"]):
            nt = ntile_of(cout)
            self.ctx.append((pack_conv(w.to(self.device), cpad_of(cin), nt), b.to(self.device).contiguous(),
                             cout, stride, nt))
        self.unet = []
        for (name, kind, cin, cout), (w, b) in zip(REFINE_LAYERS, params["unet"]):
            wd = w.to(self.device)
            if kind == "convT" and cout <= SUBPIXEL_MAX_COUT:
                # narrow decoder layers: one 3x3 sub-pixel GEMM (input read once for all 4 phases)
                nt = ntile_of(4 * cout)
                packed, bias, kind = pack_convT_subpixel(wd, cpad_of(cin), nt), b.to(self.device).repeat(4), "convT_sp"
            else:
                nt = ntile_of(cout)
                packed = pack_convT(wd, cpad_of(cin), nt) if kind == "convT" else pack_conv(wd, cpad_of(cin), nt)
                bias = b.to(self.device)
            self.unet.append((packed, bias.contiguous(), cout, kind, nt))
        self._bufs = None

    # -- buffers ------------------------------------------------------------
    def _alloc(self, B):
        import torch
        if self._bufs is not None and self._bufs["B"] >= B:
            return self._bufs
        dev, Hp, Wp = self.device, self.Hp, self.Wp
        bf = torch.bfloat16

        def act(n, k, c, zero=True):
            t = torch.empty((n, Hp >> k, Wp >> k, c), dtype=bf, device=dev)
            if zero:
                t.zero_()
            return t
        H, W = self.height, self.width
        self._bufs = {
            "B": B,
            "img": act(2, 0, 16),
            "ctx": [act(2, k + 1, CONTEXT_CH[k]) for k in range(4)],     # warped-from features, per level
            "ctmp": [act(2, k + 1, CONTEXT_CH[k]) for k in range(4)],
            "x0": act(B, 0, 32),
            "merged": torch.empty((B, 3, H, W), dtype=torch.float32, device=dev),
            "flow": [torch.empty((B, 4, Hp >> k, Wp >> k), dtype=torch.float32, device=dev) for k in range(5)],
            "t1": act(B, 1, 32), "cat1": act(B, 1, 64), "cu3": act(B, 1, 64),
            "t2": act(B, 2, 64), "cat2": act(B, 2, 128), "cu2": act(B, 2, 128),
            "t3": act(B, 3, 128), "cat3": act(B, 3, 256), "cu1": act(B, 3, 256),
            "t4": act(B, 4, 256), "cat4": act(B, 4, 512),
            "u3": act(B, 0, 16),
            "r": torch.zeros((B, Hp, Wp, 4), dtype=torch.float32, device=dev),
        }
        return self._bufs

    def _stream(self):
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    # -- stages ---------------------------------------------------------------
    def _context(self, left_ptr: int, right_ptr: int, bufs):
        """4 levels of ContextNet features of (left, right) -> bufs["ctx"][k] (2, Hp/2^(k+1), ...)."""
        L, st = self._L, self._stream()
        _lib.check(L.fvv_refine_image(ctypes.byref(self._desc), _lib.ptr_array([left_ptr, right_ptr]), 2,
                                      ctypes.c_void_p(bufs["img"].data_ptr()), st))
        x = bufs["img"]
        for k in range(4):
            w0, b0, c0, s0, n0 = self.ctx[2 * k]
            w1, b1, c1, s1, n1 = self.ctx[2 * k + 1]
            conv2d(x, w0, b0, c0, 3, s0, 1, out=bufs["ctmp"][k], ntile=n0)
            conv2d(bufs["ctmp"][k], w1, b1, c1, 3, s1, 1, out=bufs["ctx"][k], ntile=n1)
            x = bufs["ctx"][k]

    def _unet(self, B, bufs, out_ptrs):
        L, st = self._L, self._stream()
        u = self.unet
        fl = bufs["flow"]
        Hp, Wp = self.Hp, self.Wp
        for k in range(1, 5):
            _lib.check(L.fvv_refine_flow_pool(ctypes.c_void_p(fl[k - 1].data_ptr()), ctypes.c_void_p(fl[k].data_ptr()),
                                              Wp >> (k - 1), Hp >> (k - 1), B, st))

        def cv(i, x, out, coff=0, relu=True, out_f32=False):
            w, b, cout, kind, nt = u[i]
            if kind == "convT_sp":
                return conv2d(x[:B], w, b, cout, 4, 2, 1, transposed=True, subpixel=True, out=out[:B], out_coff=coff,
                              ntile=nt)
            if kind == "convT":
                return conv2d(x[:B], w, b, cout, 4, 2, 1, transposed=True, out=out[:B], out_coff=coff, ntile=nt)
            stride = 2 if kind == "conv_s2" else 1
            return conv2d(x[:B], w, b, cout, 3, stride, 1, relu=relu, out=out[:B], out_coff=coff, out_f32=out_f32,
                          ntile=nt)

        def warp_ctx(k, dst, coff):
            # level k+1 of the U-Net input: warped context features of left (flow 0:2) and right (2:4)
            c = CONTEXT_CH[k]
            feat = bufs["ctx"][k]
            h, w = Hp >> (k + 1), Wp >> (k + 1)
            for side, comp in ((0, 0), (1, 2)):
                _lib.check(L.fvv_refine_warp_features(
                    ctypes.c_void_p(feat.data_ptr()), feat.shape[-1], c, w, h, ctypes.c_void_p(fl[k + 1].data_ptr()),
                    comp, 0, side, ctypes.c_void_p(dst.data_ptr()), dst.shape[-1], coff + side * c, B, st))

        def skip(src, c, dst, coff, k):
            npix = B * (Hp >> k) * (Wp >> k)
            _lib.check(L.fvv_nhwc_copy(ctypes.c_void_p(src.data_ptr()), src.shape[-1], c,
                                       ctypes.c_void_p(dst.data_ptr()), dst.shape[-1], coff, npix, st))

        cv(0, bufs["x0"], bufs["t1"])
        cv(1, bufs["t1"], bufs["cat1"])                       # s0 -> cat1[0:32]
        warp_ctx(0, bufs["cat1"], 32)
        skip(bufs["cat1"], 32, bufs["cu3"], 32, 1)            # s0 -> up3 input [32:64]
        cv(2, bufs["cat1"], bufs["t2"])
        cv(3, bufs["t2"], bufs["cat2"])                       # s1
        warp_ctx(1, bufs["cat2"], 64)
        skip(bufs["cat2"], 64, bufs["cu2"], 64, 2)
        cv(4, bufs["cat2"], bufs["t3"])
        cv(5, bufs["t3"], bufs["cat3"])                       # s2
        warp_ctx(2, bufs["cat3"], 128)
        skip(bufs["cat3"], 128, bufs["cu1"], 128, 3)
        cv(6, bufs["cat3"], bufs["t4"])
        cv(7, bufs["t4"], bufs["cat4"])                       # s3
        warp_ctx(3, bufs["cat4"], 256)
        cv(8, bufs["cat4"], bufs["cu1"], 0)                   # up0 -> cu1[0:128]
        cv(9, bufs["cu1"], bufs["cu2"], 0)
        cv(10, bufs["cu2"], bufs["cu3"], 0)
        cv(11, bufs["cu3"], bufs["u3"], 0)
        cv(12, bufs["u3"], bufs["r"], 0, relu=False, out_f32=True)
        _lib.check(L.fvv_refine_output(ctypes.byref(self._desc), _lib.ptr_array(out_ptrs), B,
                                       ctypes.c_void_p(bufs["r"].data_ptr()), 4,
                                       ctypes.c_void_p(bufs["merged"].data_ptr()), st))

    # -- public -------------------------------------------------------------
    def views(self, left, right, state, nviews: int, out=None, ts=None):
        """Refined direct-t views t_j = j / (nviews + 1) (or `ts`) of every pair.

        left, right: (pairs, frame_bytes) uint8 CUDA; state: (pairs, 5, H, W) f32 VINet flows.
        Returns (pairs, nviews, frame_bytes) uint8."""
        import torch
        n = left.shape[0]
        if ts is None:
            ts = [(j + 1) / (nviews + 1) for j in range(nviews)]
        if len(ts) != nviews:
            raise ValueError("one view position per view")
        if out is None:
            out = torch.empty((n, nviews, self.frame_bytes), dtype=torch.uint8, device=self.device)
        bufs = self._alloc(min(self.max_views, nviews))
        L, st = self._L, self._stream()
        plane = 5 * self.width * self.height * 4
        for p in range(n):
            lp, rp = left[p].data_ptr(), right[p].data_ptr()
            self._context(lp, rp, bufs)
            sp = state.data_ptr() + p * plane
            for j0 in range(0, nviews, bufs["B"]):
                B = min(bufs["B"], nviews - j0)
                tarr = (ctypes.c_float * B)(*[float(t) for t in ts[j0:j0 + B]])
                _lib.check(L.fvv_refine_inputs(
                    ctypes.byref(self._desc), _lib.ptr_array([lp] * B), _lib.ptr_array([rp] * B),
                    _lib.ptr_array([sp] * B), tarr, B, ctypes.c_void_p(bufs["x0"].data_ptr()),
                    ctypes.c_void_p(bufs["merged"].data_ptr()), ctypes.c_void_p(bufs["flow"][0].data_ptr()), st))
                self._unet(B, bufs, [out[p, j0 + j].data_ptr() for j in range(B)])
        return out

    def hook(self):
        """A callable for InterpConfig.refine (interp.py:30, 144-145): refines the
        interpolated midpoint from its diagnostics -- flows F_m->l, F_m->r
        (flow_mid_left / flow_mid_right) and the blend mask M as the logit.
        Needs the diagnostics' source frames (`left`, `right`, filled by this
        package's interpolate())."""
        import numpy as np
        import torch
        from .frame import frame_from_packed, packed

        def refine(frame, diag):
            if getattr(diag, "left", None) is None:
                raise ValueError("RefineNet.hook needs InterpDiagnostics.left/right (this package's interpolate)")
            H, W = self.height, self.width
            m = np.clip(np.asarray(diag.mask, np.float64), 1e-12, 1.0 - 1e-12)
            st = np.empty((1, 5, H, W), np.float32)
            st[0, 0:2] = np.moveaxis(diag.flow_mid_left.vectors, -1, 0)
            st[0, 2:4] = np.moveaxis(diag.flow_mid_right.vectors, -1, 0)
            st[0, 4] = np.log(m / (1.0 - m))
            dev = self.device
            L = torch.from_numpy(packed(diag.left)).to(dev)[None]
            R = torch.from_numpy(packed(diag.right)).to(dev)[None]
            v = self.views(L, R, torch.from_numpy(st).to(dev), 1, ts=[0.5])
            return frame_from_packed(v[0, 0].cpu().numpy(), W, H, self.format, frame.timestamp)
        return refine

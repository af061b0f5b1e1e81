"""Midpoint view interpolation and recursive dense views on the B200.

Drop-in mirror of the reference's public interpolation API (fvv.interp,
interp.py:24-170): same entry points (`interpolate`, `dense_views`), same
`InterpConfig` fields and validation, same Frame layouts and error classes.
The compute is the CUDA path in libfvv_b200.so (csrc/interp_kernels.cu)
reached through the C ABI (include/fvv_b200.h); there is no CPU fallback.

Batched device entry points (`Interpolator.pairs`, `Interpolator.dense`) take
torch uint8 tensors of packed frames already resident in HBM.
"""
from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import _lib
from .frame import Frame, PixelFormat, frame_from_packed, packed

SCALE_FACTORS = (4, 2, 1)  # coarse to fine (interp.py:21)


@dataclass(frozen=True)
class InterpConfig:
    """interp.py:24-46 -- identical fields, defaults and validation."""

    block_size: tuple = (8, 8, 8)
    search_radius: tuple = (12, 4, 2)
    mask_epsilon: float = 1e-3
    border_band: int = 8
    refine: Callable | None = None

    def __post_init__(self) -> None:
        if len(self.block_size) != 3 or len(self.search_radius) != 3:
            raise ValueError("three scales need three block sizes and radii")
        if min(self.block_size) < 2 or min(self.search_radius) < 1:
            raise ValueError("degenerate block size or search radius")

    @property
    def max_span(self) -> int:
        r0, r1, r2 = self.search_radius
        return 4 * r0 + 2 * r1 + r2


@dataclass(frozen=True)
class FlowField:
    """flow.py:23-44: per-pixel (dx, dy) f32 offsets, (h, w, 2)."""

    width: int
    height: int
    vectors: np.ndarray

    def __post_init__(self) -> None:
        if self.vectors.shape != (self.height, self.width, 2):
            raise ValueError(f"flow vectors {self.vectors.shape} != {(self.height, self.width, 2)}")

    @staticmethod
    def zero(width: int, height: int) -> "FlowField":
        return FlowField(width, height, np.zeros((height, width, 2), dtype=np.float32))

    def scaled(self, factor: float) -> "FlowField":
        return FlowField(self.width, self.height, self.vectors * np.float32(factor))

    def max_magnitude(self) -> float:
        return float(np.max(np.abs(self.vectors))) if self.vectors.size else 0.0


@dataclass
class ScaleDiagnostics:  # interp.py:49-56
    flow_lr: FlowField
    flow_rl: FlowField
    match_error_lr: np.ndarray | None = None
    match_error_rl: np.ndarray | None = None
    mask: np.ndarray | None = None
    blend_luma: np.ndarray | None = None


@dataclass
class InterpDiagnostics:  # interp.py:59-64
    scales: list = field(default_factory=list)
    flow_mid_left: FlowField | None = None
    flow_mid_right: FlowField | None = None
    mask: np.ndarray | None = None
    # the two source frames (not in the reference's class): what a refine hook
    # such as refine.RefineNet.hook() needs besides the flows and the mask
    left: object = None
    right: object = None


# ---------------------------------------------------------------------------
# Device engine
# ---------------------------------------------------------------------------
class Interpolator:
    """One geometry + config + workspace (fvv_engine) on the current CUDA device.

    `max_pairs` bounds the interpolations run per recursion stage; a rig of
    C cameras at `stages` needs (C-1) * 2**(stages-1).
    """

    def __init__(self, width: int, height: int, fmt, config: InterpConfig | None = None,
                 max_pairs: int = 1, device=None):
        import torch
        L = _lib.require_cuda()
        self.config = config or InterpConfig()
        self.width, self.height, self.format = int(width), int(height), PixelFormat(int(fmt))
        self.max_pairs = int(max_pairs)
        self._desc = _lib.desc(width, height, int(fmt))
        self._params = _lib.params(self.config)
        _lib.check(L.fvv_validate_params(ctypes.byref(self._params)))
        if width % 4 or height % 4:
            raise ValueError("frame dimensions must be divisible by 4 for the 3-scale pyramid")
        self.frame_bytes = int(L.fvv_frame_bytes(ctypes.byref(self._desc)))
        ws = int(L.fvv_engine_workspace_size(ctypes.byref(self._desc), ctypes.byref(self._params),
                                             self.max_pairs))
        if ws == 0:
            _lib.check(-1)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._ws = torch.empty(ws, dtype=torch.uint8, device=self.device)
        h = ctypes.c_void_p()
        _lib.check(L.fvv_engine_create(ctypes.byref(self._desc), ctypes.byref(self._params),
                                       self.max_pairs, ctypes.c_void_p(self._ws.data_ptr()), ws,
                                       ctypes.byref(h)))
        self._h = h
        self._L = L

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                self._L.fvv_engine_destroy(self._h)
                self._h = None
        except Exception:  # noqa: BLE001
            pass

    def set_tuning(self, scan_coop_min: int | None = None, sadw_rb_min_ctas: int | None = None,
                   mask_cols2: int | None = None, pdl: int | None = None):
        """Launch-variant thresholds (fvv_engine_set_tuning); results are
        identical for every setting -- the tests use it to force each variant.
        None leaves a knob unchanged, -1 restores its default."""
        if scan_coop_min is not None:
            _lib.check(self._L.fvv_engine_set_tuning(self._h, _lib.FVV_TUNE_SCAN_COOP_MIN, int(scan_coop_min)))
        if sadw_rb_min_ctas is not None:
            _lib.check(self._L.fvv_engine_set_tuning(self._h, _lib.FVV_TUNE_SADW_RB_MIN_CTAS,
                                                     int(sadw_rb_min_ctas)))
        if mask_cols2 is not None:
            _lib.check(self._L.fvv_engine_set_tuning(self._h, _lib.FVV_TUNE_MASK_COLS2, int(mask_cols2)))
        if pdl is not None:
            _lib.check(self._L.fvv_engine_set_tuning(self._h, _lib.FVV_TUNE_PDL, int(pdl)))
        return self

    @property
    def workspace_bytes(self) -> int:
        return int(self._ws.numel())

    @staticmethod
    def _stream():
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def _check_frames(self, t, n=None):
        import torch
        if t.dtype != torch.uint8 or not t.is_cuda or not t.is_contiguous():
            raise ValueError("frames must be contiguous uint8 CUDA tensors of packed planes")
        if t.shape[-1] != self.frame_bytes:
            raise ValueError(f"packed frame is {t.shape[-1]} bytes, expected {self.frame_bytes}")

    def pairs(self, left, right, out=None):
        """interpolate() over a batch: left/right (n, frame_bytes) -> out (n, frame_bytes)."""
        import torch
        self._check_frames(left)
        self._check_frames(right)
        if left.shape != right.shape:
            raise ValueError("interpolation inputs must share size and format")
        n = left.shape[0]
        if out is None:
            out = torch.empty_like(left)
        fb = self.frame_bytes
        lp = _lib.ptr_array([left.data_ptr() + i * fb for i in range(n)])
        rp = _lib.ptr_array([right.data_ptr() + i * fb for i in range(n)])
        op = _lib.ptr_array([out.data_ptr() + i * fb for i in range(n)])
        _lib.check(self._L.fvv_interpolate_pairs(self._h, lp, rp, op, n, self._stream()))
        return out

    def diagnostics(self, pair: int = 0):
        """Final flows + mask of pair `pair` of the most recent `pairs` call (device tensors)."""
        import torch
        H, W = self.height, self.width
        flr = torch.empty((H, W, 2), dtype=torch.float32, device=self.device)
        frl = torch.empty_like(flr)
        m = torch.empty((H, W), dtype=torch.float64, device=self.device)
        _lib.check(self._L.fvv_interp_diagnostics(self._h, pair, ctypes.c_void_p(flr.data_ptr()),
                                                  ctypes.c_void_p(frl.data_ptr()),
                                                  ctypes.c_void_p(m.data_ptr()), self._stream()))
        return flr, frl, m

    def level_diagnostics(self, pair: int, level: int):
        """InterpDiagnostics.scales[level] of pair `pair` of the most recent `pairs` call:
        (flow_lr, flow_rl, match_error_lr, match_error_rl) device tensors."""
        import torch
        f = SCALE_FACTORS[level]
        h, w = self.height // f, self.width // f
        flr = torch.empty((h, w, 2), dtype=torch.float32, device=self.device)
        frl = torch.empty_like(flr)
        elr = torch.empty((h, w), dtype=torch.float64, device=self.device)
        erl = torch.empty_like(elr)
        _lib.check(self._L.fvv_interp_level_diagnostics(
            self._h, pair, level, ctypes.c_void_p(flr.data_ptr()), ctypes.c_void_p(frl.data_ptr()),
            ctypes.c_void_p(elr.data_ptr()), ctypes.c_void_p(erl.data_ptr()), self._stream()))
        return flr, frl, elr, erl

    def level_mask(self, pair: int, level: int):
        """ScaleDiagnostics.mask / .blend_luma of level 0 or 1 (interp.py:119-127) of pair
        `pair` of the most recent `pairs` call: (mask, blend_luma) f64 device tensors."""
        import torch
        f = SCALE_FACTORS[level]
        h, w = self.height // f, self.width // f
        nb = int(self._L.fvv_interp_level_mask_scratch(self._h, level))
        scratch = torch.empty(max(1, nb), dtype=torch.uint8, device=self.device)
        m = torch.empty((h, w), dtype=torch.float64, device=self.device)
        b = torch.empty_like(m)
        _lib.check(self._L.fvv_interp_level_mask(self._h, pair, level, ctypes.c_void_p(scratch.data_ptr()), nb,
                                                 ctypes.c_void_p(m.data_ptr()), ctypes.c_void_p(b.data_ptr()),
                                                 self._stream()))
        return m, b

    def dense(self, left, right, stages: int, views=None, mode: int = 0):
        """dense_views() on device: left/right (frame_bytes,) -> (2**stages - 1, frame_bytes).

        mode 0 (FVV_DENSE_RECURSIVE): the reference's recursive midpoints, bit-exact.
        mode 1 (FVV_DENSE_DIRECT): direct-t -- one interpolation (its output is the
        t = 1/2 view, bit-exact) and every other view from the same flows and mask."""
        import torch
        if stages < 1:
            raise ValueError("stages must be >= 1")
        if stages > 6:
            raise ValueError("stages > 6 refused: 2**n - 1 views grows too fast")
        self._check_frames(left)
        self._check_frames(right)
        if views is None:
            views = torch.empty(((1 << stages) - 1, self.frame_bytes), dtype=torch.uint8, device=left.device)
        nb = int(self._L.fvv_dense_views_scratch(self._h, int(mode)))
        scratch = torch.empty(max(1, nb), dtype=torch.uint8, device=left.device) if nb else None
        _lib.check(self._L.fvv_dense_views(self._h, ctypes.c_void_p(left.data_ptr()),
                                           ctypes.c_void_p(right.data_ptr()), stages, int(mode),
                                           ctypes.c_void_p(views.data_ptr()),
                                           ctypes.c_void_p(scratch.data_ptr() if scratch is not None else 0), nb,
                                           self._stream()))
        return views

    def rig(self, cams, stages: int, views=None, mode: int = 0):
        """server/pipeline.py:254-271: cams (C, fb) -> all global views (T, fb).
        mode 1: direct-t gaps (fvv_rig_views_mode, see dense())."""
        import torch
        self._check_frames(cams)
        C = cams.shape[0]
        total = (C - 1) * (1 << stages) + 1
        if views is None:
            views = torch.empty((total, self.frame_bytes), dtype=torch.uint8, device=cams.device)
        if mode == 0:
            _lib.check(self._L.fvv_rig_views(self._h, ctypes.c_void_p(cams.data_ptr()), C, stages,
                                             ctypes.c_void_p(views.data_ptr()), self._stream()))
            return views
        nb = int(self._L.fvv_rig_views_scratch(self._h, C, int(mode)))
        if getattr(self, "_rig_scratch", None) is None or self._rig_scratch.numel() < nb:
            self._rig_scratch = torch.empty(max(1, nb), dtype=torch.uint8, device=cams.device)
        _lib.check(self._L.fvv_rig_views_mode(self._h, ctypes.c_void_p(cams.data_ptr()), C, stages, int(mode),
                                              ctypes.c_void_p(views.data_ptr()),
                                              ctypes.c_void_p(self._rig_scratch.data_ptr()), nb, self._stream()))
        return views


class _ThreadState(threading.local):
    """Per-thread engines, stream and pinned staging buffers.

    The reference runs `dense_views` from a 2-worker ThreadPoolExecutor
    (server/pipeline.py:219-220, 264-268) and ctypes releases the GIL, so two
    calls can be in flight at once.  An engine's workspace holds the pair
    slots of ONE batch, so every thread gets its own engines and its own CUDA
    stream; nothing mutable is shared between threads.
    """

    def __init__(self):
        self.engines: dict = {}
        self.streams: dict = {}
        self.pinned: dict = {}


_tls = _ThreadState()


def _engine(width, height, fmt, cfg: InterpConfig, max_pairs: int) -> Interpolator:
    import torch
    _lib.require_cuda()
    key = (width, height, int(fmt), tuple(cfg.block_size), tuple(cfg.search_radius),
           float(cfg.mask_epsilon), max_pairs, torch.cuda.current_device())
    eng = _tls.engines.get(key)
    if eng is None:
        eng = Interpolator(width, height, fmt, cfg, max_pairs)
        _tls.engines[key] = eng
    return eng


def _thread_stream():
    """This thread's CUDA stream on the current device (created on first use)."""
    import torch
    dev = torch.cuda.current_device()
    s = _tls.streams.get(dev)
    if s is None:
        s = torch.cuda.Stream(device=dev)
        _tls.streams[dev] = s
    return s


def _pinned(slot: str, nbytes: int):
    """A reusable pinned host buffer of at least `nbytes` (per thread and slot).

    Safe to reuse across calls: every drop-in call synchronises its stream
    before it returns, so no copy from an earlier call is still in flight."""
    import torch
    buf = _tls.pinned.get(slot)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True)
        _tls.pinned[slot] = buf
    return buf[:nbytes]


def _to_device(frame, slot: str = "in0"):
    """Frame -> packed device tensor on the current stream (pinned staging, async H2D)."""
    import torch
    src = packed(frame)
    host = _pinned(slot, src.size)
    host.numpy()[:] = src
    return host.to("cuda", non_blocking=True)


def _to_host(dev, slot: str = "out") -> np.ndarray:
    """Device tensor -> numpy copy (pinned staging; synchronises this thread's stream)."""
    import torch
    flat = dev.contiguous().reshape(-1).view(torch.uint8)
    host = _pinned(slot, flat.numel())
    host.copy_(flat, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    np_dtype = torch.empty(0, dtype=dev.dtype).numpy().dtype
    return host.numpy().copy().view(np_dtype).reshape(tuple(dev.shape))


def _check_pair(left, right):
    if (left.width, left.height, int(left.format)) != (right.width, right.height, int(right.format)):
        raise ValueError("interpolation inputs must share size and format")
    if left.width % 4 or left.height % 4:
        raise ValueError("frame dimensions must be divisible by 4 for the 3-scale pyramid")


# ---------------------------------------------------------------------------
# Reference-facing API (interp.py:97-170)
# ---------------------------------------------------------------------------
def interpolate(left, right, config: InterpConfig | None = None, diagnostics: bool = False):
    """Synthesize the midpoint view between two same-size views (interp.py:97-148).

    Returns the interpolated Frame, or (Frame, InterpDiagnostics).  Bit-exact
    with the reference on the same inputs (tests/test_gpu_parity.py).
    """
    import torch
    cfg = config or InterpConfig()
    _check_pair(left, right)
    eng = _engine(left.width, left.height, left.format, cfg, 1)
    with torch.cuda.stream(_thread_stream()):
        dl = _to_device(left, "in0")[None]
        dr = _to_device(right, "in1")[None]
        out = eng.pairs(dl, dr)
        res = frame_from_packed(_to_host(out[0]), left.width, left.height, left.format,
                                left.timestamp)
        diag = InterpDiagnostics()
        if diagnostics or cfg.refine is not None:
            diag = _diagnostics(eng, coarse_masks=diagnostics)
            diag.left, diag.right = left, right
    if cfg.refine is not None:  # the reference's one plugin hook (interp.py:144-145)
        res = cfg.refine(res, diag)
    if diagnostics:
        return res, diag
    return res


def _diagnostics(eng: Interpolator, coarse_masks: bool = True) -> InterpDiagnostics:
    """InterpDiagnostics of pair 0 of the engine's most recent batch (interp.py:114-141).
    coarse_masks: the levels 0-1 mask / blend_luma, which the reference fills only
    when diagnostics were requested (interp.py:119)."""
    diag = InterpDiagnostics()
    # per-level flows and match errors (interp.py:114-128)
    for s in range(3):
        flr, frl, elr, erl = (_to_host(t, "diag") for t in eng.level_diagnostics(0, s))
        h, w = flr.shape[:2]
        sd = ScaleDiagnostics(FlowField(w, h, flr), FlowField(w, h, frl), elr, erl)
        if coarse_masks and s < 2:
            m, b = eng.level_mask(0, s)
            sd.mask, sd.blend_luma = _to_host(m, "diag"), _to_host(b, "diag")
        diag.scales.append(sd)
    _, _, m = eng.diagnostics(0)
    m = _to_host(m, "diag")
    f_lr, f_rl = diag.scales[-1].flow_lr, diag.scales[-1].flow_rl
    diag.flow_mid_left = f_lr.scaled(-0.5)
    diag.flow_mid_right = f_rl.scaled(-0.5)
    diag.mask = m
    diag.scales[-1].mask = m
    return diag


def dense_views(left, right, stages: int, config: InterpConfig | None = None, mode: str = "recursive") -> list:
    """2**stages - 1 views between left and right, left to right (interp.py:151-170).

    mode "recursive" (the reference's algorithm, bit-exact), or -- extensions
    the reference does not have -- "direct" (one SAD-flow interpolation per pair,
    its t = 1/2 view bit-exact, the other views direct-t from the same flows and
    mask) and "vinet" (the paper's CNN flows, direct-t synthesis; width and
    height >= 64)."""
    if stages < 1:
        raise ValueError("stages must be >= 1")
    if stages > 6:
        raise ValueError("stages > 6 refused: 2**n - 1 views grows too fast")
    if mode not in ("recursive", "direct", "vinet"):
        raise ValueError(f"unknown dense_views mode {mode!r}")
    cfg = config or InterpConfig()
    _check_pair(left, right)
    if cfg.refine is not None and mode == "recursive":
        # the hook runs on every intermediate view, so recursion goes pair by pair
        seq = [left, right]
        for _ in range(stages):
            nxt = []
            for a, b in zip(seq, seq[1:]):
                nxt.append(a)
                nxt.append(interpolate(a, b, cfg))
            nxt.append(seq[-1])
            seq = nxt
        return seq[1:-1]
    import torch
    with torch.cuda.stream(_thread_stream()):
        dl, dr = _to_device(left, "in0"), _to_device(right, "in1")
        if mode == "vinet":
            net = _vinet(left.width, left.height, left.format)
            views = net.dense_views(dl[None], dr[None], (1 << stages) - 1)[0]
        else:
            eng = _engine(left.width, left.height, left.format, cfg, 1 << (stages - 1) if mode == "recursive" else 1)
            views = eng.dense(dl, dr, stages, mode=0 if mode == "recursive" else 1)
        views = _to_host(views)
    return [frame_from_packed(v, left.width, left.height, left.format, left.timestamp) for v in views]


def _vinet(width, height, fmt):
    """This thread's VINet engine for a geometry (seeded weights, vinet_params)."""
    import torch
    key = ("vinet", width, height, int(fmt), torch.cuda.current_device())
    net = _tls.engines.get(key)
    if net is None:
        from .vinet import VINet
        net = VINet(width, height, fmt, max_pairs=1)
        _tls.engines[key] = net
    return net

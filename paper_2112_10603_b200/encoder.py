"""FVT1 tile encoding with the transform stage on the B200 (SURVEY.md sec.
8(f) row 2: the encoder hand-off after the tiling).

The reference encodes every tile of every cluster frame on the host
(server/pipeline.py:294-318 PipelineHandle._encode -> codec.TileEncoder,
codec.py:138-216, dct.py): per plane, 8x8 blocks -> DCT -> rint(c / step) ->
zigzag -> (run, level) tokens -> DEFLATE, closed loop on the reconstruction.
Here the blocks, transform, quantisation, reconstruction (kept on the device
for the next P record), zigzag and token stream run in
csrc/encode_kernels.cu over every (tile, plane) of a rig frame in one batch,
and so does DEFLATE: csrc/deflate_kernels.cu compresses every plane's token
stream at once, byte-identical to zlib.compress(tokens, 6) (deflate.py).  The
host only frames the records.  Records are byte-identical to
codec.TileEncoder's (tests/test_gpu_encoder.py against reference-generated
goldens).  deflate="host" runs zlib on a host thread pool instead (the
previous design, kept for timing comparisons).

    enc = RigEncoder(layouts, 1920, 1080, PixelFormat.YUV420, quality=75, gop=30)
    records = enc.encode(clusters, sizes)   # per cluster: [FrameRecord bytes per tile]
"""
from __future__ import annotations

import ctypes
import struct
import zlib
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import _lib
from .cluster import tile_rects
from .frame import PixelFormat, frame_nbytes, plane_shapes

# dct.py:9-17 _C as the reference computes it (numpy cos / sqrt), bit for bit:
# a matrix re-derived on another host's libm could differ in the last place
_DCT_HEX = (
    "0x1.6a09e667f3bcdp-2", "0x1.6a09e667f3bcdp-2", "0x1.6a09e667f3bcdp-2", "0x1.6a09e667f3bcdp-2", "0x1.6a09e667f3bcdp-2", "0x1.6a09e667f3bcdp-2", "0x1.6a09e667f3bcdp-2", "0x1.6a09e667f3bcdp-2",
    "0x1.f6297cff75cb0p-2", "0x1.a9b66290ea1a3p-2", "0x1.1c73b39ae68c9p-2", "0x1.8f8b83c69a60dp-4", "-0x1.8f8b83c69a608p-4", "-0x1.1c73b39ae68c6p-2", "-0x1.a9b66290ea1a4p-2", "-0x1.f6297cff75cb0p-2",
    "0x1.d906bcf328d46p-2", "0x1.87de2a6aea964p-3", "-0x1.87de2a6aea962p-3", "-0x1.d906bcf328d46p-2", "-0x1.d906bcf328d47p-2", "-0x1.87de2a6aea96dp-3", "0x1.87de2a6aea967p-3", "0x1.d906bcf328d44p-2",
    "0x1.a9b66290ea1a3p-2", "-0x1.8f8b83c69a608p-4", "-0x1.f6297cff75cb0p-2", "-0x1.1c73b39ae68c8p-2", "0x1.1c73b39ae68c5p-2", "0x1.f6297cff75cb0p-2", "0x1.8f8b83c69a61dp-4", "-0x1.a9b66290ea1a2p-2",
    "0x1.6a09e667f3bcdp-2", "-0x1.6a09e667f3bccp-2", "-0x1.6a09e667f3bcep-2", "0x1.6a09e667f3bcbp-2", "0x1.6a09e667f3bcep-2", "-0x1.6a09e667f3bc5p-2", "-0x1.6a09e667f3bc9p-2", "0x1.6a09e667f3bc4p-2",
    "0x1.1c73b39ae68c9p-2", "-0x1.f6297cff75cb0p-2", "0x1.8f8b83c69a60cp-4", "0x1.a9b66290ea1a5p-2", "-0x1.a9b66290ea1a2p-2", "-0x1.8f8b83c69a602p-4", "0x1.f6297cff75cb2p-2", "-0x1.1c73b39ae68c2p-2",
    "0x1.87de2a6aea964p-3", "-0x1.d906bcf328d47p-2", "0x1.d906bcf328d44p-2", "-0x1.87de2a6aea965p-3", "-0x1.87de2a6aea971p-3", "0x1.d906bcf328d46p-2", "-0x1.d906bcf328d43p-2", "0x1.87de2a6aea95fp-3",
    "0x1.8f8b83c69a60dp-4", "-0x1.1c73b39ae68c8p-2", "0x1.a9b66290ea1a5p-2", "-0x1.f6297cff75cb2p-2", "0x1.f6297cff75cb0p-2", "-0x1.a9b66290ea1a1p-2", "0x1.1c73b39ae68c2p-2", "-0x1.8f8b83c69a616p-4",

)
DCT = np.array([float.fromhex(h) for h in _DCT_HEX], dtype=np.float64).reshape(8, 8)


def zigzag_order() -> np.ndarray:
    """dct.py:84-91: anti-diagonals d = u + v; even ones run from high u to low u."""
    out = []
    for d in range(15):
        us = list(range(max(0, d - 7), min(d, 7) + 1))
        if d % 2 == 0:
            us = us[::-1]
        out += [u * 8 + (d - u) for u in us]
    return np.array(out, dtype=np.uint8)


ZIGZAG = zigzag_order()
FRAME_I, FRAME_P = 0, 1
_PAYLOAD_HEAD = struct.Struct("<BBHHB")  # codec.py:28 quality, format, width, height, plane_count
_RECORD_HEAD = struct.Struct("<BI")      # codec.py:27 frame_type, payload_len


def quant_step(quality: int) -> int:
    """codec.py:46-49 (Python's round: half to even)."""
    if not 0 <= quality <= 100:
        raise ValueError(f"quality {quality} outside 0..100")
    return max(1, int(round((100 - quality) * 0.5)) + 1)


_JOB = np.dtype([("src", "<u8"), ("prev", "<u8"), ("recon", "<u8"), ("block0", "<i8"), ("pitch", "<i4"),
                 ("w", "<i4"), ("h", "<i4"), ("nbx", "<i4"), ("nby", "<i4"), ("is_p", "<i4"), ("step", "<i4"),
                 ("pad", "<i4")])
assert _JOB.itemsize == 64


def _sig(L):
    P, I, LL = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong
    L.fvv_encode_set_tables.restype = I
    L.fvv_encode_set_tables.argtypes = [P, P]
    L.fvv_encode_blocks.restype = I
    L.fvv_encode_blocks.argtypes = [P, I, LL, I, P, P, P]
    L.fvv_encode_tokens.restype = I
    L.fvv_encode_tokens.argtypes = [P, P, LL, P, P]


_tables_set: set = set()


class _Tile:
    """One tile: its frame geometry, plane jobs (offsets inside the stitched
    frame) and two reconstruction banks (ping-pong: a block's edge-clamped
    reads of the previous reconstruction never race with its writes)."""

    def __init__(self, x, y, w, h, fmt, sw, sh, device):
        import torch
        self.w, self.h, self.fmt = w, h, int(fmt)
        self.planes = []  # (byte offset in the stitched frame, pitch, plane w in bytes, plane h)
        if self.fmt == PixelFormat.RGB8:
            self.planes.append((3 * (y * sw + x), 3 * sw, 3 * w, h))
        else:
            self.planes.append((y * sw + x, sw, w, h))
            if self.fmt == PixelFormat.YUV420:
                cw, ch = (sw + 1) // 2, (sh + 1) // 2
                for p in range(2):
                    self.planes.append((sw * sh + p * cw * ch + (y // 2) * cw + x // 2, cw, (w + 1) // 2,
                                        (h + 1) // 2))
        self.recon = [[torch.empty(pw * ph, dtype=torch.uint8, device=device) for (_, _, pw, ph) in self.planes]
                      for _ in range(2)]
        self.index = 0  # frames encoded (TileEncoder.index)


class RigEncoder:
    """Closed-loop FVT1 encoders for every tile of every cluster frame of a rig
    (one codec.TileEncoder per (cluster, tile) in the reference), quality and
    GOP as PipelineConfig.quality / .gop."""

    def __init__(self, layouts, width: int, height: int, fmt, quality: int = 75, gop: int = 30, device=None,
                 threads: int = 8, deflate: str = "device"):
        import torch
        self._L = _lib.require_cuda()
        _sig(self._L)
        if gop < 1:
            raise ValueError("gop must be >= 1")
        if deflate not in ("device", "host"):
            raise ValueError("deflate must be 'device' or 'host'")
        self.deflate = deflate
        self.step = quant_step(quality)
        self.quality, self.gop, self.lossless = int(quality), int(gop), quality == 100
        self.width, self.height, self.format = int(width), int(height), PixelFormat(int(fmt))
        self.device = torch.device(device or "cuda")
        self.layouts = list(layouts)
        self.tiles = []  # per cluster: [(rect, _Tile)]
        self.frame_sizes = []
        for lay in self.layouts:
            rects = tile_rects(lay, width, height)
            nsmall = sum(1 for t in lay.tiles if t.tier == "quarter")
            sw = width + ((nsmall + 3) // 4) * (width // 4)
            self.frame_sizes.append(frame_nbytes(sw, height, fmt))
            self.tiles.append([(r, _Tile(r.x, r.y, r.width, r.height, fmt, sw, height, self.device)) for r in rects])
        dev_idx = self.device.index if self.device.index is not None else torch.cuda.current_device()
        if dev_idx not in _tables_set:
            with torch.cuda.device(dev_idx):
                _lib.check(self._L.fvv_encode_set_tables(DCT.ctypes.data_as(ctypes.c_void_p),
                                                         ZIGZAG.ctypes.data_as(ctypes.c_void_p)))
            _tables_set.add(dev_idx)
        nblocks = sum(((pw + 7) // 8) * ((ph + 7) // 8) for c in self.tiles for _, t in c for (_, _, pw, ph) in t.planes)
        self.nblocks = nblocks
        self.zz = torch.empty((max(1, nblocks), 64), dtype=torch.int16, device=self.device)
        self.ntok = torch.empty(max(1, nblocks), dtype=torch.int32, device=self.device)
        self.tok_off = torch.empty(max(1, nblocks) + 1, dtype=torch.int64, device=self.device)
        self.tokens = torch.empty(max(1, nblocks) * 65 * 3, dtype=torch.uint8, device=self.device)
        self._pool = ThreadPoolExecutor(max_workers=max(1, threads))

    def _build_job_tables(self):
        """The per-plane job fields that never change (geometry, block offsets,
        reconstruction bank addresses) and the plane metadata, built once."""
        import torch
        rows, meta, block0 = [], [], 0
        flat = 0
        for c, tl in enumerate(self.tiles):
            for ti, (rect, t) in enumerate(tl):
                for pi, (off, pitch, pw, ph) in enumerate(t.planes):
                    nbx, nby = (pw + 7) // 8, (ph + 7) // 8
                    rows.append((c, flat, off, t.recon[0][pi].data_ptr(), t.recon[1][pi].data_ptr()))
                    meta.append((c, ti, pi, block0, nbx * nby))
                    block0 += nbx * nby
                flat += 1
        n = len(rows)
        js = np.zeros(n, dtype=[("cluster", "<i8"), ("tile", "<i8"), ("off", "<u8"), ("bank0", "<u8"),
                                ("bank1", "<u8")])
        for i, r in enumerate(rows):
            js[i] = r
        jobs = np.zeros(n, dtype=_JOB)
        for i, m in enumerate(meta):
            _, ti, pi, b0, _nb = m
            off, pitch, pw, ph = self.tiles[m[0]][ti][1].planes[pi]
            jobs[i]["block0"], jobs[i]["pitch"], jobs[i]["w"], jobs[i]["h"] = b0, pitch, pw, ph
            jobs[i]["nbx"], jobs[i]["nby"], jobs[i]["step"] = (pw + 7) // 8, (ph + 7) // 8, self.step
        self._jobs_static, self._meta, self._nblocks_total = js, meta, block0
        self._jobs_host = jobs
        self._jobs_pinned = torch.empty(jobs.nbytes, dtype=torch.uint8, pin_memory=True)
        self._jobs_dev = torch.empty(jobs.nbytes, dtype=torch.uint8, device=self.device)

    def _stream(self):
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def encode(self, clusters, offsets=None) -> list:
        """clusters: the rig's stitched cluster frames packed back to back (uint8
        CUDA, fvv_rig_clusters layout); offsets: byte offset of each cluster
        (default: cumulative sizes).  Returns per cluster the list of record
        bytes (FrameRecord.to_bytes(), codec.py:123-133) in tile-map order."""
        import torch
        if offsets is None:
            offsets = np.concatenate([[0], np.cumsum(self.frame_sizes)[:-1]]).tolist()
        base = clusters.data_ptr()
        if getattr(self, "_jobs_static", None) is None:
            self._build_job_tables()
        js, meta, block0 = self._jobs_static, self._meta, self._nblocks_total
        # per call: source addresses, reconstruction banks and frame type (vectorised)
        idx = np.array([t.index for tl in self.tiles for _, t in tl], dtype=np.int64)[js["tile"]]
        is_p = (idx % self.gop) != 0
        par = (idx & 1).astype(bool)
        jobs = self._jobs_host
        jobs["src"] = np.uint64(base) + np.asarray(offsets, dtype=np.uint64)[js["cluster"]] + js["off"]
        jobs["recon"] = np.where(par, js["bank1"], js["bank0"])
        jobs["prev"] = np.where(is_p, np.where(par, js["bank0"], js["bank1"]), np.uint64(0))
        jobs["is_p"] = is_p.astype(np.int32)
        self._jobs_pinned.numpy()[:] = jobs.view(np.uint8)
        jt = self._jobs_dev
        jt.copy_(self._jobs_pinned, non_blocking=True)
        self._last_jobs, self._last_njobs = jt, len(jobs)
        L, st = self._L, self._stream()
        _lib.check(L.fvv_encode_blocks(ctypes.c_void_p(jt.data_ptr()), len(jobs), block0, int(self.lossless),
                                       ctypes.c_void_p(self.zz.data_ptr()), ctypes.c_void_p(self.ntok.data_ptr()), st))
        self.tok_off[0] = 0
        torch.cumsum(self.ntok[:block0], 0, out=self.tok_off[1:block0 + 1])
        _lib.check(L.fvv_encode_tokens(ctypes.c_void_p(self.zz.data_ptr()), ctypes.c_void_p(self.tok_off.data_ptr()),
                                       block0, ctypes.c_void_p(self.tokens.data_ptr()), st))
        for tl in self.tiles:
            for _, t in tl:
                t.index += 1
        if self.deflate == "device":  # raw DEFLATE of every plane's tokens at once (codec.py:148)
            from .deflate import deflate_streams
            # token offsets at the plane boundaries only (not every block's)
            if getattr(self, "_plane_idx", None) is None or self._plane_idx.numel() != len(meta) + 1:
                self._plane_idx = torch.tensor([m[3] for m in meta] + [block0], dtype=torch.int64,
                                               device=self.device)
            po = (self.tok_off.index_select(0, self._plane_idx) * 3).cpu().numpy()
            plane_offs = [int(v) for v in po]
            self._last_plane_offs = plane_offs
            out, out_off = deflate_streams(self.tokens[:plane_offs[-1]], plane_offs)
            oo = out_off.cpu().numpy()
            nraw = int(oo[-1])
            if getattr(self, "_pinned", None) is None or self._pinned.numel() < nraw:
                self._pinned = torch.empty(max(nraw, 1 << 20), dtype=torch.uint8, pin_memory=True)
            self._pinned[:nraw].copy_(out[:nraw], non_blocking=True)
            torch.cuda.current_stream(self.device).synchronize()
            raw = memoryview(self._pinned.numpy())[:nraw]  # zero-copy views; each record copies once (join)
            datas = [raw[oo[i]:oo[i + 1]] for i in range(len(meta))]
        else:
            offs = self.tok_off[:block0 + 1].cpu().numpy()
            ntot = int(offs[-1])
            tok = self.tokens[:ntot * 3].cpu().numpy().tobytes()

            def deflate(m):
                _, _, _, b0, nb = m
                return zlib.compress(tok[offs[b0] * 3:offs[b0 + nb] * 3], 6)[2:-4]  # raw DEFLATE (codec.py:148)
            datas = list(self._pool.map(deflate, meta))
        out = [[None] * len(tl) for tl in self.tiles]
        parts = {}
        for m, d in zip(meta, datas):
            parts.setdefault((m[0], m[1]), []).append(d)
        for c, tl in enumerate(self.tiles):
            for ti, (rect, t) in enumerate(tl):
                is_p = (t.index - 1) % self.gop != 0
                body = [_PAYLOAD_HEAD.pack(self.quality, int(self.format), t.w, t.h, len(t.planes))]
                for d in parts[(c, ti)]:
                    body += [struct.pack("<I", len(d)), d]
                payload = b"".join(body)
                out[c][ti] = _RECORD_HEAD.pack(FRAME_P if is_p else FRAME_I, len(payload)) + payload
        return out

    def reconstruction(self, cluster: int, tile: int) -> list:
        """The committed reconstruction planes of a tile (host numpy), as
        TileEncoder.reconstruction holds them."""
        _, t = self.tiles[cluster][tile]
        bank = t.recon[(t.index - 1) & 1]
        return [bank[p].cpu().numpy().reshape(ph, pw) for p, (_, _, pw, ph) in enumerate(t.planes)]

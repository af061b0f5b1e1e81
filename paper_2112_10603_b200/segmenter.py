"""TS/HLS packaging of the encoded cluster streams (
the reference's mpegts.py:188-212 mux_segment, playlist.py:54-88 and the
pipeline's _segment stage, server/pipeline.py:320-338).

The muxer is native (csrc/ts_mux.cpp, fvv_ts_mux_segment) and runs without
the interpreter lock, so at every segment boundary all cluster segments are
muxed concurrently instead of one after another.  Segments are byte-identical
to mux_segment's (tests/test_segmenter.py); playlists render exactly as
render_playlist.
"""
from __future__ import annotations

import ctypes
import math
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import _lib

PTS_CLOCK = 90000
_PTS_MASK = (1 << 33) - 1


class GopAlignmentError(Exception):
    """mpegts.GopAlignmentError: a segment must start on intra records."""


def _sig(L):
    P, I, Z = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    L.fvv_ts_segment_bytes.restype = Z
    L.fvv_ts_segment_bytes.argtypes = [P, I, I]
    L.fvv_ts_mux_segment.restype = I
    L.fvv_ts_mux_segment.argtypes = [P, P, I, I, P, P, Z, ctypes.POINTER(Z)]


def frame_pts(nframes: int, fps: int, start_pts: int = 0) -> list:
    """PTS of frame i: start + round(i * 90000 / fps), 33-bit (mpegts.py:199)."""
    return [(start_pts + round(i * PTS_CLOCK / fps)) & _PTS_MASK for i in range(nframes)]


def mux_segment(frames: list, fps: int, start_pts: int = 0) -> bytes:
    """One cluster's TS segment from per-frame lists of tile records (bytes)."""
    if fps <= 0:
        raise ValueError("fps must be positive")
    L = _lib.load()
    _sig(L)
    nframes = len(frames)
    ntiles = len(frames[0]) if frames else 0
    if any(len(f) != ntiles for f in frames):
        raise ValueError("every frame of a segment carries the same tiles")
    recs = [bytes(r) for f in frames for r in f]
    lens = np.array([len(r) for r in recs], dtype=np.uint32)
    bufs = [ctypes.create_string_buffer(r, len(r)) if r else ctypes.create_string_buffer(1) for r in recs]
    ptrs = (ctypes.c_void_p * max(1, len(recs)))(*[ctypes.addressof(b) for b in bufs])
    pts = np.array(frame_pts(nframes, fps, start_pts), dtype=np.int64)
    size = int(L.fvv_ts_segment_bytes(lens.ctypes.data_as(ctypes.c_void_p), ntiles, nframes))
    out = ctypes.create_string_buffer(max(1, size))
    written = ctypes.c_size_t(0)
    rc = L.fvv_ts_mux_segment(ptrs, lens.ctypes.data_as(ctypes.c_void_p), ntiles, nframes,
                              pts.ctypes.data_as(ctypes.c_void_p), out, size, ctypes.byref(written))
    if rc == -2:
        bad = next(k for k, r in enumerate(frames[0]) if not r or r[0] != 0)
        raise GopAlignmentError(f"segment does not start on an intra record (tile {bad})")
    if rc != 0:
        raise RuntimeError(f"fvv_ts_mux_segment failed ({rc})")
    return out.raw[:written.value]


class SegmentMuxer:
    """Concurrent per-cluster muxing at a segment boundary."""

    def __init__(self, threads: int = 8):
        self._pool = ThreadPoolExecutor(max_workers=max(1, threads))

    def mux_clusters(self, per_cluster_frames: list, fps: int, start_pts: int) -> list:
        futs = [self._pool.submit(mux_segment, frames, fps, start_pts) for frames in per_cluster_frames]
        return [f.result() for f in futs]


# ---------------------------------------------------------------------------
# HLS playlists (playlist.py:23-88): a sliding window of segments per cluster
# ---------------------------------------------------------------------------
@dataclass
class PlaylistWindow:
    target_duration: int
    window_size: int = 6
    media_sequence: int = 0
    entries: tuple = ()
    ended: bool = False
    version: int = 3

    @staticmethod
    def for_segments(segment_duration: float, window_size: int = 6) -> "PlaylistWindow":
        return PlaylistWindow(math.ceil(segment_duration), window_size)

    @property
    def next_sequence(self) -> int:
        return self.media_sequence + len(self.entries)

    def rotate(self, sequence: int, duration: float) -> str:
        """Append segment `sequence`, evict beyond the window, return the m3u8 text."""
        if self.ended:
            raise ValueError("playlist already ended")
        if sequence != self.next_sequence:
            raise ValueError(f"segment {sequence} out of order, expected {self.next_sequence}")
        entries = self.entries + ((f"seg{sequence:05d}.ts", duration),)
        drop = max(0, len(entries) - self.window_size)
        self.entries = entries[drop:]
        self.media_sequence += drop
        return self.render()

    def end(self) -> str:
        self.ended = True
        return self.render()

    def render(self) -> str:
        out = ["#EXTM3U", f"#EXT-X-VERSION:{self.version}", f"#EXT-X-TARGETDURATION:{self.target_duration}",
               f"#EXT-X-MEDIA-SEQUENCE:{self.media_sequence}"]
        for uri, dur in self.entries:
            out += [f"#EXTINF:{dur:.3f},", uri]
        if self.ended:
            out.append("#EXT-X-ENDLIST")
        return "\n".join(out) + "\n"

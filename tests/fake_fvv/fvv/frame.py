import enum
from dataclasses import dataclass

import numpy as np


class PixelFormat(enum.IntEnum):
    GRAY8 = 0
    YUV420 = 1
    RGB8 = 2


@dataclass(frozen=True)
class Frame:
    width: int
    height: int
    format: PixelFormat
    planes: tuple
    timestamp: int = 0


def frame_from_planes(planes, fmt, timestamp=0):
    h, w = planes[0].shape[:2]
    return Frame(w, h, fmt, tuple(np.ascontiguousarray(p) for p in planes), timestamp)

from dataclasses import dataclass
from typing import Callable


@dataclass(frozen=True)
class InterpConfig:
    block_size: tuple = (8, 8, 8)
    search_radius: tuple = (12, 4, 2)
    mask_epsilon: float = 1e-3
    border_band: int = 8
    refine: Callable | None = None


def interpolate(left, right, config=None, diagnostics=False):
    raise AssertionError("CPU interpolate called: plugin not installed")


def dense_views(left, right, stages, config=None):
    raise AssertionError("CPU dense_views called: plugin not installed")

from dataclasses import dataclass


class LayoutError(Exception):
    pass


@dataclass(frozen=True)
class TileRect:
    index: int
    tier: str
    x: int
    y: int
    width: int
    height: int


@dataclass(frozen=True)
class ClusterFrame:
    cluster_id: int
    frame: object
    tile_map: tuple


def downscale(frame, factor):
    raise AssertionError("CPU downscale called: plugin not installed")


def assemble_cluster_frame(anchor_frame, interp_frames, layout):
    raise AssertionError("CPU assemble called: plugin not installed")

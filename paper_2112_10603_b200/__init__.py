"""B200-native dense view synthesis (arXiv 2112.10603 hot path).

Drop-in for the reference package's interpolation / tiling API (fvv.interp,
fvv.cluster); compute runs in hand-written sm_100a CUDA kernels behind the
C ABI of include/fvv_b200.h.  See DESIGN.md.
"""
from .frame import Frame, PixelFormat, frame_from_planes, frame_from_packed, gray, packed  # noqa: F401
from .interp import (FlowField, InterpConfig, InterpDiagnostics, Interpolator,  # noqa: F401
                     ScaleDiagnostics, dense_views, interpolate)
from .viewmodel import CameraRig, ViewIndexModel  # noqa: F401
from .cluster import (ClusterFrame, ClusterLayout, LayoutError, TileRect, TileRef,  # noqa: F401
                      assemble_cluster_frame, build_layouts, cluster_geometry, crop_frame, downscale,
                      rig_clusters, tile_rects)

from .pipeline import RigPipeline  # noqa: F401

__version__ = "0.1.0"

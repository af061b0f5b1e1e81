from ..cluster import assemble_cluster_frame, downscale  # noqa: F401  (bound at import, as the reference does)
from ..interp import dense_views  # noqa: F401

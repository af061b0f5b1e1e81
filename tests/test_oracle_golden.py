"""The CPU oracle (oracle/) against the reference's own golden vectors.

These pin the oracle before it is trusted as the parity checker for the
CUDA path (tests/test_gpu_parity.py).  CPU only.
"""
import numpy as np
import pytest

from conftest import golden_names, load_golden
from oracle import oracle as O


@pytest.mark.parametrize("name", golden_names("interp"))
def test_oracle_interpolate_matches_golden(name):
    g = load_golden(name)
    w, h, fmt = int(g["w"]), int(g["h"]), int(g["fmt"])
    if "flow_lr" in g:
        out, diag = O.interpolate(g["left"], g["right"], w, h, fmt, with_diag=True)
        assert np.array_equal(diag["flow_lr"], g["flow_lr"])
        assert np.array_equal(diag["flow_rl"], g["flow_rl"])
        assert np.array_equal(diag["mask"], g["mask"])
    else:
        out = O.interpolate(g["left"], g["right"], w, h, fmt)
    assert np.array_equal(out, g["out"])


def test_oracle_dense_views_matches_golden():
    g = load_golden("dense3_yuv420_64x48")
    out = O.dense_views(g["left"], g["right"], int(g["w"]), int(g["h"]), int(g["fmt"]), int(g["stages"]))
    assert np.array_equal(out, g["out"])


def test_oracle_rig_and_clusters_match_golden():
    g = load_golden("rig3_s2_vps2_yuv420_64x48")
    w, h, fmt, stages = int(g["w"]), int(g["h"]), int(g["fmt"]), int(g["stages"])
    views = O.rig_dense_views(g["cams"], w, h, fmt, stages)
    assert np.array_equal(views, g["views"])
    q = np.stack([O.downscale(v, w, h, fmt, 4) for v in views])
    assert np.array_equal(q, g["quarters"])


def test_candidate_order_tie_rule():
    # flow.py:57-66: primary d^2, then |dy|, then dy, then dx
    dx, dy, idx = O.candidate_order(2)
    keys = [(x * x + y * y, abs(y), y, x) for x, y in zip(dx, dy)]
    assert keys == sorted(keys)
    assert (dx[0], dy[0]) == (0, 0)
    side = 5
    assert np.array_equal(idx, (dy + 2) * side + (dx + 2))

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


# ---------------------------------------------------------------------------
# 1080p pins (tests/golden/make_golden_1080p.py): the reference's outputs on
# bench.synth_rig inputs, regenerated here from the stored seed
# ---------------------------------------------------------------------------
def sha(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_oracle_1080p_pair_matches_reference_golden():
    from bench import synth_rig
    g = load_golden("ref1080_pair")
    w, h = int(g["w"]), int(g["h"])
    cams = synth_rig(w, h, 1, int(g["cams"]), seed=int(g["seed"]))
    out, diag = O.interpolate(cams[0], cams[1], w, h, 1, with_diag=True)
    assert np.array_equal(out, g["out"])
    assert sha(diag["flow_lr"]) == str(g["flow_lr_sha"])
    assert sha(diag["flow_rl"]) == str(g["flow_rl_sha"])
    assert sha(diag["mask"]) == str(g["mask_sha"])


def cfg3_clusters(views, w, h, fmt, C, stages, vps):
    step = 1 << stages
    total = views.shape[0]
    out = []
    for c in range(C):
        a = c * step
        lo, hi = max(0, a - vps), min(total - 1, a + vps)
        smalls = np.stack([O.downscale(views[i], w, h, fmt, 4) for i in range(lo, hi + 1) if i != a])
        out.append(O.assemble_cluster(views[a], w, h, fmt, smalls))
    return out


def test_oracle_1080p_cfg3_rig_matches_reference_golden():
    """BASELINE config 3 (4-camera 1080p rig, 45 views, 4 cluster frames): every
    view and cluster frame of the oracle hashes to the reference's."""
    from bench import synth_rig
    g = load_golden("ref1080_cfg3")
    w, h, C, S, vps = int(g["w"]), int(g["h"]), int(g["cams"]), int(g["stages"]), int(g["vps"])
    cams = synth_rig(w, h, 1, C, seed=int(g["seed"]))
    views = O.rig_dense_views(cams, w, h, 1, S)
    assert [sha(v) for v in views] == [str(s) for s in g["view_sha"]]
    cl = cfg3_clusters(views, w, h, 1, C, S, vps)
    assert [sha(c) for c, _ in cl] == [str(s) for s in g["cluster_sha"]]
    assert [sw for _, sw in cl] == list(g["cluster_w"])

"""plugin.install(fvv) rebinds the reference's names (including the copies
bound at import time in fvv.server.pipeline) to the B200 path; results come
back as the package's own Frame type and match the reference's golden output."""
import importlib
import os
import sys

import numpy as np
import pytest

from conftest import load_golden

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture()
def fake_fvv():
    sys.path.insert(0, os.path.join(HERE, "fake_fvv"))
    for m in [m for m in sys.modules if m == "fvv" or m.startswith("fvv.")]:
        del sys.modules[m]
    fvv = importlib.import_module("fvv")
    for sub in ("frame", "interp", "cluster", "server.pipeline"):
        importlib.import_module("fvv." + sub)
    yield fvv
    from paper_2112_10603_b200 import plugin
    plugin.uninstall()
    sys.path.remove(os.path.join(HERE, "fake_fvv"))
    for m in [m for m in sys.modules if m == "fvv" or m.startswith("fvv.")]:
        del sys.modules[m]


def test_install_rebinds_every_seam(fake_fvv):
    from paper_2112_10603_b200 import plugin
    before = (fake_fvv.interp.interpolate, fake_fvv.server.pipeline.dense_views,
              fake_fvv.server.pipeline.downscale)
    plugin.install(fake_fvv)
    after = (fake_fvv.interp.interpolate, fake_fvv.server.pipeline.dense_views,
             fake_fvv.server.pipeline.downscale)
    assert all(a is not b for a, b in zip(after, before))
    assert fake_fvv.server.pipeline.dense_views is fake_fvv.interp.dense_views
    plugin.uninstall()
    assert fake_fvv.interp.interpolate is before[0]


@pytest.mark.gpu
def test_installed_interpolate_matches_golden(fake_fvv):
    from paper_2112_10603_b200 import plugin
    from paper_2112_10603_b200.frame import frame_from_packed
    plugin.install(fake_fvv)
    g = load_golden("scene_yuv420_96x72")
    ours = [frame_from_packed(g[k], 96, 72, 1) for k in ("left", "right")]
    L, R = (fake_fvv.frame.Frame(f.width, f.height, fake_fvv.frame.PixelFormat.YUV420, f.planes)
            for f in ours)
    out = fake_fvv.interp.interpolate(L, R)
    assert isinstance(out, fake_fvv.frame.Frame)
    assert np.array_equal(np.concatenate([p.reshape(-1) for p in out.planes]), g["out"])
    views = fake_fvv.server.pipeline.dense_views(L, R, 2)
    assert len(views) == 3 and isinstance(views[0], fake_fvv.frame.Frame)

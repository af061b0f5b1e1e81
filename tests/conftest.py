import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HERE = os.path.dirname(os.path.abspath(__file__))
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA product path)")
    config.addinivalue_line("markers", "reference: needs /root/reference (build container only)")


GOLDEN_DIR = os.path.join(HERE, "golden")


def load_golden(name):
    d = np.load(os.path.join(GOLDEN_DIR, name + ".npz"))
    return {k: d[k] for k in d.files}


def golden_names(kind=None):
    out = []
    for f in sorted(os.listdir(GOLDEN_DIR)):
        if f.endswith(".npz"):
            name = f[:-4]
            if kind is None or str(np.load(os.path.join(GOLDEN_DIR, f))["kind"]) == kind:
                out.append(name)
    return out


@pytest.fixture()
def rng():
    return np.random.default_rng(1234)

"""CPU check of the DEFLATE restatement the device kernels run
(csrc/zdeflate_core.h): tools/zdeflate_model.cpp runs its steps as plain loops
and compares ~180 streams byte for byte with the system zlib (1.3, the same
library version the interpreter's zlib module reports)."""
import shutil
import subprocess
import zlib
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(shutil.which("g++") is None or not Path("/usr/include/zlib.h").exists(),
                    reason="needs g++ and zlib headers")
def test_model_identical_to_system_zlib(tmp_path):
    assert zlib.ZLIB_RUNTIME_VERSION.startswith("1.3")
    exe = tmp_path / "zdm"
    subprocess.run(["g++", "-O2", "-std=c++17", str(ROOT / "tools" / "zdeflate_model.cpp"), "-o", str(exe), "-lz"],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "all identical" in r.stdout, r.stdout[-3000:]
    assert "NIL hits: 0" not in r.stdout  # the end-of-input slide edge is exercised

"""Runs the C++ drop-in test (tests/cpp/test_dropin.cpp): the reference's own
raster.hpp API linked against paper_2412_04459_b200/cpp/raster_dropin.cpp
(instead of raster.cpp) on the GPU, checked against the C oracle."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2412_04459_b200", "cpp", "build", "test_dropin")


def test_cpp_dropin_suite():
    if not os.path.exists(BIN):
        pytest.skip("drop-in test binary not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "ALL PASSED" in r.stdout

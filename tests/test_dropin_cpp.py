"""The reference C++ API drives the B200 engine unchanged (include/splbm/engine_device.hpp):
oracle/_ref/dropin_test (built from tests/cpp/dropin_test.cpp against the reference headers)
runs the reference TileEngineT2C<double> and TileEngineT2CDevice side by side — bitwise equal."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "dropin_test")


def test_reference_api_drives_device_engine():
    if not os.path.exists(BIN):
        pytest.skip("dropin_test not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout

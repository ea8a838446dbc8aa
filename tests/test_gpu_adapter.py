"""Drop-in check through the C++ boundary: the reference's own host objects
driven through include/dgb_reference_adapter.hpp (libdgb.so) and through the
unmodified reference operators, in one process (oracle/adapter_parity.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_objects_through_adapter_match_reference():
    exe = os.path.join(ROOT, "oracle", "_ref", "adapter_parity")
    if not os.path.exists(exe):
        pytest.skip("adapter_parity not built (make -C oracle adapter)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "adapter parity ok" in r.stdout

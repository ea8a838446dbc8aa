"""The reference's own six doctest suites (proj/tests/*.cpp, 48 test cases,
~49k checks), compiled unchanged against oracle/_ref with the from-scratch
doctest shim (oracle/doctest_shim/doctest.h): proves the oracle build is the
reference.  CPU only; skipped where the binaries were not built."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITES = ["test_kernels", "test_quadrature", "test_mesh", "test_space", "test_forms", "test_krylov"]


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes(suite):
    exe = os.path.join(ROOT, "oracle", "_ref", suite)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (make -C oracle tests)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout

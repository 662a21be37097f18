"""The C++ drop-in shim (include/pyrit_b200_shim.hpp) used exactly like the reference:
oracle/_ref/shim_check is built against the unmodified reference headers and
compares pyrit::cuda::encode/decode with the reference's own encode()/encode_crs()
and round-trips decode on five field/code shapes."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "shim_check")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="shim_check not built (needs the reference headers)")
def test_shim_matches_reference(cuda):
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "SHIM CHECK PASSED" in r.stdout


SAN = os.path.join(ROOT, "build", "sanitize_check")


@pytest.mark.skipif(not os.path.exists(SAN), reason="build/sanitize_check not built")
def test_sanitize_driver_plain(cuda):
    """The compute-sanitizer driver (tests/sanitize_check.cpp) passes without the sanitizer:
    every kernel shape on exact-size buffers matches the host interpreter."""
    r = subprocess.run([SAN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "SANITIZE CHECK PASSED" in r.stdout

"""The C++20 drop-in (include/pmmf_b200/dropin.hpp) compiled against the
reference headers (oracle/_ref/dropin_check, built in the build container):
pmmf_b200::factorize and GpuOperator equal pmmf::factorize / MmfOperator under
the reference's own operator== on a seeded R-MAT input."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_check")


@pytest.mark.gpu
def test_cpp_dropin_matches_reference():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/dropin_check not built")
    out = subprocess.run([BIN, "11"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "PASS" in out.stdout

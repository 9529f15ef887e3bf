"""GPU: the C++ operator API (include/vattn_b200/mha.hpp) as a drop-in for the
reference's vattn::forward_fused / backward_fused, checked in one C++ program
against the reference library itself (tests/cpp/mha_cpp_parity.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(__file__), "cpp", "_build", "mha_cpp_parity")


@pytest.mark.skipif(not os.path.exists(BIN), reason="C++ parity driver not built (needs the reference headers)")
def test_cpp_api_parity_against_reference_library():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failure(s)" in r.stdout

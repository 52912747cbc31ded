"""C++ drop-in check: the reference's own SparseMatrix/Hierarchy types go
through paper_2408_08262_b200/cpp/airgraph_gpu.hpp into the GPU engine and
the results equal the reference functions' results under the reference's
exact operator== (oracle/dropin_test.cpp; the binary is built here from
/root/reference and travels with oracle/_ref)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "dropin_test")


@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/dropin_test not built (needs /root/reference)")
def test_cpp_dropin_with_reference_types():
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "FAIL" not in out.stdout

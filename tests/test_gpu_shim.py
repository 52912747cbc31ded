"""The reference's OWN unit tests (tests/unit/test_sparse.cpp,
test_coarsening.cpp, test_gmres_poly.cpp, test_air.cpp, test_solve.cpp)
linked unchanged against the airgraph:: shim (paper_2408_08262_b200/cpp/
airgraph_shim.cpp) over the C-ABI: every hot-path function of the
reference's API runs on the GPU (SURVEY §8b drop-in). Built here by
oracle/Makefile `shim` (needs /root/reference); the binary travels in
oracle/_ref. The only failures allowed are the reference's dense
exact-inverse / exact-coarse-solve test hooks (air.cpp:13-54), which the GPU
setup does not offer (out of scope)."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "ref_unit_tests_gpu")
HOOKS = {
    "isolated F rows stay empty and the two-level solve still works",
    "two-level hook reduces any residual to round-off in one cycle",
    "single-level hierarchy: the V-cycle is just the coarse solve",
    "richardson on b = 0 converges in zero iterations",
}


@pytest.mark.skipif(not os.path.exists(BIN), reason="shim test binary not built (needs /root/reference)")
def test_reference_unit_tests_pass_on_gpu_backend():
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    text = out.stdout + out.stderr
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", text)
    assert m, text[-2000:]
    total, passed, failed = map(int, m.groups())
    failing = set(re.findall(r'test "(.*?)" (?:threw|failed)', text))
    assert failing <= HOOKS, sorted(failing - HOOKS)
    assert total == 72 and passed >= total - len(HOOKS), text[-2000:]

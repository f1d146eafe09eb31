"""The C++ drop-in boundary: include/bmatch_b200.hpp behind the reference's own
registry, driver and suite-runner API (tests/cpp/shim_test.cpp, built by
`make shimtest` against the reference compiled from its sources)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "oracle", "_ref", "shim_test")

needs_shim = pytest.mark.skipif(not os.path.exists(SHIM), reason="shim_test not built (needs /root/reference at build time)")


@needs_shim
def test_shim_registers_and_has_no_cpu_fallback():
    out = subprocess.run([SHIM, "--no-gpu"], capture_output=True, text=True, timeout=120,
                         env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    assert out.returncode == 0, out.stderr
    assert out.stdout.startswith("PASS"), out.stdout


@pytest.mark.gpu
@needs_shim
def test_shim_reference_api_on_gpu():
    out = subprocess.run([SHIM], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("PASS"), out.stdout

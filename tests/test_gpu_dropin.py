"""GPU: the reference's executor tests run through the C++ drop-in dcp::gpu::run
(include/dcp_gpu.hpp) — same signature as dcp::run (simexec.hpp:207)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_build", "test_dcp_gpu_run")


def test_dropin_reference_suite():
    assert os.path.exists(BIN), "drop-in test binary not built (tools/build.py)"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0 and "DROPIN PASS" in r.stdout, r.stdout + r.stderr

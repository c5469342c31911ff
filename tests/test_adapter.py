"""The ttune adapter (integration/ttune_gpu_executor.cpp) compiled against the
reference's own headers and linked with the reference library and libttb.so
(oracle/Makefile target `adapter`, run by build()).

CPU: every user error of ttune::gpu::reference_transpose / execute_plan is the
reference's exception type and message on the same arguments (run_any order,
executor.cpp:371-385; check_buffers executor.cpp:315-322).  The GPU half is
tests/test_gpu_adapter.py.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "adapter_check")


def test_adapter_errors_match_reference():
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/adapter_check not built (reference tree absent)")
    r = subprocess.run([EXE, "errors"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "errors: 12 cases checked" in r.stdout

"""GPU half of the adapter check: ttune::gpu::{reference_transpose,
execute_plan, transpose_device} (integration/ttune_gpu_executor.cpp) write the
same bytes as ttune::reference_transpose -- the unmodified reference library
-- into ttune TensorBuffers, whole B buffer with padding, for problems shaped
like BASELINE's configs, mixed kinds, identity and rank 1.  The binary is
prebuilt in this container (oracle/_ref travels to the GPU box)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "adapter_check")


@pytest.mark.gpu
def test_adapter_bytes_match_reference_library():
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/adapter_check not built")
    r = subprocess.run([EXE, "all"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "gpu: 11 problems checked" in r.stdout, r.stdout

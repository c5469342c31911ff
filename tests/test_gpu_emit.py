"""Emitted kernels compute the same bytes as the oracle (test_emit.cpp:207-239:
"emitted kernels compute the same bytes as the executor"): each emitted .cu is
built into a shared object with nvcc, loaded, and its reference-shaped entry
(device pointers, default stream) run on the device; the whole B buffer,
padding included, must equal the CPU oracle's bytes.
"""
import ctypes as C
import shutil
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1603_02297_b200 as ttb  # noqa: E402
from oracle import COMPONENTS, SCALAR, kind_id  # noqa: E402
from problems import b_sizes  # noqa: E402

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"

# the reference's compile-and-check problems (test_emit.cpp:208-238) and its golden ones
CASES = [
    ("kss", "s", "s", [2, 1], [41, 23], [44, 23], [25, 41], 1.5, 0.0),
    ("ksd", "s", "d", [3, 1, 2], [19, 5, 7], [19, 6, 7], None, 2.0, 3.0),
    ("kds", "d", "s", [2, 1], [33, 12], None, None, 0.5, 1.0),
    ("kzz", "z", "z", [2, 1], [21, 10], None, None, 2.0, 1.5),
    ("kc1", "s", "s", [1, 3, 2], [13, 6, 10], [14, 6, 10], [13, 11, 6], 1.5, 0.5),
    ("k1d", "c", "c", [1], [2311], None, None, 2.0, 3.0),
    ("kpl", "s", "s", [2, 1], [26, 18], None, None, 2.0, 0.0),
    ("g1", "s", "s", [3, 2, 1], [48, 7, 32], None, None, 2.0, 1.0),
    ("g2", "d", "d", [2, 1], [17, 19], None, None, 1.0, 0.0),
    ("g3", "s", "s", [1, 3, 2], [16, 7, 9], None, None, 2.0, 1.0),
    ("r6", "d", "d", [3, 5, 2, 6, 4, 1], [6, 5, 4, 3, 4, 6], None, None, 0.7, 1.1),
]


@pytest.mark.parametrize("tag,ka,kb,perm,sizes,lda,ldb,alpha,beta", CASES, ids=[c[0] for c in CASES])
def test_emitted_kernel_matches_oracle(tmp_path, coracle, tag, ka, kb, perm, sizes, lda, ldb, alpha,
                                       beta):
    p = ttb.make_problem(perm, sizes, ka, kb, alpha, beta, lda, ldb)
    plan = ttb.GpuPlan(p, cache=False)
    for which, text in (("heur", plan.describe()), ("tile", None)):
        k = ttb.emit_source(p, text, f"{tag}_{which}")
        src, _ = ttb.write_kernel_files(k, tmp_path / f"{tag}_{which}")
        so = tmp_path / f"lib{tag}_{which}.so"
        r = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-fmad=false",
                            "-Xcompiler", "-fPIC", "-shared", "-o", str(so), src],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-3000:]
        lib = C.CDLL(str(so))
        fn = getattr(lib, k.entry_symbol)
        dbl = kind_id(ka) in (1, 3) or kind_id(kb) in (1, 3)
        W = C.c_double if dbl else C.c_float
        fn.argtypes = [C.c_void_p, C.c_void_p, W, W]
        fn.restype = None
        rng = np.random.default_rng(len(tag))
        na = coracle.required_elements_a(sizes, lda)
        nb = coracle.required_elements_b(perm, sizes, ldb)
        A = np.zeros(na * COMPONENTS[kind_id(ka)], SCALAR[kind_id(ka)])
        B = np.zeros(nb * COMPONENTS[kind_id(kb)], SCALAR[kind_id(kb)])
        coracle.fill_sentinel(ka, A)
        coracle.fill_sentinel(kb, B)
        coracle.fill_uniform(ka, sizes, lda, int(rng.integers(1 << 30)), A)
        if beta != 0.0:
            coracle.fill_uniform(kb, b_sizes(perm, sizes), ldb, int(rng.integers(1 << 30)), B)
        want = B.copy()
        coracle.transpose(ka, kb, perm, sizes, lda, ldb, alpha, A, beta, want)
        dA = torch.from_numpy(A).cuda()
        dB = torch.from_numpy(B.copy()).cuda()
        torch.cuda.synchronize()
        fn(dA.data_ptr(), dB.data_ptr(), alpha, beta)
        torch.cuda.synchronize()
        assert dB.cpu().numpy().tobytes() == want.tobytes(), (tag, which, k.entry_symbol)

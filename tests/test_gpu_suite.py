"""The paper's 57-case benchmark suite (build_benchmark,
benchmark.cpp:166-220, alpha = beta = 1) on the GPU: every case, at a small
volume, through the heuristic plan and the autotuned plan, each output's u64
checksum equal to the CPU oracle's on the same inputs (the reference's
run_benchmark verifies every tuned case the same way, benchmark.cpp:238-246).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1603_02297_b200 as ttb  # noqa: E402
from oracle import COMPONENTS, SCALAR, kind_id  # noqa: E402


@pytest.mark.parametrize("kind,mib", [("s", 4), ("d", 4), ("c", 2), ("z", 2)])
def test_suite_every_case_matches_oracle(coracle, kind, mib):
    cases = ttb.build_benchmark(mib << 20, kind, 42)
    assert len(cases) == 57
    for i, c in enumerate(cases):
        p = c.problem
        na, nb = ttb.required_elements_a(p), ttb.required_elements_b(p)
        sb = ttb.sizes_b(p)
        A = np.zeros(na * COMPONENTS[kind_id(kind)], SCALAR[kind_id(kind)])
        B = np.zeros(nb * COMPONENTS[kind_id(kind)], SCALAR[kind_id(kind)])
        coracle.fill_uniform(kind, p.sizes, None, 2 * i + 1, A)
        coracle.fill_uniform(kind, sb, None, 2 * i + 2, B)
        want_B = B.copy()
        coracle.transpose(kind, kind, p.perm.map, p.sizes, None, None, 1.0, A, 1.0, want_B)
        want = coracle.checksum(kind, sb, None, want_B)
        a, b = ttb.TensorBuffer(kind, na), ttb.TensorBuffer(kind, nb)
        ttb.fill_uniform(kind, p.sizes, None, 2 * i + 1, a.data_ptr())
        ttb.fill_uniform(kind, sb, None, 2 * i + 2, b.data_ptr())
        plan = ttb.GpuPlan(p, cache=False)
        plan.execute(a, b)                        # heuristic plan, one application
        assert ttb.checksum(kind, sb, None, b.data_ptr()) == want, (c.id, plan.describe())
        ttb.fill_uniform(kind, sb, None, 2 * i + 2, b.data_ptr())
        plan.autotune(a, b, warmups=1, reps=2)   # beta != 0: tunes on scratch, one application
        assert ttb.checksum(kind, sb, None, b.data_ptr()) == want, (c.id, plan.describe())

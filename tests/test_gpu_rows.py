"""Bulk row copies (rows.cuh, plan text ``bulk=``): permutations that keep the
stride-1 index (run_case1 / run_copy_1d, executor.cpp:164-211) with rows of
at least 1 KB at any element alignment -- rows whose A and B starts sit at
different 16-byte phases, padded rows, rank 1, segments that split rows,
every kind pair and alpha/beta -- bit-exact bytes of the whole B buffer
against the oracle, for every bulk candidate.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1603_02297_b200 as ttb  # noqa: E402
from oracle import COMPONENTS, SCALAR, kind_id  # noqa: E402
from problems import b_sizes  # noqa: E402

PAIRS = [("s", "s"), ("d", "d"), ("c", "c"), ("z", "z"), ("s", "d"), ("d", "s"), ("c", "z"),
         ("z", "c")]

CASES = [
    ([1, 3, 2], [1501, 7, 9], None, None),            # odd rows: every 16-byte phase
    ([1, 3, 2], [374, 20, 13], None, None),           # the suite's d3 case-1 shape, smaller
    ([1, 3, 2], [1030, 5, 4], [1033, 5, 4], [1031, 4, 5]),  # padded rows, different phases
    ([1, 2], [70001, 3], None, None),                 # identity: one merged row of 210003, split in segments
    ([1, 4, 3, 2], [600, 3, 4, 5], None, None),
    ([1, 3, 2], [301, 37, 23], [303, 37, 23], None),      # 1204-byte rows, padded A
]


def _inputs(coracle, rng, ka, kb, perm, sizes, lda, ldb, beta):
    na = coracle.required_elements_a(sizes, lda)
    nb = coracle.required_elements_b(perm, sizes, ldb)
    A = np.zeros(na * COMPONENTS[kind_id(ka)], SCALAR[kind_id(ka)])
    B = np.zeros(nb * COMPONENTS[kind_id(kb)], SCALAR[kind_id(kb)])
    coracle.fill_sentinel(ka, A)
    coracle.fill_sentinel(kb, B)
    coracle.fill_uniform(ka, sizes, lda, int(rng.integers(1 << 30)), A)
    if beta != 0.0:
        coracle.fill_uniform(kb, b_sizes(perm, sizes), ldb, int(rng.integers(1 << 30)), B)
    return A, B


@pytest.mark.parametrize("ka,kb", PAIRS)
def test_bulk_rows_every_candidate_bit_exact(coracle, ka, kb):
    rng = np.random.default_rng(990 + kind_id(ka) * 4 + kind_id(kb))
    n_run = 0
    for perm, sizes, lda, ldb in CASES:
        for alpha, beta in [(1.0, 0.0), (1.3, 0.0), (0.7, 1.1)]:
            p = ttb.make_problem(perm, sizes, ka, kb, alpha, beta, lda, ldb)
            A, B = _inputs(coracle, rng, ka, kb, perm, sizes, lda, ldb, beta)
            want = B.copy()
            coracle.transpose(ka, kb, perm, sizes, lda, ldb, alpha, A, beta, want)
            texts = [t for t in ttb.GpuPlan(p, cache=False).candidates() if "bulk=" in t]
            texts.append("kern=copy;v=1;kx=0;ky=0;tx=1;ty=1;order=0;occ=0;bulk=1;st=2")  # tiny segments
            for text in texts:
                plan = ttb.GpuPlan(p, cache=False)
                try:
                    plan.select(text)
                except ValueError:
                    continue
                dA = torch.from_numpy(A.copy()).cuda()
                dB = torch.from_numpy(B.copy()).cuda()
                plan.execute(dA, dB)
                torch.cuda.synchronize()
                assert dB.cpu().numpy().tobytes() == want.tobytes(), (perm, sizes, lda, ldb, alpha, beta, text)
                n_run += 1
    assert n_run > 0


def test_bulk_rows_at_element_offsets(coracle):
    """Buffers at 4-byte offsets (fp32): bulk rows read the aligned superset
    and store at B's own phase, so no fallback is needed."""
    perm, sizes = [1, 3, 2], [1501, 7, 9]
    p = ttb.make_problem(perm, sizes, "s", "s", 0.5, 2.0)
    rng = np.random.default_rng(5)
    A, B = _inputs(coracle, rng, "s", "s", perm, sizes, None, None, 2.0)
    want = B.copy()
    coracle.transpose("s", "s", perm, sizes, None, None, 0.5, A, 2.0, want)
    for off_a, off_b in [(1, 0), (0, 3), (2, 1)]:
        dA = torch.zeros(A.size + 4, device="cuda")
        dB = torch.zeros(B.size + 4, device="cuda")
        dA[off_a:off_a + A.size] = torch.from_numpy(A).cuda()
        dB[off_b:off_b + B.size] = torch.from_numpy(B).cuda()
        plan = ttb.GpuPlan(p, cache=False)
        plan.select("kern=copy;v=1;kx=0;ky=0;tx=1;ty=1;order=0;occ=0;bulk=16;st=4")
        plan.execute(dA.data_ptr() + 4 * off_a, dB.data_ptr() + 4 * off_b)
        torch.cuda.synchronize()
        assert dB[off_b:off_b + B.size].cpu().numpy().tobytes() == want.tobytes(), (off_a, off_b)

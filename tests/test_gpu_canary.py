"""Out-of-bounds and race evidence without compute-sanitizer (closed on this
pool): every candidate plan of small problems that exercise the asynchronous
kernels (bulk-copy ring, tensor maps, work-stealing counters, copy rows) runs
on buffers embedded in 64 KB canary regions on both sides.  After five
repeated executions the canaries around A and B must be untouched (no write
outside B's footprint, none into A), B must equal the oracle bit for bit
(padding included), and every repetition must give identical bytes (no
schedule-dependent result) -- the reference's invariance gate
(test_executor.cpp:195-210) applied across plans and repetitions.
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

GUARD = 64 * 1024  # bytes of canary on each side
CASES = [
    ("s", [2, 1], [300, 260], None, None, 1.0, 0.0),
    ("s", [2, 1], [300, 260], None, None, 0.7, 1.1),
    ("d", [3, 1, 2], [40, 21, 33], [41, 21, 33], [22, 34, 40], 1.0, 0.5),
    ("c", [3, 2, 1], [4, 96, 70], [8, 96, 70], [70, 96, 8], 1.0, 0.0),
    ("s", [1, 3, 2], [48, 30, 17], None, None, 1.0, 0.5),
    ("s", [5, 2, 4, 1, 3], [10, 16, 6, 12, 5], None, None, 1.0, 0.5),
    ("z", [2, 1], [64, 36], None, None, 2.0, 0.0),
    ("d", [1, 3, 2], [1030, 9, 7], None, None, 1.0, 0.5),
]


def _guarded(host: np.ndarray):
    """Device buffer: canary | data | canary; returns (whole, data view offset)."""
    raw = np.frombuffer(host.tobytes(), dtype=np.uint8)
    whole = torch.empty(GUARD * 2 + raw.size, dtype=torch.uint8, device="cuda")
    whole.fill_(0xA5)
    whole[GUARD:GUARD + raw.size] = torch.from_numpy(raw.copy()).cuda()
    return whole


@pytest.mark.parametrize("case", range(len(CASES)))
def test_every_plan_stays_inside_its_buffers_and_is_repeatable(coracle, case):
    kind, perm, sizes, lda, ldb, alpha, beta = CASES[case]
    p = ttb.make_problem(perm, sizes, kind, kind, alpha, beta, lda, ldb)
    na = coracle.required_elements_a(sizes, lda)
    nb = coracle.required_elements_b(perm, sizes, ldb)
    A = np.zeros(na * COMPONENTS[kind_id(kind)], SCALAR[kind_id(kind)])
    B = np.zeros(nb * COMPONENTS[kind_id(kind)], SCALAR[kind_id(kind)])
    coracle.fill_sentinel(kind, A)
    coracle.fill_sentinel(kind, B)
    coracle.fill_uniform(kind, sizes, lda, 17, A)
    if beta != 0.0:
        coracle.fill_uniform(kind, b_sizes(perm, sizes), ldb, 18, B)
    want = B.copy()
    coracle.transpose(kind, kind, perm, sizes, lda, ldb, alpha, A, beta, want)
    plan = ttb.GpuPlan(p, cache=False)
    gA = _guarded(A)
    nbytes_b = B.nbytes
    for text in plan.candidates():
        plan.select(text)
        outs = []
        for _ in range(5):
            gB = _guarded(B)
            plan.execute(gA.data_ptr() + GUARD, gB.data_ptr() + GUARD)
            torch.cuda.synchronize()
            h = gB.cpu().numpy()
            assert (h[:GUARD] == 0xA5).all() and (h[GUARD + nbytes_b:] == 0xA5).all(), \
                ("write outside B", text)
            outs.append(h[GUARD:GUARD + nbytes_b].tobytes())
        ha = gA.cpu().numpy()
        assert (ha[:GUARD] == 0xA5).all() and (ha[GUARD + A.nbytes:] == 0xA5).all(), ("A canary", text)
        assert ha[GUARD:GUARD + A.nbytes].tobytes() == A.tobytes(), ("A written", text)
        assert all(o == outs[0] for o in outs), ("not repeatable", text)
        assert outs[0] == want.tobytes(), ("wrong bytes", text)

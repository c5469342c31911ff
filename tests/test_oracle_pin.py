"""Pin the plain-C oracle restatement to the reference (CPU only).

The reference sources are compiled in place into oracle/_ref (oracle/Makefile);
these tests skip when that build is absent (e.g. on the GPU box), where the
committed golden fixtures (tests/test_golden.py) pin the oracle instead.
"""
import numpy as np
import pytest

from oracle import COMPONENTS, SCALAR, kind_id
from problems import b_sizes, random_problem

PAIRS = [("s", "s"), ("d", "d"), ("c", "c"), ("z", "z"), ("s", "d"), ("d", "s"), ("c", "z"),
         ("z", "c")]


def _buffers(coracle, rng, ka, kb, perm, sizes, lda, ldb, integer=False):
    na = coracle.required_elements_a(sizes, lda)
    nb = coracle.required_elements_b(perm, sizes, ldb)
    ka_, kb_ = kind_id(ka), kind_id(kb)
    if integer:  # small positive integers (support.hpp:78-91)
        A = (rng.integers(1, 33, na * COMPONENTS[ka_])).astype(SCALAR[ka_])
        B = (rng.integers(1, 33, nb * COMPONENTS[kb_])).astype(SCALAR[kb_])
    else:
        A = rng.uniform(-1, 1, na * COMPONENTS[ka_]).astype(SCALAR[ka_])
        B = rng.uniform(-1, 1, nb * COMPONENTS[kb_]).astype(SCALAR[kb_])
    return A, B


def test_validate_messages_match_reference(coracle, refo):
    cases = [
        ([], [], None, None, "s", "s"),
        ([1, 1], [2, 2], None, None, "s", "s"),
        ([0, 1, 2], [2, 2, 2], None, None, "s", "s"),
        ([2, 1], [2], None, None, "s", "s"),
        ([2, 1], [2, 0], None, None, "s", "s"),
        ([2, 1], [4, 4], [3, 4], None, "s", "s"),
        ([2, 1], [4, 4], [4, 4], [4, 3], "s", "s"),
        ([2, 1], [4, 4], [4], None, "s", "s"),
        ([2, 1], [4, 4], None, [4, 4, 4], "s", "s"),
        ([2, 1], [4, 4], None, None, "d", "z"),
        ([2, 1], [4, 4], None, None, "s", "c"),
        ([2, 1], [1 << 40, 1 << 40], None, None, "s", "s"),
        # BASELINE c4s read literally: ldb (8,4096,3072) is rejected
        ([3, 2, 1], [4, 4096, 3072], [8, 4096, 3072], [8, 4096, 3072], "c", "c"),
        ([3, 2, 1], [4, 4096, 3072], [8, 4096, 3072], [3072, 4096, 8], "c", "c"),
    ]
    for perm, sizes, lda, ldb, ka, kb in cases:
        assert coracle.validate(perm, sizes, lda, ldb, ka, kb) == refo.validate(
            perm, sizes, lda, ldb, ka, kb), (perm, sizes, lda, ldb)
    assert coracle.validate([3, 2, 1], [4, 4096, 3072], [8, 4096, 3072], [8, 4096, 3072],
                            "c", "c") == "ldb[1] = 8 < size 3072"


def test_validate_random_matches_reference(coracle, refo):
    rng = np.random.default_rng(11)
    for _ in range(300):
        perm, sizes, lda, ldb = random_problem(rng, 5)
        # corrupt one field now and then
        r = rng.integers(0, 6)
        if r == 0:
            lda = [max(0, v - 2) for v in lda]
        elif r == 1:
            ldb = [max(0, v - 2) for v in ldb]
        elif r == 2:
            perm = [p if rng.integers(0, 4) else 1 for p in perm]
        ka, kb = PAIRS[rng.integers(0, len(PAIRS))]
        if rng.integers(0, 8) == 0:
            kb = "c" if ka in "sd" else "s"
        assert coracle.validate(perm, sizes, lda, ldb, ka, kb) == refo.validate(
            perm, sizes, lda, ldb, ka, kb)


def test_merge_matches_reference(coracle, refo):
    rng = np.random.default_rng(2024)
    for t in range(500):
        perm, sizes, lda, ldb = random_problem(rng, 6, allow_padding=(t % 2 == 0))
        assert coracle.merge(perm, sizes, lda, ldb) == refo.merge(perm, sizes, lda, ldb)


@pytest.mark.parametrize("ka,kb", PAIRS)
def test_odometer_matches_reference_transpose(coracle, refo, ka, kb):
    rng = np.random.default_rng(501 + kind_id(ka) * 7 + kind_id(kb))
    for t in range(40):
        perm, sizes, lda, ldb = random_problem(rng, 5)
        alpha, beta = [(1.0, 0.0), (2.0, 0.0), (2.0, 3.0), (0.7, 1.1), (1.3, 0.0), (0.5, 1.0)][t % 6]
        A, B0 = _buffers(coracle, rng, ka, kb, perm, sizes, lda, ldb, integer=(t % 3 == 0))
        want = B0.copy()
        refo.run(ka, kb, perm, sizes, lda, ldb, alpha, A, beta, want, threads=1 + t % 3)
        got = B0.copy()
        coracle.transpose(ka, kb, perm, sizes, lda, ldb, alpha, A, beta, got)
        assert got.tobytes() == want.tobytes(), (perm, sizes, lda, ldb, alpha, beta)
        # the reference test suite's own oracle agrees too (support.hpp:18-73)
        tsup = B0.copy()
        refo.run(ka, kb, perm, sizes, lda, ldb, alpha, A, beta, tsup, which=1)
        assert tsup.tobytes() == want.tobytes()
        nest = B0.copy()
        coracle.reference_nest(ka, kb, perm, sizes, lda, ldb, alpha, A, beta, nest,
                               threads=1 + t % 4)
        assert nest.tobytes() == want.tobytes()


def test_execute_plan_matches_odometer(coracle, refo):
    """The reference's tuned executor (execute_plan) agrees with the oracle."""
    rng = np.random.default_rng(9001)
    for t in range(30):
        perm, sizes, lda, ldb = random_problem(rng, 4, allow_ones=False)
        beta = 1.0 if t % 2 else 0.0
        A, B0 = _buffers(coracle, rng, "s", "s", perm, sizes, lda, ldb, integer=True)
        d = len(perm)
        order = ",".join(str(i) for i in range(1, d + 1))
        plan = f"order={order};bA=8;bB=8;d=0;ss=0;w=4"
        want = B0.copy()
        coracle.transpose("s", "s", perm, sizes, lda, ldb, 2.0, A, beta, want)
        got = B0.copy()
        refo.run("s", "s", perm, sizes, lda, ldb, 2.0, A, beta, got, which=2, plan=plan)
        assert got.tobytes() == want.tobytes()


def test_fill_is_shard_consistent(coracle):
    sizes, ld = [5, 7, 3], [6, 7, 4]
    g = np.zeros(6 * 7 * 4, np.float64)
    coracle.fill_uniform("d", sizes, ld, 9, g)
    # a sub-box generated alone with its global origin gives the same values
    sub_sizes, origin = [5, 3, 2], [0, 2, 1]
    s = np.zeros(5 * 3 * 2, np.float64)
    coracle.fill_uniform("d", sub_sizes, None, 9, s, origin=origin, global_sizes=sizes)
    gv = g.reshape(4, 7, 6)[1:3, 2:5, 0:5]
    assert np.array_equal(s.reshape(2, 3, 5), gv)
    assert np.all(s >= -1) and np.all(s < 1)
    # and checksums of the pieces add up to the checksum of the whole
    whole = coracle.checksum("d", sizes, ld, g)
    parts = 0
    for k in range(3):
        box = np.ascontiguousarray(g.reshape(4, 7, 6)[k, :, :5]).ravel()
        parts += coracle.checksum("d", [5, 7, 1], None, box, origin=[0, 0, k],
                                  global_sizes=sizes)
    assert parts % (1 << 64) == whole


def test_known_answers(coracle):
    # perm (2,1), sizes (2,2), A=[1,2,3,4] -> B=[1,3,2,4]
    A = np.array([1, 2, 3, 4], np.float32)
    B = np.zeros(4, np.float32)
    coracle.transpose("s", "s", [2, 1], [2, 2], None, None, 1.0, A, 0.0, B)
    assert B.tolist() == [1, 3, 2, 4]
    # alpha=0, beta=1 leaves B unchanged
    B2 = np.array([5, 6, 7, 8], np.float32)
    coracle.transpose("s", "s", [2, 1], [2, 2], None, None, 0.0, A, 1.0, B2)
    assert B2.tolist() == [5, 6, 7, 8]
    # geometry known answers (test_problem.cpp:42-64)
    assert coracle.required_elements_a([4, 5, 6]) == 120
    assert coracle.required_elements_a([4, 6], [5, 6]) == 1 + 3 * 1 + 5 * 5
    assert coracle.required_elements_b([2, 1], [4, 6], [8, 4]) == 1 + 5 * 1 + 3 * 8
    # merge known answers (test_problem.cpp:93-147)
    assert coracle.merge([3, 1, 2], [4, 5, 6])[:4] == ([2, 1], [4, 30], [4, 30], [30, 4])
    assert coracle.merge([1, 2, 3], [3, 4, 5])[1] == [60]
    assert len(coracle.merge([1, 2], [3, 4], [4, 4], [3, 4])[0]) == 2
    assert len(coracle.merge([1, 2], [3, 4], [3, 4], [4, 4])[0]) == 2
    assert coracle.merge([1, 2, 3], [3, 1, 4])[1] == [12]
    assert coracle.merge([1, 2], [1, 5])[1] == [5]
    assert coracle.merge([2, 1, 3], [3, 4, 1])[1] == [3, 4]
    assert coracle.merge([2, 1, 3], [1, 1, 1])[1] == [1]
    assert len(coracle.merge([1, 2], [1, 5], [2, 5], [1, 5])[0]) == 2


def test_merge_fixpoint_and_bytes(coracle):
    """acceptance.cpp:96-125 (C2): merging changes no bytes and is a fixpoint."""
    rng = np.random.default_rng(777)
    for t in range(200):
        perm, sizes, lda, ldb = random_problem(rng, 6)
        mp, ms, mla, mlb, trace = coracle.merge(perm, sizes, lda, ldb)
        assert coracle.merge(mp, ms, mla, mlb)[:4] == (mp, ms, mla, mlb)
        assert trace[0][0] == 1 and trace[-1][1] == len(perm)
        A, B0 = _buffers(coracle, rng, "s", "s", perm, sizes, lda, ldb, integer=True)
        w1, w2 = B0.copy(), B0.copy()
        coracle.transpose("s", "s", perm, sizes, lda, ldb, 2.0, A, 3.0, w1)
        coracle.transpose("s", "s", mp, ms, mla, mlb, 2.0, A, 3.0, w2)
        assert w1.tobytes() == w2.tobytes()

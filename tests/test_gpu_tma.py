"""GPU parity of the tensor-map tile (tma.cuh, plan text ``kern=tma``) against
the CPU oracle: bit-exact bytes of the whole B buffer (padding included,
support.hpp:93-96) for every kind pair, alpha/beta, case 1 and case 2,
partial tiles (zero-filled loads, clipped stores), padded outer sizes,
non-dense tile groups, folded carrier dims and every TMA candidate.
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

# (perm map, sizes, lda, ldb): strides that are multiples of 16 bytes for
# every kind (leading extents / pads multiples of 4)
CASES = [
    ([2, 1], [64, 48], None, None),
    ([2, 1], [132, 76], None, None),                          # partial tiles both sides
    ([2, 1], [36, 44], [40, 44], [48, 36]),                   # padded outer sizes
    ([3, 1, 2], [20, 12, 9], None, None),                     # Y group spans 2 axes
    ([3, 2, 1], [4, 40, 28], [8, 40, 28], [28, 40, 8]),       # c4s-like: X group not dense in A
    ([2, 4, 1, 3], [12, 8, 20, 5], None, None),               # carrier folds two axes
    ([5, 2, 4, 1, 3], [8, 6, 3, 12, 5], None, None),          # rank 5
    ([3, 5, 2, 6, 4, 1], [8, 5, 6, 3, 4, 4], None, None),     # rank 6 (c3-like)
    ([1, 3, 2], [8, 21, 13], None, None),                     # case 1: shared run of 8
    ([1, 4, 3, 2], [12, 5, 7, 9], [12, 6, 7, 9], [16, 9, 7, 6]),  # case 1, padded
    # B rows (23 / 57 elements) that end inside a 16-byte chunk, padded after:
    # a store clips them at 16-byte granularity, so no tile may be partial
    # along them (found by the random-problem parity test)
    ([3, 2, 1, 4], [45, 53, 23, 45], [45, 56, 23, 45], [24, 56, 45, 47]),
    ([3, 1, 2], [56, 57, 63], [56, 57, 65], [58, 63, 56]),
    ([2, 1], [64, 57], None, [58, 64]),
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


def _run(p, text, A, B):
    dA = torch.from_numpy(A.copy()).cuda()
    dB = torch.from_numpy(B.copy()).cuda()
    plan = ttb.GpuPlan(p, cache=False)
    plan.select(text)
    assert plan.describe().endswith("fn=tma"), plan.describe()
    plan.execute(dA, dB)
    torch.cuda.synchronize()
    return dB.cpu().numpy()


def _tma_texts(p):
    return [t for t in ttb.GpuPlan(p, cache=False).candidates() if t.startswith("kern=tma")]


@pytest.mark.parametrize("ka,kb", PAIRS)
def test_tma_every_candidate_bit_exact(coracle, ka, kb):
    rng = np.random.default_rng(900 + kind_id(ka) * 4 + kind_id(kb))
    n_run = 0
    for perm, sizes, lda, ldb in CASES:
        shared = perm[0] == 1
        if shared and ka != kb:
            continue
        for alpha, beta in [(1.0, 0.0), (1.3, 0.0), (0.7, 1.1), (0.0, 1.0)]:
            p = ttb.make_problem(perm, sizes, ka, kb, alpha, beta, lda, ldb)
            A, B = _inputs(coracle, rng, ka, kb, perm, sizes, lda, ldb, beta)
            want = B.copy()
            coracle.transpose(ka, kb, perm, sizes, lda, ldb, alpha, A, beta, want)
            texts = _tma_texts(p)
            for text in texts:
                got = _run(p, text, A, B)
                assert got.tobytes() == want.tobytes(), (perm, sizes, lda, ldb, alpha, beta, text)
                n_run += 1
    assert n_run > 0


@pytest.mark.parametrize("kind", ["s", "d", "c", "z"])
def test_tma_explicit_tiles(coracle, kind):
    """Hand-picked tile shapes: odd and even 16-byte row counts, tiles larger
    than the tensor on one side, a partial axis inside a two-axis group."""
    rng = np.random.default_rng(950 + kind_id(kind))
    perm, sizes = [3, 1, 2], [24, 20, 36]   # X = A0 (24), Y = A2 (36) then A0..
    for alpha, beta in [(1.0, 0.0), (0.5, -2.0)]:
        p = ttb.make_problem(perm, sizes, kind, kind, alpha, beta)
        A, B = _inputs(coracle, rng, kind, kind, perm, sizes, None, None, beta)
        want = B.copy()
        coracle.transpose(kind, kind, perm, sizes, None, None, alpha, A, beta, want)
        ran = 0
        for kx, ky, tx, ty, order, st in [(1, 1, 24, 36, 0, 2), (1, 1, 12, 20, 1, 3), (1, 1, 8, 8, 0, 4),
                                          (2, 1, 48, 36, 0, 2), (2, 1, 24 * 3, 12, 1, 2),
                                          (1, 2, 24, 36 * 2, 0, 2), (1, 1, 4, 4, 0, 2)]:
            text = f"kern=tma;kx={kx};ky={ky};tx={tx};ty={ty};order={order};occ=0;st={st}"
            plan = ttb.GpuPlan(p, cache=False)
            try:
                plan.select(text)
            except ValueError:
                continue
            got = _run(p, text, A, B)
            assert got.tobytes() == want.tobytes(), (kind, alpha, beta, text)
            ran += 1
        assert ran >= 3, kind


def test_tma_not_offered_for_misaligned_strides():
    # fp32 lead of 79 elements: A's second stride is 316 bytes (not a multiple of 16)
    p = ttb.make_problem([2, 1], [79, 64], "s", "s", 1.0, 0.0)
    plan = ttb.GpuPlan(p, cache=False)
    for t in plan.candidates():
        assert not t.startswith("kern=tma")
    with pytest.raises(ValueError, match="tma"):
        plan.select("kern=tma;kx=1;ky=1;tx=16;ty=16;order=0;occ=0;st=2")


BTILE_CASES = CASES + [
    ([2, 1], [516, 130], None, None),                 # B rows of 130: only A aligned (fp32)
    ([2, 1], [130, 516], None, None),                 # only B aligned
    ([3, 1, 2], [60, 7, 33], None, None),             # A lead 60, B lead 33
]


@pytest.mark.parametrize("ka,kb", PAIRS)
def test_bulk_tile_tensor_map_sides_bit_exact(coracle, ka, kb):
    """btile with the A tile and / or the B tile (beta != 0) arriving as one
    tensor-map box (plan key ts=1|2|3) while the other side keeps its bulk
    copies; every such candidate bit-exact."""
    rng = np.random.default_rng(970 + kind_id(ka) * 4 + kind_id(kb))
    n_run = 0
    for perm, sizes, lda, ldb in BTILE_CASES:
        if perm[0] == 1:
            continue
        for alpha, beta in [(1.0, 0.0), (0.7, 1.1)]:
            p = ttb.make_problem(perm, sizes, ka, kb, alpha, beta, lda, ldb)
            A, B = _inputs(coracle, rng, ka, kb, perm, sizes, lda, ldb, beta)
            want = B.copy()
            coracle.transpose(ka, kb, perm, sizes, lda, ldb, alpha, A, beta, want)
            for text in [t for t in ttb.GpuPlan(p, cache=False).candidates() if ";ts=" in t]:
                dA = torch.from_numpy(A.copy()).cuda()
                dB = torch.from_numpy(B.copy()).cuda()
                plan = ttb.GpuPlan(p, cache=False)
                plan.select(text)
                plan.execute(dA, dB)
                torch.cuda.synchronize()
                assert dB.cpu().numpy().tobytes() == want.tobytes(), (perm, sizes, alpha, beta, text)
                n_run += 1
    assert n_run > 0


# (perm map, sizes, lda, ldb): B columns that cover their whole group and
# continue into the next column (X's first axis is B's next position), with B
# rows that are not 16-byte multiples (c5_t14's shape in small)
WHOLE_COLUMN_CASES = [
    ([2, 1, 3], [256, 70, 5], None, None),        # B rows of 70 elements, A rows aligned
    ([2, 1, 3], [250, 67, 3], None, None),        # neither side aligned, partial tiles along X
    ([2, 1], [300, 131], None, None),             # 2D, odd B rows
]


@pytest.mark.parametrize("ka,kb", [("s", "s"), ("d", "d"), ("c", "c"), ("s", "d"), ("z", "c")])
def test_whole_column_tiles_offered_and_bit_exact(coracle, ka, kb):
    """beta != 0: tiles that span the whole Y group, whose B columns arrive as a
    few long bulk copies (plan.cpp whole-column candidates); every such
    candidate, with and without the A side by tensor map, bit-exact."""
    rng = np.random.default_rng(4100 + kind_id(ka) * 4 + kind_id(kb))
    n_run = 0
    for perm, sizes, lda, ldb in WHOLE_COLUMN_CASES:
        p = ttb.make_problem(perm, sizes, ka, kb, 0.7, 1.1, lda, ldb)
        A, B = _inputs(coracle, rng, ka, kb, perm, sizes, lda, ldb, 1.1)
        want = B.copy()
        coracle.transpose(ka, kb, perm, sizes, lda, ldb, 0.7, A, 1.1, want)
        ny = sizes[1]
        texts = [t for t in ttb.GpuPlan(p, cache=False).candidates()
                 if f";ty={ny};" in t and "vec=3" in t and "bp=1" in t]
        assert texts, (perm, sizes, ka, kb)
        for text in texts:
            dA = torch.from_numpy(A.copy()).cuda()
            dB = torch.from_numpy(B.copy()).cuda()
            plan = ttb.GpuPlan(p, cache=False)
            plan.select(text)
            plan.execute(dA, dB)
            torch.cuda.synchronize()
            assert dB.cpu().numpy().tobytes() == want.tobytes(), (perm, sizes, text)
            n_run += 1
    assert n_run >= len(WHOLE_COLUMN_CASES)

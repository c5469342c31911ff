"""Random problem generators for the parity tests (test infrastructure).

``random_problem`` follows the shape distribution of the reference's own
``tsup::random_problem`` (proj/tests/support.hpp:122-142): rank 1..max_rank,
extents 1..5 (or 2..5), and with probability 1/3 per index a leading
dimension padded by 1..3 on either tensor.
"""
import numpy as np


def random_perm(rng, d):
    p = list(range(1, d + 1))
    rng.shuffle(p)
    return p


def b_sizes(perm, sizes):
    sb = [0] * len(perm)
    for a, p in enumerate(perm):
        sb[p - 1] = sizes[a]
    return sb


def random_problem(rng, max_rank, allow_padding=True, allow_ones=True, lo=None, hi=None):
    d = int(rng.integers(1, max_rank + 1))
    if lo is None:
        lo, hi = (1, 5) if allow_ones else (2, 5)
    sizes = [int(rng.integers(lo, hi + 1)) for _ in range(d)]
    perm = random_perm(rng, d)
    lda = list(sizes)
    ldb = b_sizes(perm, sizes)
    if allow_padding:
        lda = [v + int(rng.integers(1, 4)) if rng.integers(0, 3) == 0 else v for v in lda]
        ldb = [v + int(rng.integers(1, 4)) if rng.integers(0, 3) == 0 else v for v in ldb]
    return perm, sizes, lda, ldb


def gather_to_scatter(gather):
    """BASELINE tuples are the paper's gather form (B index k = A index
    gather[k]); ttune's map is the 1-based scatter form."""
    m = [0] * len(gather)
    for k, a in enumerate(gather):
        m[a] = k + 1
    return m

#!/usr/bin/env python3
"""Run every candidate plan of one problem against the CPU oracle and report
the plans whose output differs (index of the first differing element, and
whether it lies in B's padding).  Debugging aid for the parity tests.

    python scripts/repro_plans.py KIND PERM SIZES [LDA] [LDB] ALPHA BETA
    e.g. python scripts/repro_plans.py d 3,2,1,4 45,53,23,45 45,56,23,45 24,56,45,47 0.7 1.1
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]


def main():
    import torch
    import paper_1603_02297_b200 as ttb
    from oracle import COMPONENTS, SCALAR, COracle, kind_id
    from problems import b_sizes
    kind = sys.argv[1]
    ints = lambda s: [int(x) for x in s.split(",")] if s != "-" else None  # noqa: E731
    perm, sizes, lda, ldb = ints(sys.argv[2]), ints(sys.argv[3]), ints(sys.argv[4]), ints(sys.argv[5])
    alpha, beta = float(sys.argv[6]), float(sys.argv[7])
    co = COracle()
    rng = np.random.default_rng(1)
    na, nb = co.required_elements_a(sizes, lda), co.required_elements_b(perm, sizes, ldb)
    A = np.zeros(na * COMPONENTS[kind_id(kind)], SCALAR[kind_id(kind)])
    B = np.zeros(nb * COMPONENTS[kind_id(kind)], SCALAR[kind_id(kind)])
    co.fill_sentinel(kind, A)
    co.fill_sentinel(kind, B)
    co.fill_uniform(kind, sizes, lda, 5, A)
    if beta != 0.0:
        co.fill_uniform(kind, b_sizes(perm, sizes), ldb, 6, B)
    want = B.copy()
    co.transpose(kind, kind, perm, sizes, lda, ldb, alpha, A, beta, want)
    p = ttb.make_problem(perm, sizes, kind, kind, alpha, beta, lda, ldb)
    plan = ttb.GpuPlan(p, cache=False)
    print("merged", ttb.merge_indices(p).problem.perm.map, ttb.merge_indices(p).problem.sizes)
    bad = 0
    for t in plan.candidates():
        plan.select(t)
        dA = torch.from_numpy(A.copy()).cuda()
        dB = torch.from_numpy(B.copy()).cuda()
        plan.execute(dA, dB)
        torch.cuda.synchronize()
        got = dB.cpu().numpy()
        diff = np.nonzero(got.view(np.uint8) != want.view(np.uint8))[0]
        if len(diff):
            bad += 1
            e = diff[0] // got.itemsize
            print(f"MISMATCH {plan.describe()}  first scalar {e}, {len(diff)} bytes differ; "
                  f"got {got[e]!r} want {want[e]!r}")
    print(f"{bad} of {len(plan.candidates())} plans differ")


if __name__ == "__main__":
    main()

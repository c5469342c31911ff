#!/usr/bin/env python3
"""Small problems through the asynchronous kernels, for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per run):

    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py

btile_kernel (bulk-copy ring with mbarriers, work-stealing counter and its
reset by the last CTA, column and linear walks, B through the ring and read
directly (bp=0), the big warp roles), tma_kernel (tensor-map loads / stores,
A and B rings, case 1 and 2, beta != 0) and copy_rows_kernel.  Every output
is checked against the CPU oracle, so a run is also a parity run; the exit
code is non-zero on a mismatch.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

CASES = [  # kind, perm map, sizes, alpha, beta, plan-text filters (substring per plan)
    ("s", [2, 1], [300, 260], 1.0, 0.0, ["vec=3", "vec=4", "kern=tma"]),
    ("s", [2, 1], [300, 260], 0.7, 1.1, ["vec=3;", "bp=0", "kern=tma"]),
    ("d", [3, 1, 2], [40, 21, 33], 1.0, 0.5, ["vec=3", "vec=4", "kern=tma"]),
    ("c", [3, 2, 1], [4, 96, 70], 1.0, 0.0, ["vec=3", "kern=tma"]),
    ("s", [1, 3, 2], [48, 30, 17], 1.0, 0.5, ["vec=3", "kern=tma", "kern=copy"]),
    ("s", [5, 2, 4, 1, 3], [10, 16, 6, 12, 5], 1.0, 0.5, ["xp=1", "vec=4"]),
    ("s", [2, 1], [1100, 900], 1.3, 0.0, ["vec=3"]),   # 32-64 KB tiles: big warp roles
    ("d", [1, 3, 2], [1030, 9, 7], 1.0, 0.5, ["fn=copy_rows", "order=2", "order=4"]),
]


def main():
    import torch
    import paper_1603_02297_b200 as ttb
    from oracle import COMPONENTS, SCALAR, COracle, kind_id
    from problems import b_sizes
    co = COracle()
    bad = runs = 0
    for kind, perm, sizes, alpha, beta, filters in CASES:
        p = ttb.make_problem(perm, sizes, kind, kind, alpha, beta)
        na, nb = ttb.required_elements_a(p), ttb.required_elements_b(p)
        A = np.zeros(na * COMPONENTS[kind_id(kind)], SCALAR[kind_id(kind)])
        B = np.zeros(nb * COMPONENTS[kind_id(kind)], SCALAR[kind_id(kind)])
        co.fill_uniform(kind, sizes, None, 3, A)
        if beta != 0.0:
            co.fill_uniform(kind, b_sizes(perm, sizes), None, 4, B)
        want = B.copy()
        co.transpose(kind, kind, perm, sizes, None, None, alpha, A, beta, want)
        plan = ttb.GpuPlan(p, cache=False)
        texts = plan.candidates()
        chosen = []
        for f in filters:
            chosen += [t for t in texts if f in t][:2]
        for t in dict.fromkeys(chosen):
            plan.select(t)
            dA = torch.from_numpy(A).cuda()
            dB = torch.from_numpy(B.copy()).cuda()
            for _ in range(3):  # the counter slot is reused: reset by the last CTA each time
                dB.copy_(torch.from_numpy(B))
                plan.execute(dA, dB)
            torch.cuda.synchronize()
            ok = dB.cpu().numpy().tobytes() == want.tobytes()
            runs += 1
            bad += not ok
            print(f"{'ok ' if ok else 'BAD'} {kind} {perm} {sizes} {plan.describe()}", flush=True)
    print(f"{runs} plan runs, {bad} mismatches")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())

#!/usr/bin/env python3
"""Randomised parity stress beyond the fixed seeds of tests/: medium problems
(rank 2-5, extents lo..hi, padded outer sizes) through EVERY candidate plan of
the planner, bit for bit against the CPU oracle (test infrastructure as the
checker).

    python scripts/stress_parity.py --seed 1 --count 40 [--lo 9 --hi 130] [--kinds ss,dd,cc,sd]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    sys.path.insert(0, p)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--count", type=int, default=40)
    ap.add_argument("--lo", type=int, default=9)
    ap.add_argument("--hi", type=int, default=130)
    ap.add_argument("--max-elems", type=int, default=3_000_000)
    ap.add_argument("--kinds", default="ss,dd,cc,zz,sd,zc")
    args = ap.parse_args()

    import numpy as np
    import torch
    import paper_1603_02297_b200 as ttb
    from oracle import COMPONENTS, SCALAR, COracle, kind_id
    from problems import b_sizes, random_problem

    co = COracle()
    rng = np.random.default_rng(args.seed)
    pairs = [(k[0], k[1]) for k in args.kinds.split(",")]
    n_plans = n_prob = 0
    fams = {}
    t0 = time.time()
    while n_prob < args.count:
        perm, sizes, lda, ldb = random_problem(rng, 5, allow_padding=bool(rng.integers(0, 2)),
                                               allow_ones=False, lo=args.lo, hi=args.hi)
        if len(sizes) < 2 or int(np.prod(lda)) > args.max_elems or int(np.prod(ldb)) > args.max_elems:
            continue
        ka, kb = pairs[int(rng.integers(len(pairs)))]
        alpha, beta = [(1.0, 0.0), (1.3, 0.0), (0.7, 1.1), (1.0, 0.5)][int(rng.integers(4))]
        na = co.required_elements_a(sizes, lda)
        nb = co.required_elements_b(perm, sizes, ldb)
        A = np.zeros(na * COMPONENTS[kind_id(ka)], SCALAR[kind_id(ka)])
        B = np.zeros(nb * COMPONENTS[kind_id(kb)], SCALAR[kind_id(kb)])
        co.fill_sentinel(ka, A)
        co.fill_sentinel(kb, B)
        co.fill_uniform(ka, sizes, lda, int(rng.integers(1 << 30)), A)
        if beta != 0.0:
            co.fill_uniform(kb, b_sizes(perm, sizes), ldb, int(rng.integers(1 << 30)), B)
        want = B.copy()
        co.transpose(ka, kb, perm, sizes, lda, ldb, alpha, A, beta, want)
        p = ttb.make_problem(perm, sizes, ka, kb, alpha, beta, lda, ldb)
        dA = torch.from_numpy(A).cuda()
        plan = ttb.GpuPlan(p, cache=False)
        for text in plan.candidates():
            dB = torch.from_numpy(B.copy()).cuda()
            plan.select(text)
            plan.execute(dA, dB)
            torch.cuda.synchronize()
            if dB.cpu().numpy().tobytes() != want.tobytes():
                print("MISMATCH", ka, kb, perm, sizes, lda, ldb, alpha, beta, text, flush=True)
                return 1
            fn = plan.describe().split("fn=")[-1].split(";")[0]
            fams[fn] = fams.get(fn, 0) + 1
            n_plans += 1
        n_prob += 1
    print(f"seed {args.seed}: {n_prob} problems, {n_plans} plans bit-exact in {time.time() - t0:.0f}s; "
          f"by kernel {dict(sorted(fams.items()))}", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())

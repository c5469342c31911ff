#!/usr/bin/env python3
"""The paper's benchmark suite on the GPU (run_benchmark,
benchmark.cpp:222-256, write_benchmark_csv 272-285).

    python scripts/suite.py [--volume-mib 200] [--kind s] [--seed 42] [--ref]
                            [--verify] [--cache FILE] [--csv OUT]

For each of the 57 cases (build_benchmark, alpha = beta = 1): device buffers
filled by the counter generator, the engine's plan autotuned (or taken from /
stored to a solution cache with --cache), then the best of R event-timed
executions.  tunedGiBs uses the reference's formula (tuner.cpp:18-25, 2^30).
refGiBs is the reference's own nest (reference_transpose, oracle/_ref) on all
host cores when --ref is given (else empty); speedup = tuned / ref as in the
reference's CSV.  --verify compares a u64 checksum of every GPU output with
the CPU oracle's (oracle/, test infrastructure) on the same inputs.
"""
import argparse
import csv
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--volume-mib", type=int, default=200)
    ap.add_argument("--kind", default="s")
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--ref", action="store_true", help="time the reference nest on host cores")
    ap.add_argument("--verify", action="store_true", help="checksum every output vs the oracle")
    ap.add_argument("--cache", default=None, help="solution cache file (tune_cached)")
    ap.add_argument("--csv", default=None)
    ap.add_argument("--no-tune", action="store_true",
                    help="time the planner's heuristic first choice (the one-shot API's plan)")
    args = ap.parse_args()

    import numpy as np
    import torch
    import paper_1603_02297_b200 as ttb

    cases = ttb.build_benchmark(args.volume_mib << 20, args.kind, args.seed)
    ref = co = None
    if args.ref:
        from oracle import RefOracle, RefSession
        ref = RefOracle()
    if args.verify:
        from oracle import COMPONENTS, SCALAR, COracle, kind_id
        co = COracle()
    threads = os.cpu_count() or 1
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    rows = []
    for i, c in enumerate(cases):
        p = c.problem
        k = p.kind_a.code
        na, nb = ttb.required_elements_a(p), ttb.required_elements_b(p)
        a, b = ttb.TensorBuffer(k, na), ttb.TensorBuffer(k, nb)
        sb = ttb.sizes_b(p)
        ttb.fill_uniform(k, p.sizes, None, 2 * i + 1, a.data_ptr())
        ttb.fill_uniform(k, sb, None, 2 * i + 2, b.data_ptr())
        plan = ttb.GpuPlan(p, cache=False)
        if args.no_tune:
            plan.execute(a, b)
        elif args.cache:
            plan.tune_cached(a, b, args.cache)
        else:
            plan.autotune(a, b)
        ck_gpu = ttb.checksum(k, sb, None, b.data_ptr()) if args.verify else None
        best = math.inf
        for _ in range(args.reps):
            e0.record()
            plan.execute(a, b)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
        nbytes = p.total_elements() * (p.kind_a.bytes + 2 * p.kind_b.bytes)  # beta != 0
        tuned = nbytes / 2 ** 30 / best
        del a, b
        torch.cuda.empty_cache()
        ok = ""
        if args.verify:
            # the oracle on the same inputs: B0 = gen(seed_b), one application
            A = np.zeros(na * COMPONENTS[kind_id(k)], SCALAR[kind_id(k)])
            B = np.zeros(nb * COMPONENTS[kind_id(k)], SCALAR[kind_id(k)])
            co.fill_uniform(k, p.sizes, None, 2 * i + 1, A)
            co.fill_uniform(k, sb, None, 2 * i + 2, B)
            co.transpose(k, k, p.perm.map, p.sizes, None, None, 1.0, A, 1.0, B)
            ok = "ok" if co.checksum(k, sb, None, B) == ck_gpu else "MISMATCH"
        refg = ""
        if ref is not None:
            s = RefSession(ref, k, k, p.perm.map, p.sizes, alpha=1.0, beta=1.0)
            s.run(threads)
            t = min(s.run(threads) for _ in range(3))
            s.close()
            refg = nbytes / 2 ** 30 / t
        row = {"caseId": c.id, "dim": p.rank(), "perm": "-".join(map(str, p.perm.map)),
               "sizes": "x".join(map(str, p.sizes)), "category": c.category,
               "config": c.config, "refGiBs": f"{refg:.6g}" if refg != "" else "",
               "tunedGiBs": f"{tuned:.6g}",
               "speedup": f"{tuned / refg:.6g}" if refg != "" else "",
               "plan": plan.describe()}
        rows.append(dict(row, _ok=ok))
        print(f"{c.id:24s} {tuned * 1.073741824:8.1f} GB/s  ref {row['refGiBs']:>8s} GiB/s  "
              f"{ok} {row['plan']}", flush=True)
    fields = ["caseId", "dim", "perm", "sizes", "category", "config", "refGiBs", "tunedGiBs",
              "speedup", "plan"]
    if args.csv:
        with open(args.csv, "w", newline="") as f:
            w = csv.DictWriter(f, fieldnames=fields, extrasaction="ignore")
            w.writeheader()
            w.writerows(rows)
    g = [float(r["tunedGiBs"]) for r in rows]
    print(f"# {len(rows)} cases: tuned GB/s geo-mean {math.exp(sum(map(math.log, g)) / len(g)) * 1.073741824:.1f}, "
          f"min {min(g) * 1.073741824:.1f}, max {max(g) * 1.073741824:.1f}")
    if args.ref:
        s = [float(r["speedup"]) for r in rows]
        print(f"# speedup vs reference nest on {threads} host threads: geo-mean "
              f"{math.exp(sum(map(math.log, s)) / len(s)):.1f}x")
    if args.verify:
        bad = [r["caseId"] for r in rows if r.get("_ok") != "ok"]
        print("# verify: all outputs match the oracle" if not bad else f"# verify MISMATCH: {bad}")
        if bad:
            sys.exit(1)


if __name__ == "__main__":
    main()

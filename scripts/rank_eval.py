#!/usr/bin/env python3
"""Score the planner's heuristic ranking against measured candidate times.

    python scripts/rank_eval.py DIR    # DIR holds cands_<case>.log from scripts/run_case.py <case>

For every workload: the measured rate of the planner's current first choice
(host-only ttb_debug_candidates) against the best measured candidate, and
where the best one ranks.  Host only: re-run after editing the cost model.
"""
import glob
import math
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_1603_02297_b200 as ttb
    from paper_1603_02297_b200.workloads import BY_NAME

    d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
    verbose = "-v" in sys.argv
    ratios = []
    for path in sorted(glob.glob(os.path.join(d, "cands_*.log"))):
        name = os.path.basename(path)[len("cands_"):-len(".log")]
        w = BY_NAME[name]
        meas = {}
        for line in open(path):
            m = re.match(r"\s*([\d.]+) us\s+([\d.]+) GB/s\s+(\S+)", line)
            if m:
                meas[m.group(3)] = float(m.group(2))
        if not meas:
            continue
        p = ttb.make_problem(w.perm, list(w.sizes), w.kind, w.kind, w.alpha, w.beta,
                             w.lda and list(w.lda), w.ldb and list(w.ldb))
        cands = ttb.debug_candidates(p)
        best_t, best = max(meas.items(), key=lambda kv: kv[1])
        first = next((c for c in cands if c in meas), None)
        rank_best = cands.index(best_t) if best_t in cands else -1
        unmeasured_first = cands[0] not in meas
        r = meas[first] / best if first else float("nan")
        ratios.append(r)
        print(f"{name:8s} first {meas.get(first, 0):7.1f} / best {best:7.1f} = {100 * r:5.1f}%"
              f"{' (first unmeasured: ' + cands[0] + ')' if unmeasured_first else ''}  best ranks #{rank_best}"
              f"  F: {first}  B: {best_t}")
        if verbose:
            for i, c in enumerate(cands[:8]):
                print(f"      #{i} {meas.get(c, float('nan')):7.1f} {c}")
    g = math.exp(sum(math.log(r) for r in ratios) / len(ratios))
    print(f"# first / best: geo-mean {100 * g:.1f}%, worst {100 * min(ratios):.1f}%, {len(ratios)} workloads")


if __name__ == "__main__":
    main()

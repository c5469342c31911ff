#!/usr/bin/env python3
"""How far the planner's heuristic first choice is from the autotuned plan, per
BASELINE workload (the one-shot ttb_transpose path runs the heuristic choice).

    python scripts/heuristic_gap.py [case ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1603_02297_b200 as ttb
    from paper_1603_02297_b200.workloads import BY_NAME, C5, CONFIGS

    names = sys.argv[1:] or [w.name for w in list(CONFIGS) + list(C5)]
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)

    def best_of(plan, a, b, n=6):
        t = 1e30
        for _ in range(n):
            e0.record()
            plan.execute(a, b)
            e1.record()
            e1.synchronize()
            t = min(t, e0.elapsed_time(e1))
        return t

    ratios = []
    for name in names:
        w = BY_NAME[name]
        p = ttb.make_problem(w.perm, list(w.sizes), w.kind, w.kind, w.alpha, w.beta,
                             w.lda and list(w.lda), w.ldb and list(w.ldb))
        a = ttb.TensorBuffer(w.kind, ttb.required_elements_a(p))
        b = ttb.TensorBuffer(w.kind, ttb.required_elements_b(p))
        ttb.fill_uniform(w.kind, list(w.sizes), w.lda and list(w.lda), w.seed_a, a.data_ptr())
        plan = ttb.GpuPlan(p, cache=False)
        first = plan.describe()
        plan.execute(a, b)
        t_h = best_of(plan, a, b)
        plan.autotune(a, b, warmups=2, reps=6)
        t_t = best_of(plan, a, b)
        gb = w.algorithmic_bytes / 1e9
        ratios.append(t_t / t_h)
        print(f"{name:8s} heuristic {gb / t_h * 1e3:7.1f} GB/s  tuned {gb / t_t * 1e3:7.1f} GB/s  "
              f"{100 * t_t / t_h:5.1f}%  H: {first}  T: {plan.describe()}", flush=True)
        del a, b, plan
        torch.cuda.empty_cache()
    import math
    print(f"# heuristic / tuned geo-mean {100 * math.exp(sum(math.log(r) for r in ratios) / len(ratios)):.1f}%, "
          f"worst {100 * min(ratios):.1f}%")


if __name__ == "__main__":
    main()

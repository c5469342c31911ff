"""Run-to-run spread of one plan (kernel-design probe): event times of N
back-to-back executions, and of N executions interleaved with another row."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1603_02297_b200 as ttb  # noqa: E402
from paper_1603_02297_b200.workloads import BY_NAME  # noqa: E402


def setup(name, plan_text):
    w = BY_NAME[name]
    p = ttb.make_problem(w.perm, list(w.sizes), w.kind, w.kind, w.alpha, w.beta)
    a = ttb.TensorBuffer(w.kind, ttb.required_elements_a(p))
    b = ttb.TensorBuffer(w.kind, ttb.required_elements_b(p))
    ttb.fill_uniform(w.kind, list(w.sizes), None, w.seed_a, a.data_ptr())
    plan = ttb.GpuPlan(p, cache=False)
    plan.select(plan_text)
    return w, plan, a, b


def times(runs, n):
    e = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(n)]
    for i in range(n):
        for k, (w, plan, a, b) in enumerate(runs):
            if k == 0:
                e[i][0].record()
            plan.execute(a, b)
            if k == 0:
                e[i][1].record()
    torch.cuda.synchronize()
    w = runs[0][0]
    return [round(w.algorithmic_bytes / 1e9 / (x.elapsed_time(y) / 1e3)) for x, y in e]


main = setup(sys.argv[1], sys.argv[2])
other = setup(sys.argv[3], sys.argv[4]) if len(sys.argv) > 4 else None
print("alone      ", times([main], 12), flush=True)
if other:
    print("interleaved", times([main, other], 12), flush=True)

import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_1603_02297_b200 as ttb
from paper_1603_02297_b200.workloads import BY_NAME
def setup(name):
    w = BY_NAME[name]
    p = ttb.make_problem(w.perm, list(w.sizes), w.kind, w.kind, w.alpha, w.beta)
    na, nb = ttb.required_elements_a(p), ttb.required_elements_b(p)
    a, b = ttb.TensorBuffer(w.kind, na), ttb.TensorBuffer(w.kind, nb)
    ttb.fill_uniform(w.kind, list(w.sizes), None, w.seed_a, a.data_ptr())
    return w, p, a, b
def t(plan, a, b, n=5):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(n):
        e0.record(); plan.execute(a, b); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
cases = [("c5_t08", "kern=smem;kx=2;ky=2;tx=64;ty=66;order=0;occ=0;st=2;bp=1;vec=1"),
         ("c5_t18", "kern=smem;kx=2;ky=1;tx=80;ty=36;order=0;occ=0;st=2;bp=0;vec=1"),
         ("c5_t20", "kern=smem;kx=2;ky=1;tx=64;ty=76;order=0;occ=0;st=2;bp=1;vec=1")]
bufs = []
for name, text in cases:
    w, p, a, b = setup(name)
    plan = ttb.GpuPlan(p, cache=False); plan.select(text)
    bufs.append((name, w, plan, a, b))
def report(tag):
    for name, w, plan, a, b in bufs:
        ms = t(plan, a, b)
        print(f"{tag:10s} {name} {w.algorithmic_bytes/1e9/(ms/1e3):7.1f} GB/s", flush=True)
report("alone")
dummy = torch.empty(int(70e9), dtype=torch.uint8, device="cuda")
report("+70GB")
# back-to-back: each row right after the previous one, timed per row
e = [torch.cuda.Event(True) for _ in range(len(bufs) + 1)]
for rep in range(3):
    e[0].record()
    for i, (name, w, plan, a, b) in enumerate(bufs):
        plan.execute(a, b); e[i + 1].record()
    e[-1].synchronize()
for i, (name, w, plan, a, b) in enumerate(bufs):
    ms = e[i].elapsed_time(e[i + 1])
    print(f"chained    {name} {w.algorithmic_bytes/1e9/(ms/1e3):7.1f} GB/s")

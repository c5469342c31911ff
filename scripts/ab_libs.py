#!/usr/bin/env python3
"""Interleaved A/B timing of several libttb builds on one problem and plan.

    python scripts/ab_libs.py c5_t00 "kern=smem;..." lib1.so lib2.so [--rounds 5]

Every library is loaded side by side (separate ctypes handles, one CUDA
context); rounds alternate between them so clock/thermal drift hits all
equally.  Prints the median device time per library.
"""
import argparse
import ctypes as C
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case")
    ap.add_argument("plan")
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--rounds", type=int, default=7)
    ap.add_argument("--iters", type=int, default=5)
    args = ap.parse_args()
    import torch
    import paper_1603_02297_b200 as ttb
    from paper_1603_02297_b200.workloads import BY_NAME
    w = BY_NAME[args.case]
    p = ttb.make_problem(w.perm, list(w.sizes), w.kind, w.kind, w.alpha, w.beta,
                         w.lda and list(w.lda), w.ldb and list(w.ldb))
    na, nb = ttb.required_elements_a(p), ttb.required_elements_b(p)
    a, b = ttb.TensorBuffer(w.kind, na), ttb.TensorBuffer(w.kind, nb)
    ttb.fill_uniform(w.kind, list(w.sizes), w.lda and list(w.lda), w.seed_a, a.data_ptr())
    handles = []
    for path in args.libs:
        L = C.CDLL(os.path.abspath(path))
        L.ttb_plan_create.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int,
                                      C.POINTER(C.c_int), C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_double,
                                      C.c_double, C.c_int]
        L.ttb_plan_select.argtypes = [C.c_void_p, C.c_char_p]
        L.ttb_plan_execute.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        h = C.c_void_p()
        rc = L.ttb_plan_create(C.byref(h), *p._args(), p.alpha, p.beta, 1)
        assert rc == 0, rc
        assert L.ttb_plan_select(h, args.plan.encode()) == 0, "plan not applicable"
        handles.append((path, L, h))
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    times = {path: [] for path, _, _ in handles}
    for _ in range(args.rounds):
        for path, L, h in handles:
            L.ttb_plan_execute(h, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), stream)
            best = 1e30
            for _ in range(args.iters):
                e0.record()
                L.ttb_plan_execute(h, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), stream)
                e1.record()
                e1.synchronize()
                best = min(best, e0.elapsed_time(e1))
            times[path].append(best)
    for path, ts in times.items():
        med = statistics.median(ts)
        print(f"{os.path.basename(path):20s} median {med * 1e3:9.1f} us "
              f"{w.algorithmic_bytes / 1e9 / (med / 1e3):8.1f} GB/s  spread "
              f"{(max(ts) - min(ts)) / med * 100:4.1f}%  {args.case} {args.plan}")


if __name__ == "__main__":
    main()

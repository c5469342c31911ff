#!/usr/bin/env python3
"""Probe: cudaLimitMaxL2FetchGranularity (32 / 64 / 128 bytes) on c4s, whose A rows use
32 bytes of every 64 (DRAM over-fetch bound).

    python scripts/l2fetch_probe.py [case ...]
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1603_02297_b200 as ttb
    from paper_1603_02297_b200.workloads import BY_NAME

    torch.cuda.init()
    rt = C.CDLL("libcudart.so")
    LIMIT = 0x05  # cudaLimitMaxL2FetchGranularity
    names = sys.argv[1:] or ["c4s", "c4", "c1"]
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    for name in names:
        w = BY_NAME[name]
        p = ttb.make_problem(w.perm, list(w.sizes), w.kind, w.kind, w.alpha, w.beta,
                             w.lda and list(w.lda), w.ldb and list(w.ldb))
        a = ttb.TensorBuffer(w.kind, ttb.required_elements_a(p))
        b = ttb.TensorBuffer(w.kind, ttb.required_elements_b(p))
        ttb.fill_uniform(w.kind, list(w.sizes), w.lda and list(w.lda), w.seed_a, a.data_ptr())
        plan = ttb.GpuPlan(p, cache=False)
        plan.autotune(a, b, warmups=2, reps=6)
        for gran in (64, 32, 128, 64):
            rc = rt.cudaDeviceSetLimit(LIMIT, C.c_size_t(gran))
            got = C.c_size_t(0)
            rt.cudaDeviceGetLimit(C.byref(got), LIMIT)
            for _ in range(3):
                plan.execute(a, b)
            best = 1e30
            for _ in range(10):
                e0.record()
                plan.execute(a, b)
                e1.record()
                e1.synchronize()
                best = min(best, e0.elapsed_time(e1))
            print(f"{name} granularity set {gran} (rc {rc}, now {got.value}): {best * 1e3:.1f} us "
                  f"{w.algorithmic_bytes / 1e9 / (best / 1e3):.1f} GB/s  {plan.describe()}", flush=True)


if __name__ == "__main__":
    main()

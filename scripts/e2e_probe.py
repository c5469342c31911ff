"""Probe the end-to-end host path: raw PCIe copy ceilings (H2D, D2H, both at
once) and, per sweep row, execute_host time for the staged and the overlapped
paths.  Usage: python scripts/e2e_probe.py [row ...]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1603_02297_b200 as ttb  # noqa: E402
from paper_1603_02297_b200.workloads import BY_NAME  # noqa: E402


def pcie_ceilings(nbytes=1 << 30):
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    for name in ("h2d", "d2h", "both"):
        for it in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if name in ("h2d", "both"):
                with torch.cuda.stream(s1):
                    d.copy_(h, non_blocking=True)
            if name in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    h2.copy_(d2, non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        out[name] = round(nbytes * (2 if name == "both" else 1) / dt / 1e9, 1)
    print("pcie GB/s", out, flush=True)


def row(name):
    w = BY_NAME[name]
    q = ttb.make_problem(w.perm, list(w.sizes), w.kind, w.kind, w.alpha, w.beta)
    sz = 8 if w.kind in "dz" else 4
    na, nb = ttb.required_elements_a(q), ttb.required_elements_b(q)
    ha = torch.empty(na * sz, dtype=torch.uint8, pin_memory=True)
    hb = torch.empty(nb * sz, dtype=torch.uint8, pin_memory=True)
    plan = ttb.GpuPlan(q)
    res = {}
    for path in os.environ.get("PROBE_PATHS", "staged,overlap").split(","):
        os.environ["TTB_HOST_PATH"] = path
        plan.execute_host(ha, hb)
        t0 = time.perf_counter()
        for _ in range(2):
            plan.execute_host(ha, hb)
        res[path] = round(w.algorithmic_bytes / 1e9 / ((time.perf_counter() - t0) / 2), 1)
    print(name, "beta", w.beta, plan.describe().split(";fn=")[-1], res, flush=True)


if __name__ == "__main__":
    if not os.environ.get("PROBE_NO_PCIE"):
        pcie_ceilings()
    for n in sys.argv[1:] or [f"c5_t{t:02d}" for t in range(24)]:
        row(n)

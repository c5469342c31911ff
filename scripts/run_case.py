#!/usr/bin/env python3
"""Time one BASELINE workload (config or c5 row) under every candidate plan, or
under one given plan -- the driver for kernel tuning and ncu captures.

    python scripts/run_case.py c5_t00 [--plan TEXT] [--iters 20] [--check]

Prints one line per plan: device time (CUDA events, best of iters) and GB/s
(tuner.cpp:18-25 byte count).  --check compares the output checksum with the
reference's golden checksum (tests/golden/config_checksums.json).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case")
    ap.add_argument("--plan", default=None)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--top", type=int, default=0, help="only the first N candidates")
    ap.add_argument("--filter", default=None, help="only candidates containing this text")
    ap.add_argument("--extra", action="append", default=[], help="additional plan texts")
    ap.add_argument("--kinds", default=None, help="override the kind pair, e.g. sd or cz")
    ap.add_argument("--beta", type=float, default=None, help="override beta (probe: the same shape without / with the B read)")
    args = ap.parse_args()

    import torch
    import paper_1603_02297_b200 as ttb
    from paper_1603_02297_b200.workloads import BY_NAME

    w = BY_NAME[args.case]
    if args.beta is not None:
        import dataclasses
        w = dataclasses.replace(w, beta=args.beta)
    ka, kb = (args.kinds[0], args.kinds[1]) if args.kinds else (w.kind, w.kind)
    from paper_1603_02297_b200.workloads import KIND_BYTES
    nbytes = w.elements * (KIND_BYTES[ka] + KIND_BYTES[kb] * (2 if w.beta != 0.0 else 1))
    p = ttb.make_problem(w.perm, list(w.sizes), ka, kb, w.alpha, w.beta,
                         w.lda and list(w.lda), w.ldb and list(w.ldb))
    na, nb = ttb.required_elements_a(p), ttb.required_elements_b(p)
    a, b = ttb.TensorBuffer(ka, na), ttb.TensorBuffer(kb, nb)
    ttb.fill_sentinel(ka, na, a.data_ptr())
    ttb.fill_uniform(ka, list(w.sizes), w.lda and list(w.lda), w.seed_a, a.data_ptr())
    plan = ttb.GpuPlan(p, cache=False)
    texts = [args.plan] if args.plan else plan.candidates()
    if args.filter:
        texts = [t for t in texts if args.filter in t]
    if args.top:
        texts = texts[:args.top]
    texts = texts + args.extra
    golden = None
    if args.check:
        with open(os.path.join(ROOT, "tests", "golden", "config_checksums.json")) as f:
            golden = int(json.load(f)[w.name]["checksum"])
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    merged = ttb.merge_indices(p).problem
    print(f"# {w.name} kind={w.kind} merged perm={merged.perm.map} sizes={merged.sizes} "
          f"bytes={nbytes} kinds={ka}{kb}", flush=True)
    for t in texts:
        try:
            plan.select(t)
        except Exception as e:  # a hand-written plan text that does not apply
            print(f"   skip {t}: {e}", flush=True)
            continue
        if w.beta != 0.0:
            ttb.fill_uniform(kb, w.sizes_b, w.ldb and list(w.ldb), w.seed_b, b.data_ptr())
        plan.execute(a, b)
        ok = ""
        if golden is not None and not args.kinds:
            ck = ttb.checksum(w.kind, w.sizes_b, w.ldb and list(w.ldb), b.data_ptr())
            ok = " ok" if ck == golden else " MISMATCH"
        best = 1e30
        for _ in range(args.iters):
            e0.record()
            plan.execute(a, b)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"{best * 1e3:9.1f} us {nbytes / 1e9 / (best / 1e3):8.1f} GB/s  {t}{ok}",
              flush=True)


if __name__ == "__main__":
    main()

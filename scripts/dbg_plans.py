#!/usr/bin/env python3
"""Run every candidate plan of the golden small cases on the GPU and report the
plans that fail to launch or mismatch (debug aid for new kernel variants)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    sys.path.insert(0, p)

from golden_util import case_inputs, load_small_cases  # noqa: E402
from oracle import COracle  # noqa: E402
from test_gpu_parity import all_plans, run_gpu  # noqa: E402


def main():
    only = sys.argv[1] if len(sys.argv) > 1 else ""
    co = COracle()
    meta, arrays = load_small_cases()
    bad = n = 0
    for case in meta:
        A, B = case_inputs(co, case, arrays)
        want = arrays[f"out{case['id']}"]
        args = (case["kind_a"], case["kind_b"], case["perm"], case["sizes"], case["lda"], case["ldb"])
        for text in all_plans(*args, case["alpha"], case["beta"]):
            if only not in text:
                continue
            n += 1
            try:
                got = run_gpu(*args, case["alpha"], A, case["beta"], B, plan_text=text)
                if got.tobytes() != want.tobytes():
                    bad += 1
                    print("MISMATCH", case["id"], args, case["alpha"], case["beta"], text)
            except Exception as e:  # noqa: BLE001
                bad += 1
                print("ERROR", case["id"], args, case["alpha"], case["beta"], text, e)
    print(f"{n} plans, {bad} bad")


if __name__ == "__main__":
    main()

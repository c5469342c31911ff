#!/usr/bin/env python3
"""Predicted multi-GPU sweep throughput from one GPU: every rank's share of
every c5 row (bench.py's Row: its boxes on bounding-box buffers, autotuned),
timed alone on this device.  Ranks of an 8-GPU box run independently (no
collective on the data path), so the job's step time is the slowest rank's
sum over rows.  This measures the partition (imbalance, sub-box plans), not
NVLink, and is not a multi-GPU measurement.

    python scripts/predict_scaling.py [--worlds 1,2,4,8] [--reps 3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--rows", default=None, help="comma-separated row names (default: all c5)")
    args = ap.parse_args()
    import torch
    import bench
    import paper_1603_02297_b200 as ttb
    from paper_1603_02297_b200.workloads import C5
    rows = [w for w in C5 if not args.rows or w.name in args.rows.split(",")]
    total = sum(w.algorithmic_bytes for w in rows)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    out = {}
    for world in [int(x) for x in args.worlds.split(",")]:
        rank_ms = [0.0] * world
        per_row = {}
        for w in rows:
            ts = []
            for rank in range(world):
                r = bench.Row(w, world, rank, torch, ttb)
                r.allocate()
                r.autotune()
                r.refill_b()
                r.run()
                best = 1e30
                for _ in range(args.reps):
                    e0.record()
                    r.run()
                    e1.record()
                    e1.synchronize()
                    best = min(best, e0.elapsed_time(e1))
                ts.append(best)
                rank_ms[rank] += best
                r.free()
                torch.cuda.empty_cache()
            per_row[w.name] = {"max_ms": round(max(ts), 4), "mean_ms": round(sum(ts) / world, 4),
                               "imbalance": round(max(ts) * world / sum(ts), 3)}
        step = max(rank_ms)
        out[world] = {"predicted_gbs": round(total / 1e9 / (step / 1e3), 1), "step_ms": round(step, 3),
                      "rank_ms": [round(x, 3) for x in rank_ms], "rows": per_row}
        print(f"world {world}: predicted {out[world]['predicted_gbs']} GB/s "
              f"(step {step:.3f} ms, ranks {min(rank_ms):.3f}-{max(rank_ms):.3f} ms)", flush=True)
    if 1 in out:
        for world, v in out.items():
            v["speedup_vs_1"] = round(v["predicted_gbs"] / out[1]["predicted_gbs"], 3)
    print(json.dumps(out))


if __name__ == "__main__":
    main()

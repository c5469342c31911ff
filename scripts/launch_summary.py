#!/usr/bin/env python3
"""Summarize an ncu launch list of bench.py's timed region.

    python scripts/launch_summary.py profiles/rNN_launches.csv [--md out.md] [--traffic out.json]

Input: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--clock-control none --nvtx --nvtx-include "ttb_timed/" --csv --log-file F
python bench.py --steps 1 ...` (one launch per c5 row, in row order).
Writes a per-launch table (time, DRAM traffic vs algorithmic bytes) and the
per-family mean DRAM bytes per launch that bench.py reports as
roofline.traffic.
"""
import argparse
import collections
import csv
import io
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TIME_US = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}
FAMILY = {"btile_kernel": "btile", "dense_kernel": "dense", "tile_kernel": "tile", "smem_kernel": "smem",
          "vtile_kernel": "vtile",
          "rt_kernel": "rt", "copy_kernel": "copy", "copy_rows_kernel": "copy_rows", "rowcopy_kernel": "rowcopy", "tma_kernel": "tma"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--md")
    ap.add_argument("--traffic")
    args = ap.parse_args()
    from paper_1603_02297_b200.workloads import C5

    txt = open(args.csv).read().splitlines()
    start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
    launches = collections.OrderedDict()
    for r in csv.DictReader(io.StringIO("\n".join(txt[start:]))):
        d = launches.setdefault(r["ID"], {"kernel": r["Kernel Name"], "grid": r["Grid Size"]})
        v, u, name = float(r["Metric Value"].replace(",", "")), r["Metric Unit"], r["Metric Name"]
        if name == "gpu__time_duration.sum":
            d["us"] = v * TIME_US[u]
        elif name == "dram__bytes_read.sum":
            d["rd"] = v * BYTES[u]
        elif name == "dram__bytes_write.sum":
            d["wr"] = v * BYTES[u]
    fam = collections.defaultdict(lambda: {"us": 0.0, "traffic": 0.0, "alg": 0, "n": 0})
    out = ["| # | row | kernel | grid | time (us) | DRAM rd+wr (GB) | algorithmic (GB) | "
           "traffic/alg | alg GB/s |", "|---|---|---|---|---|---|---|---|---|"]
    total_us = 0.0
    for i, d in enumerate(launches.values()):
        w = C5[i % len(C5)]
        alg, tr = w.algorithmic_bytes, d["rd"] + d["wr"]
        kname = re.sub(r"\(.*", "", d["kernel"]).replace("void ", "")
        f = kname.split("<")[0]
        fam[f]["us"] += d["us"]
        fam[f]["traffic"] += tr
        fam[f]["alg"] += alg
        fam[f]["n"] += 1
        total_us += d["us"]
        out.append(f"| {i} | {w.name} | `{kname}` | {d['grid']} | {d['us']:.1f} | {tr / 1e9:.3f} | "
                   f"{alg / 1e9:.3f} | {tr / alg:.3f} | {alg / 1e3 / d['us']:.0f} |")
    out += ["", "| kernel | launches | share of kernel time | alg GB/s | DRAM GB/s | traffic/alg |",
            "|---|---|---|---|---|---|"]
    agg = collections.defaultdict(lambda: [0.0, 0])
    for f, v in sorted(fam.items(), key=lambda kv: -kv[1]["us"]):
        out.append(f"| {f} | {v['n']} | {v['us'] / total_us:.3f} | {v['alg'] / 1e3 / v['us']:.0f} | "
                   f"{v['traffic'] / 1e3 / v['us']:.0f} | {v['traffic'] / v['alg']:.3f} |")
        agg[FAMILY.get(f, f)][0] += v["traffic"]
        agg[FAMILY.get(f, f)][1] += v["n"]
    alg_all = sum(v["alg"] for v in fam.values())
    out.append(f"\nsum of kernel times {total_us / 1e3:.2f} ms for {alg_all / 1e9:.1f} GB "
               f"algorithmic -> {alg_all / 1e3 / total_us:.0f} GB/s (cold-cache, serialised)")
    text = "\n".join(out) + "\n"
    print(text)
    if args.md:
        open(args.md, "w").write(text)
    if args.traffic:
        t = {k: round(a / n) for k, (a, n) in agg.items()}
        t["_source"] = (f"{args.csv}: ncu dram__bytes_read.sum + dram__bytes_write.sum over the "
                        "NVTX range ttb_timed of bench.py (1 step, cold-cache, serialised); mean "
                        "DRAM bytes per launch per kernel family")
        json.dump(t, open(args.traffic, "w"), indent=1)


if __name__ == "__main__":
    main()

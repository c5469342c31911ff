#!/usr/bin/env python3
"""Summarize an ncu report (--set full) into the numbers the roofline needs.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep|raw.csv [--json out.json] [--bytes N]

Prints per kernel launch: duration, DRAM read/write bytes (traffic), DRAM
throughput, sectors per request (ld/st), shared-memory bank conflicts,
occupancy, issue activity and the top warp-stall reasons.  --bytes gives the
algorithmic bytes of one launch (the over-fetch ratio is traffic / bytes).
"""
import argparse
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_bytes": ("dram__bytes_read.sum", 1),
    "dram_write_bytes": ("dram__bytes_write.sum", 1),
    "dram_pct_peak": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "ld_sectors": ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", 1),
    "ld_requests": ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", 1),
    "st_sectors": ("l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", 1),
    "st_requests": ("l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", 1),
    "ldgsts_sectors": ("l1tex__t_sectors_pipe_lsu_mem_global_op_ldgsts.sum", 1),
    "ldgsts_requests": ("l1tex__t_requests_pipe_lsu_mem_global_op_ldgsts.sum", 1),
    "smem_ld_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", 1),
    "smem_st_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", 1),
    "registers": ("launch__registers_per_thread", 1),
    "achieved_occupancy_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "issue_active_pct": ("sm__inst_issued.avg.pct_of_peak_sustained_active", 1),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "grid": ("launch__grid_size", 1),
    "inst_executed": ("smsp__inst_executed.sum", 1),
    "smem_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1),
    "l2_read_sectors": ("lts__t_sectors_op_read.sum", 1),
    "l2_write_sectors": ("lts__t_sectors_op_write.sum", 1),
    "block": ("launch__block_size", 1),
}

BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "B": 1, "KB": 1e3,
         "MB": 1e6, "GB": 1e9}
NANOSECONDS = {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3,
               "ms": 1e6, "s": 1e9}


def raw(rep):
    if rep.endswith(".csv"):  # `ncu -i X --page raw --csv` exported on the GPU box
        with open(rep) as f:
            out = f.read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--json")
    ap.add_argument("--bytes", type=float, default=None)
    args = ap.parse_args()
    hdr, units, data = raw(args.rep)
    res = []
    for row in data:
        d = {"kernel": row[hdr.index("Kernel Name")][:90]}
        for key, (name, scale) in METRICS.items():
            if name not in hdr:
                continue
            i = hdr.index(name)
            try:
                v = float(row[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i].strip()
            if key == "duration_us":  # to microseconds; an unknown unit is an error, not a guess
                if u not in NANOSECONDS:
                    raise ValueError(f"{name}: unknown time unit {u!r}")
                v = v * NANOSECONDS[u] / 1e3
            elif "bytes" in key:
                if u not in BYTES:
                    raise ValueError(f"{name}: unknown byte unit {u!r}")
                v = v * BYTES[u]
            d[key] = v
        stalls = []
        for i, name in enumerate(hdr):
            if name.startswith("smsp__average_warps_issue_stalled_") and \
                    name.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(row[i].replace(",", "")),
                                   name[len("smsp__average_warps_issue_stalled_"):-len(
                                       "_per_issue_active.ratio")]))
                except ValueError:
                    pass
        d["stalls"] = {k: round(v, 2) for v, k in sorted(stalls, reverse=True)[:6]}
        if "ld_requests" in d and d["ld_requests"]:
            d["ld_sectors_per_req"] = d["ld_sectors"] / d["ld_requests"]
        if "st_requests" in d and d["st_requests"]:
            d["st_sectors_per_req"] = d["st_sectors"] / d["st_requests"]
        if "dram_read_bytes" in d:
            d["traffic_bytes"] = d["dram_read_bytes"] + d.get("dram_write_bytes", 0)
            if args.bytes:
                d["overfetch"] = d["traffic_bytes"] / args.bytes
            if d.get("duration_us"):
                d["dram_gbs"] = d["traffic_bytes"] / (d["duration_us"] * 1e3)
        res.append(d)
    for d in res:
        print(json.dumps(d))
    if args.json:
        with open(args.json, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    sys.exit(main())

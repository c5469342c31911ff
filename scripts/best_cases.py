"""Summarize scripts/run_case.py output: best plan per case."""
import re
import sys

best, cur = {}, None
for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/cases.log"):
    if line.startswith("#"):
        cur = line.split()[1]
        best[cur] = (0.0, "", "")
        continue
    m = re.match(r"\s*([\d.]+) us\s+([\d.]+) GB/s\s+(\S+)(.*)", line)
    if m and cur:
        g = float(m.group(2))
        if "MISMATCH" in line:
            print("MISMATCH", cur, line.strip())
        if g > best[cur][0]:
            best[cur] = (g, m.group(3), m.group(4))
for k, v in best.items():
    print(f"{k:8s} {v[0]:8.1f} {v[1]} {v[2]}")

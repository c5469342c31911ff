#!/usr/bin/env python3
"""Top SASS instructions of an `ncu --page source --csv` export by stall samples,
with each one's dominant stall reasons (kernel-design aid).

    python scripts/ncu_source_top.py gpurun_out/ncu_X_source.csv [N]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    col = {n: i for i, n in enumerate(hdr)}
    stall = [n for n in hdr if n.startswith("stall_") and "Not Issued" not in n]
    data = []
    for k, r in enumerate(rows[hi + 1:]):
        if len(r) < len(hdr):
            continue
        try:
            n = int(r[col["# Samples"]] or 0)
        except ValueError:
            continue
        data.append((n, k, r))
    total = sum(d[0] for d in data) or 1
    inst = sum(int(d[2][col["Instructions Executed"]] or 0) for d in data)
    print(f"{len(data)} instructions, {total} samples, {inst} warp instructions executed")
    tot_st = {s: sum(int(d[2][col[s]] or 0) for d in data) for s in stall}
    print("stalls overall:", ", ".join(f"{s[6:]} {100 * v / total:.1f}%" for s, v in
                                       sorted(tot_st.items(), key=lambda x: -x[1])[:8]))
    for n, k, r in sorted(data, reverse=True)[:top]:
        st = sorted(((int(r[col[s]] or 0), s[6:]) for s in stall), reverse=True)[:3]
        print(f"{100 * n / total:5.1f}% #{k:4d} exec={r[col['Instructions Executed']]:>9} "
              f"{r[col['Source']][:70]:70s} " + " ".join(f"{s}:{v}" for v, s in st if v))


if __name__ == "__main__":
    main()

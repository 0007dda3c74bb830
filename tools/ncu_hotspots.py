#!/usr/bin/env python
"""Top SASS lines by warp-stall samples of an ncu --set full report (source
page, --import-source on), with a few lines of context around each.
usage: ncu_hotspots.py REP [top] [context]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
    ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    data = rows[2:]
    i_s = h.index("Warp Stall Sampling (All Samples)")
    i_src = h.index("Source")
    val = [float(r[i_s]) if r[i_s] not in ("", "-") else 0.0 for r in data]
    tot = sum(val) or 1.0
    order = sorted(range(len(data)), key=lambda i: -val[i])[:top]
    print(f"== {rep}: {rows[0][1][:100]}  ({int(tot)} samples)")
    for i in order:
        print(f"{val[i] / tot * 100:5.1f}%  {i:5d}  {data[i][i_src].strip()[:100]}")
        for j in range(max(0, i - ctx), min(len(data), i + ctx + 1)):
            if j != i and ctx:
                print(f"          {j:5d}  {data[j][i_src].strip()[:100]}")


if __name__ == "__main__":
    main()

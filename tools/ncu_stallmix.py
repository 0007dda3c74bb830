#!/usr/bin/env python
"""Stall-reason mix of an ncu --set full report, split by SASS region: lines
[lo, hi) of the source page (default: whole kernel), plus the top lines.
usage: ncu_stallmix.py REP [lo hi]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = rows[1], rows[2:]
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3]) if len(sys.argv) > 3 else len(data)
cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = {h[i]: 0.0 for i in cols}
n = 0.0
for r in data[lo:hi]:
    for i in cols:
        try:
            tot[h[i]] += float(r[i])
        except ValueError:
            pass
s = sum(tot.values()) or 1
print(f"lines [{lo},{hi}): {int(s)} samples")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    if v:
        print(f"  {k:28s} {v / s * 100:5.1f}%")

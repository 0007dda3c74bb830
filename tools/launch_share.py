#!/usr/bin/env python
"""Per-kernel share of an `ncu --metrics gpu__time_duration.sum` launch list."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    h = [r for r in rows if r and r[0] == "ID"][0]
    data = rows[rows.index(h) + 1:]
    kn, v = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in data:
        agg[r[kn][:90]].append(float(r[v]))
    tot = sum(sum(x) for x in agg.values())
    print(f"{'launches':>8} {'total us':>10} {'share':>6} {'avg us':>8}  kernel")
    for k, x in sorted(agg.items(), key=lambda t: -sum(t[1])):
        print(f"{len(x):8d} {sum(x) / 1e3:10.1f} {100 * sum(x) / tot:5.1f}% {sum(x) / len(x) / 1e3:8.2f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])

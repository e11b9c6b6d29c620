#!/usr/bin/env python
"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel:
launches, total/mean device time, share of the step.  Times are cold-cache and
serialised under ncu: compare shares, not absolutes (B200_PROFILING.md)."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    head = rows[0]
    ki, mi, vi, ui = (head.index("Kernel Name"), head.index("Metric Name"),
                      head.index("Metric Value"), head.index("Metric Unit"))
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "").strip()
        us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += us
    total = sum(v[1] for v in agg.values())
    print(f"{'kernel':40s} {'launches':>8s} {'total ms':>10s} {'mean us':>10s} {'share':>7s}")
    for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:40s} {n:8d} {us/1e3:10.2f} {us/n:10.1f} {100*us/total:6.1f}%")
    print(f"{'TOTAL':40s} {sum(v[0] for v in agg.values()):8d} {total/1e3:10.2f}")


if __name__ == "__main__":
    main(sys.argv[1])

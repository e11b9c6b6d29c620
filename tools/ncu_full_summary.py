#!/usr/bin/env python
"""Compact summary of the full ncu captures written by tools/ncu_kernels.sh.

    python tools/ncu_full_summary.py <tag> [vertices]   (reads gpurun_out/<tag>_*.details.txt etc.)

Per kernel: the headline details (duration, DRAM/L2 throughput, issue slots,
occupancy), DRAM bytes, and the SASS instruction mix with stall share from the
source page (thread instructions per grid vertex when `vertices` is given).
"""
import collections
import csv
import glob
import os
import re
import sys

KEYS = ["Memory Throughput", "DRAM Throughput", "Duration", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "launch__grid_size", "launch__block_size"]


def details(path):
    out = []
    seen = set()
    for line in open(path, errors="replace"):
        s = line.strip()
        for k in KEYS:
            if s.startswith(k + " ") and k not in seen:
                seen.add(k)
                out.append("    " + re.sub(r"\s{2,}", "  ", s))
    return out


def raw(path):
    rows = [r for r in csv.reader(open(path, errors="replace")) if r]
    hi = next((i for i, r in enumerate(rows) if "ID" in r and "Kernel Name" in r), None)
    if hi is None or len(rows) < hi + 3:
        return []
    head, units, vals = rows[hi], rows[hi + 1], rows[hi + 2]
    out = []
    for m in RAW:
        if m in head:
            j = head.index(m)
            out.append(f"    {m:40s} {units[j]:8s} {vals[j]}")
    return out


def sass(path, vertices):
    rows = list(csv.reader(open(path, errors="replace")))
    hi = next((i for i, r in enumerate(rows) if r and r[0] == "Address"), None)
    if hi is None:
        return []
    h = rows[hi]
    try:
        ix, isrc, ith = h.index("Instructions Executed"), h.index("Source"), h.index("Thread Instructions Executed")
        ist = h.index("Warp Stall Sampling (All Samples)")
    except ValueError:
        return []
    mix, thr, stall = collections.Counter(), collections.Counter(), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= max(ix, ith) or not r[ix].strip():
            continue
        op = r[isrc].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
        o = o.split(".")[0]
        mix[o] += int(float(r[ix].replace(",", "")))
        thr[o] += int(float(r[ith].replace(",", "")))
        stall[o] += int(float(r[ist].replace(",", "") or 0))
    tw, tt, ts = sum(mix.values()), sum(thr.values()), sum(stall.values()) or 1
    lines = [f"warp instructions {tw:,}  thread instructions {tt:,}" +
             (f"  thread-instr/vertex {tt / vertices:.1f}" if vertices else "")]
    for o, c in mix.most_common(8):
        lines.append(f"{o:10s} {c:>16,}  {100 * c / tw:4.1f}%  stall {100 * stall[o] / ts:5.1f}%" +
                     (f"  {thr[o] / vertices:7.1f}/v" if vertices else ""))
    return lines


def main():
    tag = sys.argv[1]
    vertices = float(sys.argv[2]) if len(sys.argv) > 2 else 0
    for d in sorted(glob.glob(f"gpurun_out/{tag}_*.details.txt")):
        base = d[: -len(".details.txt")]
        name = os.path.basename(base)[len(tag) + 1:]
        print(f"=== {name} ===")
        for line in details(d) + (raw(base + ".raw.csv") if os.path.exists(base + ".raw.csv") else []):
            print(line)
        if os.path.exists(base + ".source.csv"):
            for line in sass(base + ".source.csv", vertices):
                print(line)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Instruction mix and stall samples per SASS opcode from an `ncu --page source --csv` export.

    python tools/sass_mix.py gpurun_out/<rep>.source.csv [vertices]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
ix, isrc, ist = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
ith = h.index("Thread Instructions Executed")
mix = collections.Counter()
thr = collections.Counter()
stall = collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= ix or not r[ix].strip():
        continue
    op = r[isrc].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1] if len(op) > 1 else o
    o = o.split(".")[0]
    mix[o] += int(r[ix].replace(",", ""))
    thr[o] += int(r[ith].replace(",", ""))
    stall[o] += int(r[ist].replace(",", "") or 0)
tot = sum(mix.values())
tthr = sum(thr.values())
nv = float(sys.argv[2]) if len(sys.argv) > 2 else None
print(f"warp instructions {tot:,}  thread instructions {tthr:,}"
      + (f"  thread-instr/vertex {tthr / nv:.1f}" if nv else ""))
st = sum(stall.values()) or 1
for o, c in mix.most_common(30):
    print(f"{o:10s} {c:14,d} {100 * c / tot:5.1f}%  stall {100 * stall[o] / st:5.1f}%"
          + (f"  {thr[o] / nv:6.1f}/v" if nv else ""))

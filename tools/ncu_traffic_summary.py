"""Per-kernel sums of an ncu --csv metrics log (tools/ncu_class_traffic.sh)."""
import collections
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, im, iv, iu, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), \
    h.index("Metric Unit"), h.index("ID")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1.0, "%": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}
per = collections.defaultdict(lambda: collections.defaultdict(float))
launches = collections.defaultdict(set)
for r in rows[1:]:
    k = r[ik].split("(")[0]
    v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    per[k][r[im]] += v
    launches[k].add(r[iid])
out = {}
for k, m in per.items():
    n = len(launches[k])
    dram = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    t = m.get("gpu__time_duration.sum", 0)
    out[k] = {"launches": n, "dram_bytes_total": dram, "dram_bytes_per_launch": dram / n,
              "time_s_total": t, "dram_GBps": dram / t / 1e9 if t else None,
              "l2_hit_rate_pct_mean": m.get("lts__t_sector_hit_rate.pct", 0) / n}
print(json.dumps(out, indent=1))

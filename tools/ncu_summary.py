#!/usr/bin/env python
"""Summarise an ncu report (raw page) per launch: time, DRAM bytes, GB/s, occupancy.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [metric ...]
"""
import csv
import subprocess
import sys

BASE = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors.sum",
        "l1tex__t_sectors.sum", "launch__occupancy_limit_registers"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1, "nsecond": 1e-9}


def rows(rep, metrics):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(metrics)],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    head, units = r[0], r[1]
    for row in r[2:]:
        d = {}
        for k, u, v in zip(head, units, row):
            try:
                val = float(v.replace(",", "")) * SCALE.get(u, 1)
            except ValueError:
                val = v
            d[k] = val
            d[k.split(".", 2)[-1] if k.count(".") >= 3 else k] = val
        for m in metrics:
            if m not in d:
                hit = [k for k in d if k.endswith(m)]
                d[m] = d[hit[0]] if hit else float("nan")
        yield d


def main():
    rep = sys.argv[1]
    extra = sys.argv[2:]
    for d in rows(rep, BASE + extra):
        t = d["gpu__time_duration.sum"]
        dram = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
        name = d["Kernel Name"].split("(")[0].replace("void ", "")[:34]
        print(f"{name:34s} grid={d['Grid Size']:>14s} t={t*1e6:9.1f}us dram={dram/1e6:9.1f}MB "
              f"{dram/t/1e9:7.0f}GB/s warps={d['sm__warps_active.avg.pct_of_peak_sustained_active']:5.1f}% "
              f"sm={d['sm__throughput.avg.pct_of_peak_sustained_elapsed']:5.1f}% "
              f"mem={d['gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed']:5.1f}% "
              f"L2={d['lts__t_sectors.sum']*32/1e6:8.1f}MB L1={d['l1tex__t_sectors.sum']*32/1e6:8.1f}MB "
              f"regs={d['launch__registers_per_thread']:.0f}"
              + "".join(f" {m}={d.get(m)}" for m in extra))


if __name__ == "__main__":
    main()

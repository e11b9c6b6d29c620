#!/usr/bin/env python
"""Development probe: single-device engine vs the z-slab sharded schedule run as
P virtual ranks on one GPU (in-process transport).  Prints wall time per call,
stats equality and the per-kernel-class profile.

    python tools/slab_probe.py [--dims 256x256x256] [--slabs 1,2,4] [--reps 2]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_09423_b200 as P  # noqa: E402
from paper_2406_09423_b200 import inputs as I  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--dims", default="256x256x256")
ap.add_argument("--slabs", default="1,2,4")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
cfg = I.CONFIGS[a.config]
dims = tuple(int(x) for x in a.dims.split("x"))
t = time.perf_counter()
f, fh, xi = I.make_inputs(cfg, dims, np.float32)
print(f"inputs {dims} in {time.perf_counter() - t:.1f} s", flush=True)
topo = P.build_topology(dims)
opts = P.DeriveOptions(subloop_cap=cfg.subloop_cap, profile=True)
keys = ("outer_iterations", "c_passes", "sub_iterations", "r_iterations", "effective_edits", "touched")


def run(fn):
    best, out = 1e9, None
    for _ in range(a.reps):
        st = P.EditStats()
        t = time.perf_counter()
        e = fn(st)
        dt = time.perf_counter() - t
        if dt < best:
            best, out = dt, (e, st)
    return best, out


t1, (e1, s1) = run(lambda st: P.derive_edits(topo, f, fh, xi, opts, st))
print(f"single  {t1*1e3:8.1f} ms  dev {s1.device_seconds*1e3:8.1f} ms  launches {s1.kernel_launches}  "
      f"stats {[getattr(s1, k) for k in keys]}", flush=True)
print("   ", {k: (v['launches'], round(v['ms'], 1)) for k, v in s1.kernel_profile().items() if v['launches']})
for p in [int(x) for x in a.slabs.split(",")]:
    tp, (ep, sp) = run(lambda st: P.derive_edits_slabs(topo, f, fh, xi, p, opts, st))
    same = np.array_equal(ep.indices, e1.indices) and ep.values.tobytes() == e1.values.tobytes() and \
        all(getattr(sp, k) == getattr(s1, k) for k in keys)
    print(f"slabs={p} {tp*1e3:8.1f} ms  dev {sp.device_seconds*1e3:8.1f} ms  launches {sp.kernel_launches}  "
          f"identical={same}  label_passes={sp.label_passes} huge={sp.huge_batches}", flush=True)
    print("   ", {k: (v['launches'], round(v['ms'], 1)) for k, v in sp.kernel_profile().items() if v['launches']})

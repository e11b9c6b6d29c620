#!/usr/bin/env python
"""Per-class kernel times of one profiled C4 derive (after a warm-up derive):
python tools/class_times.py [config] [dims]."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_09423_b200 as P  # noqa: E402
from paper_2406_09423_b200 import inputs as I  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
dims = tuple(int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1024x1024x1024").split("x"))
f, fh, xi = I.make_inputs(I.CONFIGS[cfg], dims, np.float32)
topo = P.build_topology(dims)
for rep in range(2):
    st = P.EditStats()
    P.derive_edits(topo, f, fh, xi, P.DeriveOptions(subloop_cap=100000, profile=True), st)
print(f"{cfg} {dims}: device {st.device_seconds * 1e3:.1f} ms, touched {st.touched}, "
      f"effective {st.effective_edits}, r_iterations {st.r_iterations}, sub {list(st.sub_iterations)}")
for k, v in st.kernel_profile().items():
    if v["launches"]:
        print(f"  {k:14s} {v['launches']:5d} launches {v['ms']:8.2f} ms  {v['ms'] / v['launches']:.3f} ms/launch")

#!/usr/bin/env python
"""Times the full direction sweep (K1) through the compute_direction_codes API path
on a resident field: python tools/time_dirs.py [dims] [reps]."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_09423_b200 as P  # noqa: E402
from paper_2406_09423_b200 import inputs as I  # noqa: E402

dims = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1024x1024x1024").split("x"))
f, fh, xi = I.make_inputs(I.CONFIGS["C4"], dims, np.float32)
topo = P.build_topology(dims)
st = P.EditStats()
opts = P.DeriveOptions(subloop_cap=100000, profile=True)
P.derive_edits(topo, f, fh, xi, opts, st)
st = P.EditStats()
P.derive_edits(topo, f, fh, xi, opts, st)
kp = st.kernel_profile()["directions"]
n = topo.vertex_count
ms = kp["ms"] / kp["launches"]
print(f"K1 {dims}: {kp['launches']} launches, {ms:.3f} ms/launch, {5 * n / ms / 1e6:.0f} GB/s alg, "
      f"MINB={os.environ.get('MSSZ_K1_MINB', '1')}, total device {st.device_seconds * 1e3:.1f} ms")

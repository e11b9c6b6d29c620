#!/usr/bin/env python
"""A/B of the 3D f32 direction sweep: the register-column K1 (default,
k_directions_col3) against the shared-memory K1 (MSSZ_K1_REG3=1,
k_directions_reg3).  Codes must be identical on every shape (ties, signed
zeros, odd extents); times come from the derive profile at C4 size.

    python tools/k1_ab.py [--time]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_09423_b200 as P  # noqa: E402
from paper_2406_09423_b200 import inputs as I  # noqa: E402


def codes(dims, v, reg3):
    if reg3:
        os.environ["MSSZ_K1_REG3"] = "1"
    else:
        os.environ.pop("MSSZ_K1_REG3", None)
    return P.compute_direction_codes(P.build_topology(dims), v)


rng = np.random.default_rng(7)
shapes = [(2, 2, 2), (3, 2, 5), (31, 7, 9), (32, 64, 3), (33, 65, 17), (61, 60, 59), (177, 95, 48),
          (1000, 3, 40), (3, 1000, 40), (130, 129, 2), (512, 512, 64)]
bad = 0
for dims in shapes:
    n = int(np.prod(dims))
    for kind in ("ties", "smooth", "zeros"):
        if kind == "ties":
            v = rng.integers(-3, 4, n).astype(np.float32)
        elif kind == "zeros":
            v = rng.choice(np.array([0.0, -0.0, 1.0, -1.0], np.float32), n)
        else:
            v = rng.standard_normal(n).astype(np.float32)
        a, b = codes(dims, v, False), codes(dims, v, True)
        ok = np.array_equal(a, b)
        bad += not ok
        print(f"{dims} {kind}: {'identical' if ok else 'DIFFER at %d' % int(np.argmax(a != b))}", flush=True)
if "--time" in sys.argv:
    dims = (1024, 1024, 1024)
    f, fh, xi = I.make_inputs(I.CONFIGS["C4"], dims, np.float32)
    a, b = codes(dims, fh, False), codes(dims, fh, True)
    print("C4 f-hat codes identical:", np.array_equal(a, b), flush=True)
    bad += not np.array_equal(a, b)
    del a, b
    topo = P.build_topology(dims)
    for reg3 in (False, True, False, True):
        if reg3:
            os.environ["MSSZ_K1_REG3"] = "1"
        else:
            os.environ.pop("MSSZ_K1_REG3", None)
        st = P.EditStats()
        P.derive_edits(topo, f, fh, xi, P.DeriveOptions(subloop_cap=100000, profile=True), st)
        kp = st.kernel_profile()["directions"]
        ms = kp["ms"] / kp["launches"]
        print(f"{'reg3' if reg3 else 'col3'}: {kp['launches']} launches {ms:.3f} ms/launch "
              f"{5 * topo.vertex_count / ms / 1e6:.0f} GB/s alg, device {st.device_seconds * 1e3:.1f} ms, "
              f"touched {st.touched}", flush=True)
sys.exit(1 if bad else 0)

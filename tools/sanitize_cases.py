"""Small end-to-end workload for compute-sanitizer (memcheck / synccheck / racecheck /
initcheck): every hot-path entry point of the C ABI on fields small enough to run
under instrumentation, each result checked against the oracle so a sanitizer run
also proves the instrumented run computed the same thing.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import paper_2406_09423_b200 as P  # noqa: E402
from paper_2406_09423_b200 import inputs as I  # noqa: E402

CASES = [
    # kind, dims, seed, rel, dtype: 2D, 3D, f64, the bench generator (FPmin-heavy:
    # parked items, big batches inside the persistent kernel, sparse R pass)
    ("gaussian-mixture", [96, 80], 2, 1e-2, np.float32),
    ("random-smooth", [48, 40, 24], 1, 1e-2, np.float32),
    ("trig", [32, 28, 20], 3, 1e-2, np.float64),
    ("multi-scale", [64, 64, 32], 0, 1e-3, np.float32),
]


def main() -> None:
    orc = O.oracle()
    only = sys.argv[1] if len(sys.argv) > 1 else ""
    for kind, dims, seed, rel, dt in CASES:
        topo = P.build_topology(dims)
        f = I.generate(kind, dims, seed, dt)
        xi = I.resolve_rel(f, rel)
        fh = I.compress_base(dims, f, xi)
        st = P.EditStats()
        e = P.derive_edits(topo, f, fh, xi, P.DeriveOptions(subloop_cap=100000), st)
        jac = orc.derive_edits(dims, f, fh, xi, subloop_cap=100000, schedule=O.JACOBI)
        assert np.array_equal(e.indices, jac.indices) and e.values.tobytes() == jac.values.tobytes()
        print(f"derive {kind} {dims}: {e.size()} edits, sub {st.sub_iterations}, "
              f"R {st.r_iterations}, big {st.big_batches}, sparse {st.sparse_iterations}", flush=True)
        if only == "derive":
            continue
        g = P.apply_edits(topo, fh, e)
        d = P.compute_directions(topo, g)
        a, b = orc.compute_directions(dims, g)
        assert np.array_equal(d.asc, a) and np.array_equal(d.desc, b)
        lab = P.compute_labels(topo, d)
        M, m = orc.compute_labels(dims, a, b)
        assert np.array_equal(lab.max_label, M) and np.array_equal(lab.min_label, m)
        assert P.segmentation(topo, g) == lab
        rep = P.detect_false_critical(topo, f, fh)
        want = orc.detect_false_critical(dims, f, fh)
        assert all(np.array_equal(x, w) for x, w in
                   zip([rep.fp_max, rep.fp_min, rep.fn_max, rep.fn_min], want))
        for mode in ("tiled", "sparse"):
            P.r_targets(topo, f, g, mode)
        r = P.build_report(topo, f, g, xi, e.size())
        assert r.passed()
        recon, sym, lits = P.compress_base(topo, f, xi)
        assert recon.tobytes() == fh.tobytes()
        assert P.decompress_base(topo, sym, lits, xi, dt).tobytes() == recon.tobytes()
        P.encode_edits(e, 1)
        if len(dims) == 3 and dt == np.float32:
            s = P.derive_edits_slabs(topo, f, fh, xi, 3, P.DeriveOptions(subloop_cap=100000))
            assert np.array_equal(s.indices, e.indices) and s.values.tobytes() == e.values.tobytes()
        print(f"  kernels/report/codecs ok", flush=True)
    # the per-device workspace is a deliberate cache; free it so a leak check
    # reports only real leaks
    P.library().mssz_cu_release_workspace(-1)
    print("sanitize cases ok")


if __name__ == "__main__":
    main()

"""Parity evidence at the benchmarked scales (run on the GPU box; writes JSON).

  python tools/parity_at_scale.py c4 [--mode full|sub|both] [--out F]   C4 snapshots, per-kernel parity
  python tools/parity_at_scale.py derive [--out F] [--configs C5,C3-256,...]

c4: one full C4 correction (bench workload) with on_batch_mode="phases"; the
  g snapshots after the first C pass, the states R iterations 1 and 10 start
  from, and the converged field are checked at FULL size (1024^3, the
  reference needs ~100 GB of host RAM for it) and on the middle z-sub-volume
  1024x1024x128 (as its own grid): the engine's directions, critical sets,
  false-critical report, labels and R-batch target set (tiled and sparse
  passes) against the UNMODIFIED reference (oracle/_ref: compute_directions
  mss.cpp:11-30, classify_critical mss.cpp:40-47, detect_false_critical
  edit_engine.cpp:134-158, compute_labels mss.cpp:84-97, run_r_loop's target
  collection edit_engine.cpp:336-352).

derive: full derive_edits at config size, GPU vs the Jacobi oracle (bit-exact
  edit set and EditStats) and vs the reference (EditStats side by side, touched
  within max(4, 1e-4 ref)), postconditions checked from scratch.

Only this tool, tests/, smoke() and bench.py's CPU legs use oracle/ (checkers).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import paper_2406_09423_b200 as P  # noqa: E402
from paper_2406_09423_b200 import inputs as I  # noqa: E402

STAT_KEYS = ("outer_iterations", "c_passes", "sub_iterations", "r_iterations",
             "effective_edits", "touched")
THREADS = os.cpu_count() or 1


def eq(a, b) -> bool:
    return bool(np.array_equal(a, b))


def kernel_parity(dims, f, g, R) -> dict:
    """Per-kernel parity of one (f, g) state on a grid: GPU vs the reference.
    Arrays are released as soon as they are compared (1024^3 u64 pairs are 17 GB)."""
    import gc
    topo = P.build_topology(dims)
    n = int(np.prod(dims))
    out: dict = {}
    t = time.perf_counter()
    d = P.compute_directions(topo, g)
    out["gpu_directions_s"] = time.perf_counter() - t
    t = time.perf_counter()
    a, b = R.compute_directions(dims, g, threads=THREADS)
    out["ref_directions_s"] = time.perf_counter() - t
    out["directions_bit_exact"] = eq(d.asc, a) and eq(d.desc, b)
    del a, b
    gc.collect()
    cs = P.classify_critical(d)
    ids = np.arange(n, dtype=np.uint64)
    out["maxima"], out["minima"] = int(cs.maxima.size), int(cs.minima.size)
    out["critical_sets_equal"] = eq(cs.maxima, np.flatnonzero(d.asc == ids)) and \
        eq(cs.minima, np.flatnonzero(d.desc == ids))
    del ids, cs
    lab = P.compute_labels(topo, d)
    t = time.perf_counter()
    M, m = R.compute_labels(dims, d.asc, d.desc, threads=THREADS)
    out["ref_labels_s"] = time.perf_counter() - t
    out["labels_bit_exact"] = eq(lab.max_label, M) and eq(lab.min_label, m)
    del d, lab, M, m
    gc.collect()
    rep = P.detect_false_critical(topo, f, g)
    got = [rep.fp_max, rep.fp_min, rep.fn_max, rep.fn_min]
    del rep
    t = time.perf_counter()
    want = R.detect_false_critical(dims, f, g, threads=THREADS)
    out["ref_detect_s"] = time.perf_counter() - t
    out["false_critical_counts"] = [int(x.size) for x in got]
    out["false_critical_bit_exact"] = all(eq(x, w) for x, w in zip(got, want))
    del got, want
    gc.collect()
    t = time.perf_counter()
    tw, false_cp, sources, mism = R.r_targets(dims, f, g, threads=THREADS)
    out["ref_r_targets_s"] = time.perf_counter() - t
    out["r_batch"] = {"targets": int(tw.size), "sources": sources, "mismatched_vertices": mism,
                      "false_critical_gate": false_cp,
                      "is_a_real_r_batch": false_cp == 0 and mism > 0}
    for mode in ("tiled", "sparse"):
        t = time.perf_counter()
        r = P.r_targets(topo, f, g, mode)
        out["r_batch"][mode] = {"bit_exact": eq(r.targets, tw) and r.sources == sources
                                and r.false_critical == false_cp, "path": r.path,
                                "s": time.perf_counter() - t}
    return out


def c4(args) -> dict:
    """Snapshots of a config's correction (default C4): full-field and (3D)
    middle z-sub-volume per-kernel parity."""
    import gc
    cfg = I.CONFIGS[args.config]
    dims = list(cfg.dims)
    t = time.perf_counter()
    f, fh, xi = I.make_inputs(cfg)
    gen_s = time.perf_counter() - t
    if len(dims) == 3 and dims[2] > args.planes:
        X, Y, Z = dims
        z0 = Z // 2 - args.planes // 2
        sl = slice(z0 * X * Y, (z0 + args.planes) * X * Y)
        sub_dims = [X, Y, args.planes]
    else:  # 2D or thin: no sub-volume
        z0, sl, sub_dims = 0, None, None
        if args.mode == "sub":
            args.mode = "full"
        elif args.mode == "both":
            args.mode = "full"
    # kept states: after the first C pass; the state R iteration 1 starts from
    # (the last C pass before it); after R iterations 1, 10 and 20 of the run
    # (the start states of the next R batch when the R gate passes there); the
    # converged field
    snaps: dict = {}
    held = {}
    r_total = [0]

    def cb(g):
        kind, outer, idx = P.batch_phase()
        if kind == "c_pass":
            if (outer, idx) == (1, 1):
                snaps["after C pass 1 (outer 1)"] = g
            held["last"] = (f"after C pass {idx} (outer {outer})", g)
        else:
            r_total[0] += 1
            if r_total[0] == 1:
                label, hg = held["last"]
                snaps[f"{label}: the state R iteration 1 starts from"] = hg
            if r_total[0] in (1, 10, 20):
                snaps[f"after R iteration #{r_total[0]} of the run (outer {outer}, #{idx} of "
                      "its R loop)"] = g
            held.clear()

    st = P.EditStats()
    t = time.perf_counter()
    edits = P.derive_edits(P.build_topology(dims), f, fh, xi,
                           P.DeriveOptions(subloop_cap=cfg.subloop_cap, on_batch=cb,
                                           on_batch_mode="phases"), st)
    run_s = time.perf_counter() - t
    held.clear()
    final = fh.copy()
    final[edits.indices] = edits.values
    del edits
    snaps["converged"] = final
    del fh, final
    gc.collect()
    res = {"workload": cfg.note, "dims": dims, "xi": xi, "input_gen_s": gen_s,
           "derive_with_snapshots_s": run_s, "edit_stats": {k: getattr(st, k) for k in STAT_KEYS},
           "reference_threads": THREADS, "full_field": [],
           "sub_volume": {"dims": sub_dims, "z_planes": [z0, z0 + args.planes] if sub_dims else None,
                          "note": "the sub-volume is treated as its own grid (boundary planes clipped)",
                          "snapshots": []}}
    R = O.ref()
    for label, g in snaps.items():
        if args.mode in ("sub", "both"):
            print(f"[c4] sub-volume: {label}", file=sys.stderr, flush=True)
            k = kernel_parity(sub_dims, f[sl].copy(), g[sl].copy(), R)
            k["snapshot"] = label
            res["sub_volume"]["snapshots"].append(k)
            gc.collect()
        if args.mode in ("full", "both"):
            print(f"[c4] full field: {label}", file=sys.stderr, flush=True)
            k = kernel_parity(dims, f, g, R)
            k["snapshot"] = label
            res["full_field"].append(k)
            gc.collect()
        if args.out:
            with open(args.out, "w") as fp:
                json.dump(res, fp, indent=1, default=str)

    def ok(s):
        rb = s["r_batch"]
        return (s["directions_bit_exact"] and s["critical_sets_equal"] and s["false_critical_bit_exact"]
                and s["labels_bit_exact"] and rb["tiled"]["bit_exact"] and rb["sparse"]["bit_exact"])
    res["all_bit_exact"] = all(ok(s) for s in res["full_field"] + res["sub_volume"]["snapshots"])
    return res


DERIVE = {
    # name: (kind, dims, rel, subloop_cap, dtype)
    "C1": ("gaussian-mixture", [512, 512], 1e-3, 640, np.float32),
    "C2-rs-1e-2": ("random-smooth", [177, 95, 48], 1e-2, 640, np.float32),
    "C2-trig-1e-2": ("trig", [177, 95, 48], 1e-2, 640, np.float32),
    "C3-256": ("random-smooth", [256, 256, 256], 1e-3, 100000, np.float32),
    "C3": ("random-smooth", [512, 512, 512], 1e-3, 100000, np.float32),
    "C4-128": ("multi-scale", [128, 128, 128], 1e-3, 100000, np.float32),
    "C5": ("gaussian-mixture", [3600, 2400], 1e-4, 100000, np.float32),
}


def derive_one(name) -> dict:
    kind, dims, rel, cap, dt = DERIVE[name]
    topo = P.build_topology(dims)
    f = I.generate(kind, dims, 0, dt)
    xi = I.resolve_rel(f, rel)
    fh = I.compress_base(dims, f, xi)
    out = {"name": name, "kind": kind, "dims": dims, "rel_eb": rel, "xi": xi, "subloop_cap": cap,
           "vertices": int(np.prod(dims))}
    st = P.EditStats()
    t = time.perf_counter()
    e = P.derive_edits(topo, f, fh, xi, P.DeriveOptions(subloop_cap=cap), st)
    out["gpu_s"] = time.perf_counter() - t
    out["gpu_stats"] = {k: getattr(st, k) for k in STAT_KEYS}
    g = P.apply_edits(topo, fh, e)
    out["postconditions"] = {
        "labels_equal": P.segmentation(topo, g) == P.segmentation(topo, f),
        "bound_ok": bool(np.all(np.abs(g.astype(np.float64) - f.astype(np.float64)) <= xi)),
        "false_critical": P.detect_false_critical(topo, f, g).total(),
    }
    print(f"[derive] {name}: gpu {out['gpu_s']:.2f}s {out['gpu_stats']}", file=sys.stderr, flush=True)
    t = time.perf_counter()
    jac = O.oracle().derive_edits(dims, f, fh, xi, subloop_cap=cap, schedule=O.JACOBI)
    out["jacobi_oracle_s"] = time.perf_counter() - t
    out["jacobi_stats"] = {k: jac.stats[k] for k in STAT_KEYS}
    out["bit_exact_vs_jacobi"] = eq(e.indices, jac.indices) and \
        e.values.tobytes() == jac.values.tobytes() and out["gpu_stats"] == out["jacobi_stats"]
    del jac
    print(f"[derive] {name}: jacobi {out['jacobi_oracle_s']:.1f}s exact={out['bit_exact_vs_jacobi']}",
          file=sys.stderr, flush=True)
    t = time.perf_counter()
    ref = O.ref().derive_edits(dims, f, fh, xi, subloop_cap=cap, threads=THREADS)
    out["reference_s"] = time.perf_counter() - t
    out["reference_threads"] = THREADS
    out["reference_stats"] = {k: ref.stats[k] for k in STAT_KEYS}
    rt = ref.stats["touched"]
    out["touched_diff"] = int(st.touched) - int(rt)
    out["touched_tolerance"] = max(4, int(1e-4 * rt))
    out["touched_within_tolerance"] = abs(out["touched_diff"]) <= out["touched_tolerance"]
    both = np.intersect1d(e.indices, ref.indices, assume_unique=True)
    out["edit_index_overlap"] = {"gpu": int(e.indices.size), "reference": int(ref.indices.size),
                                 "common": int(both.size)}
    print(f"[derive] {name}: reference {out['reference_s']:.1f}s {out['reference_stats']}",
          file=sys.stderr, flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["c4", "derive"])
    ap.add_argument("--config", default="C4", help="c4: which config's correction to snapshot")
    ap.add_argument("--mode", default="both", choices=["full", "sub", "both"])
    ap.add_argument("--out", default=None)
    ap.add_argument("--planes", type=int, default=128)
    ap.add_argument("--configs", default="C1,C2-rs-1e-2,C2-trig-1e-2,C4-128,C3-256,C5")
    args = ap.parse_args()
    if args.what == "c4":
        res = c4(args)
    else:
        res = {"cases": [], "host_threads": THREADS}
        for name in args.configs.split(","):
            res["cases"].append(derive_one(name))
            if args.out:  # partial results survive a timeout
                with open(args.out, "w") as fp:
                    json.dump(res, fp, indent=1, default=str)
    text = json.dumps(res, indent=1, default=str)
    if args.out:
        with open(args.out, "w") as fp:
            fp.write(text)
    print(text)


if __name__ == "__main__":
    main()

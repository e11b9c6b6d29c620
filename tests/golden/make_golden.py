"""Generates the committed golden vectors from the UNMODIFIED reference.

Run in the build container (needs /root/reference and oracle/_ref/libmssz_ref.so):

    make -C oracle && python tests/golden/make_golden.py

Outputs (small, committed):
  golden.npz   arrays (fields, directions, labels, reports, edit sets)
  golden.json  case metadata (dims, dtype, xi, options, reference EditStats,
               sha256 of generator / base-codec outputs at larger sizes)

Every case mirrors a reference test (file:line in its 'source' field) or the
reference's own synthetic pipeline (field.cpp + base_codec.cpp).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402

R = O.ref()
arrays: dict = {}
meta: dict = {"directions": [], "derive": [], "detect": [], "troublemaker": [], "lower_step": [],
              "hashes": []}


def put(name, a):
    arrays[name] = np.ascontiguousarray(a)
    return name


def random_field(rng, n, dup, dtype=np.float64):
    # test_mss.cpp:20-33 (values from a 16-symbol alphabet to force SoS ties)
    raw = rng.integers(0, 2**63, size=n, dtype=np.uint64)
    if dup:
        return (raw % 16).astype(dtype)
    return ((raw >> np.uint64(11)).astype(np.float64) * 2.0**-53).astype(dtype)


# ---- directions / labels / critical sets -----------------------------------------
rng = np.random.default_rng(20240613)
dir_cases = [
    ("const_2x2", [2, 2], np.array([5, 5, 5, 5], np.float64), "test_mss.cpp:37-51"),
    ("ramp_5x4", [5, 4], np.arange(20, dtype=np.float64), "test_mss.cpp:53-68"),
    ("staircase_6x3", [6, 3], np.array([v * v % 37 for v in range(18)], np.float64),
     "test_mss.cpp:91-106"),
]
for t in range(12):
    dims = [8, 8] if t % 2 == 0 else [4, 4, 4]
    n = int(np.prod(dims))
    dir_cases.append((f"random_{t}", dims, random_field(rng, n, t % 3 == 0),
                      "test_mss.cpp:124-136"))
for t in range(4):
    dims = [[16, 16], [7, 6], [9, 7, 5], [5, 6, 7]][t]
    n = int(np.prod(dims))
    dt = np.float32 if t % 2 else np.float64
    dir_cases.append((f"random32_{t}", dims, random_field(rng, n, t < 2, dt), "test_mss.cpp:70-89"))
# signed zeros (SoS treats -0.0 == +0.0, grid.hpp:56)
dir_cases.append(("signed_zero_4x4", [4, 4],
                  np.array([0.0, -0.0, 0.0, -0.0, 1, -0.0, 0.0, -1, -0.0, 0.0, 2, 0.0, -0.0,
                            -0.0, 0.0, 0.0], np.float32), "grid.hpp:53-58"))
for name, dims, vals, src in dir_cases:
    asc, desc = R.compute_directions(dims, vals)
    M, m = R.compute_labels(dims, asc, desc)
    oM, om = R.oracle_labels(dims, vals)
    assert np.array_equal(M, oM) and np.array_equal(m, om)
    meta["directions"].append({"name": name, "dims": dims, "dtype": str(vals.dtype), "source": src})
    put(f"dir/{name}/values", vals)
    put(f"dir/{name}/asc", asc)
    put(f"dir/{name}/desc", desc)
    put(f"dir/{name}/max_label", M)
    put(f"dir/{name}/min_label", m)

# ---- false-critical detection KAT (test_edit_engine.cpp:104-118) ----------------
f = np.arange(9, dtype=np.float64)
fh = f.copy()
fh[4] = 8.6
rep = R.detect_false_critical([3, 3], f, fh, 5.0)
meta["detect"].append({"name": "ramp_3x3_spike", "dims": [3, 3], "xi": 5.0,
                       "source": "test_edit_engine.cpp:104-118",
                       "counts": [int(x.size) for x in rep]})
put("detect/ramp_3x3_spike/f", f)
put("detect/ramp_3x3_spike/g", fh)
for k, lst in enumerate(rep):
    put(f"detect/ramp_3x3_spike/list{k}", lst)

# ---- troublemaker KATs (test_edit_engine.cpp:138-185) ----------------------------
for name, vals, spike, desc_kind in [
    ("asc", [0, 1, 2, 3, 4, 23, 6, 22, 8], 24.0, False),
    ("desc", [0, -1, -2, -3, -4, -23, -6, -22, -8], -24.0, True),
]:
    f = np.array(vals, np.float64)
    g = f.copy()
    g[7] = spike
    vi, vt = R.find_troublemaker([3, 3], f, g, 2.5, 4, desc_kind)
    meta["troublemaker"].append({"name": name, "dims": [3, 3], "xi": 2.5, "v": 4,
                                 "descending": desc_kind, "vi": vi, "vt": vt,
                                 "source": "test_edit_engine.cpp:138-185"})
    put(f"tm/{name}/f", f)
    put(f"tm/{name}/g", g)

# ---- lower_step traces (test_edit_engine.cpp:43-95) ------------------------------
for name, fv, gv, xi, dt in [
    ("halve_10_11", 10.0, 11.0, 1.0, np.float64),
    ("floor_10_9", 10.0, 9.0, 1.0, np.float64),
    ("converge_0.3_0.4", 0.3, 0.4, 0.1, np.float64),
    ("f32_converge", 0.3, 0.4, 0.1, np.float32),
    ("f32_large", 1234.5, 1234.75, 0.37, np.float32),
    ("f32_negative", -2.5, -2.25, 0.5, np.float32),
    ("f64_tiny_xi", 1.0, 1.0 + 1e-12, 1e-12, np.float64),
]:
    f = np.array([fv, 9, 9, 9], dt)
    g = np.array([gv, 9, 9, 9], dt)
    trace, floor = R.lower_step_trace([2, 2], f, g, xi, 0, 200)
    meta["lower_step"].append({"name": name, "f": fv, "g": gv, "xi": xi, "dtype": str(np.dtype(dt)),
                               "source": "test_edit_engine.cpp:43-95"})
    put(f"ls/{name}/trace", trace)
    put(f"ls/{name}/floor", np.array([floor], dt))

# ---- derive_edits end to end (serial reference, the deterministic schedule) ------
derive_cases = [
    # (name, kind, dims, seed, rel, dtype, source)
    ("race_2x2", None, [2, 2], 0, None, np.float64, "test_edit_engine.cpp:120-136"),
    ("identity_12x12", "gaussian-mixture", [12, 12], 7, None, np.float64, "test_edit_engine.cpp:187-196"),
]
for run in range(6):  # test_edit_engine.cpp:198-230
    kinds = ["gaussian-mixture", "trig", "random-smooth"]
    dims = [8, 8, 8] if run % 2 else [24, 24]
    derive_cases.append((f"codec_run{run}", kinds[run % 3], dims, run, 1e-2, np.float64,
                         "test_edit_engine.cpp:198-230"))
derive_cases += [
    ("trig_20x20_f64", "trig", [20, 20], 5, 1e-2, np.float64, "test_edit_engine.cpp:232-254"),
    ("gm_16x16_f32", "gaussian-mixture", [16, 16], 21, 1e-2, np.float32, "test_edit_engine.cpp:332-344"),
    ("gm_16x16x8_f64", "gaussian-mixture", [16, 16, 8], 11, 1e-2, np.float64, "test_edit_engine.cpp:297-311"),
    ("gm_64x64_f32", "gaussian-mixture", [64, 64], 0, 1e-3, np.float32, "SURVEY C1 shape"),
    ("gm_96x64_f32_1e-2", "gaussian-mixture", [96, 64], 2, 1e-2, np.float32, "SURVEY C1 shape"),
    ("rs_24x20x12_f32", "random-smooth", [24, 20, 12], 0, 1e-2, np.float32, "SURVEY C2 shape"),
    ("trig_24x20x12_f32", "trig", [24, 20, 12], 1, 1e-2, np.float32, "SURVEY C2 shape"),
    ("rs_32x32x16_f32", "random-smooth", [32, 32, 16], 3, 1e-3, np.float32, "SURVEY C2 shape"),
]
for name, kind, dims, seed, rel, dt, src in derive_cases:
    n = int(np.prod(dims))
    if name == "race_2x2":
        f = np.array([1.0, 2.0, -5.0, -6.0], dt)
        fh = np.array([1.5, 1.45, -5.0, -6.0], dt)
        xi = 0.6
    elif name.startswith("identity"):
        f = R.generate(kind, dims, seed, dt)
        fh = f.copy()
        xi = 0.01
    else:
        f = R.generate(kind, dims, seed, dt)
        xi = R.resolve_rel(dims, f, rel)
        fh = R.compress_base(dims, f, xi)
    res = R.derive_edits(dims, f, fh, xi, threads=1)
    st = {k: v for k, v in res.stats.items() if not k.endswith("seconds")}
    meta["derive"].append({"name": name, "kind": kind, "dims": dims, "seed": seed, "rel": rel,
                           "dtype": str(np.dtype(dt)), "xi": xi, "stats": st, "source": src})
    put(f"derive/{name}/f", f)
    put(f"derive/{name}/fhat", fh)
    put(f"derive/{name}/indices", res.indices)
    put(f"derive/{name}/values", res.values)

# ---- generator / base-codec pins at sizes too large to store ---------------------
for kind, dims, seed, dt in [
    ("gaussian-mixture", [512, 512], 0, np.float32),
    ("random-smooth", [177, 95, 48], 0, np.float32),
    ("trig", [177, 95, 48], 0, np.float32),
    ("gaussian-mixture", [177, 95, 48], 0, np.float64),
    ("gaussian-mixture", [360, 240], 0, np.float32),
]:
    f = R.generate(kind, dims, seed, dt)
    xi = R.resolve_rel(dims, f, 1e-3)
    fh = R.compress_base(dims, f, xi)
    meta["hashes"].append({"kind": kind, "dims": dims, "seed": seed, "dtype": str(np.dtype(dt)),
                           "rel": 1e-3, "xi": xi,
                           "f_sha256": hashlib.sha256(f.tobytes()).hexdigest(),
                           "fhat_sha256": hashlib.sha256(fh.tobytes()).hexdigest()})

np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
with open(os.path.join(HERE, "golden.json"), "w") as fp:
    json.dump(meta, fp, indent=1)
print(f"{len(arrays)} arrays, {os.path.getsize(os.path.join(HERE, 'golden.npz'))} bytes")

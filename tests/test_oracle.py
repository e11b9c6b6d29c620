"""CPU: the plain-C oracle is pinned to the reference's golden vectors (and to the
reference library itself when it is built here)."""
import numpy as np
import pytest

import oracle as O


def test_directions_and_labels_match_golden(golden, oracle_lib):
    meta, arr = golden
    for case in meta["directions"]:
        p = f"dir/{case['name']}/"
        dims = case["dims"]
        asc, desc = oracle_lib.compute_directions(dims, arr[p + "values"])
        assert np.array_equal(asc, arr[p + "asc"]), case["name"]
        assert np.array_equal(desc, arr[p + "desc"]), case["name"]
        M, m = oracle_lib.compute_labels(dims, asc, desc)
        assert np.array_equal(M, arr[p + "max_label"]), case["name"]
        assert np.array_equal(m, arr[p + "min_label"]), case["name"]


def test_constant_field_corner_extrema(golden):
    # test_mss.cpp:37-51: max {3}, min {0}
    _, arr = golden
    asc, desc = arr["dir/const_2x2/asc"], arr["dir/const_2x2/desc"]
    assert [v for v in range(4) if asc[v] == v] == [3]
    assert [v for v in range(4) if desc[v] == v] == [0]


def test_odd_cycle_trips_round_cap(oracle_lib):
    # test_mss.cpp:153-166
    with pytest.raises(O.CheckerError) as e:
        oracle_lib.compute_labels([2, 2], np.array([1, 2, 0, 3], np.uint64), np.zeros(4, np.uint64))
    assert e.value.code == 7


def test_detect_kat(golden, oracle_lib):
    meta, arr = golden
    for case in meta["detect"]:
        p = f"detect/{case['name']}/"
        counts = np.zeros(4, np.uint64)
        lists = oracle_lib.detect_false_critical(case["dims"], arr[p + "f"], arr[p + "g"])
        for k in range(4):
            assert np.array_equal(lists[k], arr[p + f"list{k}"])
    # test_edit_engine.cpp:112-113
    assert list(arr["detect/ramp_3x3_spike/list0"]) == [4]
    assert list(arr["detect/ramp_3x3_spike/list2"]) == [8]


def test_lower_step_traces(golden, oracle_lib):
    meta, arr = golden
    for case in meta["lower_step"]:
        dt = np.dtype(case["dtype"])
        trace = arr[f"ls/{case['name']}/trace"]
        g = trace[0]
        for want in trace[1:]:
            moved, g = oracle_lib.lower_step(g, dt.type(case["f"]), case["xi"], dt)
            assert moved
            assert dt.type(g).tobytes() == want.tobytes(), case["name"]
        moved, _ = oracle_lib.lower_step(g, dt.type(case["f"]), case["xi"], dt)
        assert not moved, case["name"]
        fl = oracle_lib.representable_floor(dt.type(case["f"]), case["xi"], dt)
        assert dt.type(fl).tobytes() == arr[f"ls/{case['name']}/floor"][0].tobytes()
    # test_edit_engine.cpp:43-51: (11 + 10 - 1) / 2 = 10
    assert arr["ls/halve_10_11/trace"][1] == 10.0
    assert arr["ls/floor_10_9/trace"].size == 1


@pytest.mark.parametrize("schedule", [O.GAUSS_SEIDEL, O.JACOBI])
def test_derive_matches_golden(golden, oracle_lib, schedule):
    meta, arr = golden
    for case in meta["derive"]:
        p = f"derive/{case['name']}/"
        res = oracle_lib.derive_edits(case["dims"], arr[p + "f"], arr[p + "fhat"], case["xi"],
                                      schedule=schedule)
        if schedule == O.GAUSS_SEIDEL:
            # the serial reference schedule: bit-exact edit set and EditStats
            assert np.array_equal(res.indices, arr[p + "indices"]), case["name"]
            assert res.values.tobytes() == arr[p + "values"].tobytes(), case["name"]
            for k, v in case["stats"].items():
                assert res.stats[k] == v, (case["name"], k)
        else:
            tol = max(4, int(1e-4 * case["stats"]["touched"]))
            assert abs(len(res.indices) - case["stats"]["touched"]) <= tol, case["name"]


def test_derive_errors(oracle_lib):
    f = np.zeros(36, np.float64)
    fh = f.copy()
    fh[10] = 1.0
    with pytest.raises(O.CheckerError) as e:
        oracle_lib.derive_edits([6, 6], f, fh, 0.01)
    assert e.value.code == 4
    oracle_lib.derive_edits([6, 6], f, fh, 0.01, force=True)
    with pytest.raises(O.CheckerError) as e:
        oracle_lib.derive_edits([6, 6], f, f, 0.0)
    assert e.value.code == 2


@pytest.mark.parametrize("kind,dims,seed,rel,dt", [
    ("gaussian-mixture", [40, 33], 4, 1e-2, np.float32),
    ("random-smooth", [12, 11, 10], 5, 1e-2, np.float32),
    ("trig", [14, 12, 9], 6, 5e-3, np.float64),
])
def test_oracle_vs_reference_live(ref_lib, oracle_lib, kind, dims, seed, rel, dt):
    f = ref_lib.generate(kind, dims, seed, dt)
    xi = ref_lib.resolve_rel(dims, f, rel)
    fh = ref_lib.compress_base(dims, f, xi)
    r = ref_lib.derive_edits(dims, f, fh, xi, threads=1)
    o = oracle_lib.derive_edits(dims, f, fh, xi, schedule=O.GAUSS_SEIDEL)
    assert np.array_equal(r.indices, o.indices)
    assert r.values.tobytes() == o.values.tobytes()
    for k in ("outer_iterations", "c_passes", "sub_iterations", "r_iterations",
              "effective_edits", "touched"):
        assert r.stats[k] == o.stats[k], k


def test_reference_r_targets_troublemaker_kats(golden, ref_lib):
    """The shim's run_r_loop target collection reproduces the golden (v_i, v_t) of
    test_edit_engine.cpp:138-185 (the R-batch parity tests compare the GPU with it)."""
    meta, arr = golden
    for case in meta["troublemaker"]:
        f = arr[f"tm/{case['name']}/f"]
        g = arr[f"tm/{case['name']}/g"]
        targets, _false, sources, mism = ref_lib.r_targets(case["dims"], f, g)
        assert case["vt"] in targets.tolist(), case["name"]
        assert sources >= 1 and mism >= 1
        vi, vt = ref_lib.find_troublemaker(case["dims"], f, g, case["xi"], case["v"],
                                           case["descending"])
        assert (vi, vt) == (case["vi"], case["vt"])

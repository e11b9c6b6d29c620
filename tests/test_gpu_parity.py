"""GPU parity: every CUDA entry point, through the C-ABI, against the oracle and the
reference's golden vectors.

Bars:
* directions, labels, critical sets, detection lists, lower_step: bit-exact;
* derive_edits: bit-exact (edit set AND every EditStats counter) against the
  oracle's Jacobi schedule, which is the B200 fix schedule; against the serial
  reference (Gauss-Seidel) within |touched - ref| <= max(4, 1e-4 * ref);
* postconditions from scratch: labels(g) == labels(f), critical sets equal,
  f - xi < g <= fhat (double-precision check).
"""
import numpy as np
import pytest

import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(240)]

STAT_KEYS = ("outer_iterations", "c_passes", "sub_iterations", "r_iterations",
             "effective_edits", "touched")


@pytest.fixture(scope="module")
def P(mssz):
    if mssz.library().mssz_cu_device_count() == 0:
        pytest.fail("no CUDA device visible to the GPU test suite")
    return mssz


def stats_dict(st):
    return {k: getattr(st, k) for k in STAT_KEYS}


def check_postconditions(P, topo, f, g, xi):
    f64 = f.astype(np.float64)
    g64 = g.astype(np.float64)
    assert np.all(np.abs(f64 - g64) <= xi)
    df = P.compute_directions(topo, f)
    dg = P.compute_directions(topo, g)
    cf, cg = P.classify_critical(df), P.classify_critical(dg)
    assert np.array_equal(cf.maxima, cg.maxima) and np.array_equal(cf.minima, cg.minima)
    assert P.compute_labels(topo, df) == P.compute_labels(topo, dg)


# ------------------------------------------------------------------ kernels
def test_directions_labels_golden(P, golden):
    meta, arr = golden
    for case in meta["directions"]:
        p = f"dir/{case['name']}/"
        topo = P.build_topology(case["dims"])
        d = P.compute_directions(topo, arr[p + "values"])
        assert np.array_equal(d.asc, arr[p + "asc"]), case["name"]
        assert np.array_equal(d.desc, arr[p + "desc"]), case["name"]
        lab = P.compute_labels(topo, d)
        assert np.array_equal(lab.max_label, arr[p + "max_label"]), case["name"]
        assert np.array_equal(lab.min_label, arr[p + "min_label"]), case["name"]
        cs = P.classify_critical(d)
        assert np.array_equal(cs.maxima, np.flatnonzero(arr[p + "asc"] == np.arange(topo.vertex_count)))
        assert np.array_equal(cs.minima, np.flatnonzero(arr[p + "desc"] == np.arange(topo.vertex_count)))


@pytest.mark.parametrize("dims,dt", [([512, 512], np.float32), ([177, 95, 48], np.float32),
                                     ([64, 33, 17], np.float64), ([3600, 240], np.float32),
                                     ([256, 64, 40], np.float32), ([260, 30, 21], np.float32),
                                     ([131, 17, 9], np.float32), ([4, 3, 2], np.float32),
                                     ([2, 2, 2], np.float32)])
def test_directions_labels_vs_oracle(P, oracle_lib, dims, dt):
    from paper_2406_09423_b200 import inputs as I
    rng = np.random.default_rng(7)
    topo = P.build_topology(dims)
    fields = [I.generate("random-smooth", dims, 1, dt),
              (rng.integers(0, 11, topo.vertex_count)).astype(dt)]  # heavy SoS ties
    for vals in fields:
        d = P.compute_directions(topo, vals)
        a, b = oracle_lib.compute_directions(dims, vals)
        assert np.array_equal(d.asc, a) and np.array_equal(d.desc, b)
        lab = P.compute_labels(topo, d)
        M, m = oracle_lib.compute_labels(dims, a, b)
        assert np.array_equal(lab.max_label, M) and np.array_equal(lab.min_label, m)


@pytest.mark.parametrize("dims", [[31, 7, 9], [32, 64, 3], [33, 65, 17], [61, 60, 59], [1000, 3, 11],
                                  [3, 1000, 11], [130, 129, 2], [2, 2, 2]])
def test_k1_columns_vs_oracle_and_smem_k1(P, oracle_lib, dims, monkeypatch):
    """The 3D f32 K1 (k_directions_col3: 30-column warps, 8-row strips, z
    chunks) at column/row/plane boundaries, against the oracle and against the
    shared-memory K1 (k_directions_reg3, MSSZ_K1_REG3=1)."""
    rng = np.random.default_rng(11)
    topo = P.build_topology(dims)
    n = topo.vertex_count
    for vals in (rng.integers(-2, 3, n).astype(np.float32),
                 rng.choice(np.array([0.0, -0.0, 1.0, -1.0], np.float32), n),
                 rng.standard_normal(n).astype(np.float32)):
        codes = P.compute_direction_codes(topo, vals)
        d = P.compute_directions(topo, vals)
        a, b = oracle_lib.compute_directions(dims, vals)
        assert np.array_equal(d.asc, a) and np.array_equal(d.desc, b)
        monkeypatch.setenv("MSSZ_K1_REG3", "1")
        assert np.array_equal(P.compute_direction_codes(topo, vals), codes)
        monkeypatch.delenv("MSSZ_K1_REG3")


@pytest.mark.parametrize("dims", [[64, 48, 40], [96, 32, 33], [32, 16, 16], [48, 17, 31], [40, 20, 18]])
def test_label_tile_tma_vs_vector_loads(P, oracle_lib, dims, monkeypatch):
    """k_label_tile loads whole in-range 3D tiles with one TMA box
    (cp.async.bulk.tensor.3d on an mbarrier) when the field's strides allow it;
    labels must equal the vector-load path (MSSZ_LABEL_TMA=0) and the oracle,
    including partial tiles and fields whose strides rule TMA out."""
    from paper_2406_09423_b200 import inputs as I
    rng = np.random.default_rng(5)
    topo = P.build_topology(dims)
    for vals in (I.generate("random-smooth", dims, 3, np.float32),
                 rng.integers(0, 7, topo.vertex_count).astype(np.float32)):
        lab = P.segmentation(topo, vals)
        a, b = oracle_lib.compute_directions(dims, vals)
        M, m = oracle_lib.compute_labels(dims, a, b)
        assert np.array_equal(lab.max_label, M) and np.array_equal(lab.min_label, m)
        monkeypatch.setenv("MSSZ_LABEL_TMA", "0")
        assert P.segmentation(topo, vals) == lab
        monkeypatch.delenv("MSSZ_LABEL_TMA")


def test_signed_zero_ties(P):
    vals = np.array([0.0, -0.0] * 8, np.float32)
    topo = P.build_topology([4, 4])
    d = P.compute_directions(topo, vals)
    # all equal under SoS value order: the index decides
    assert P.classify_critical(d).maxima.tolist() == [15]
    assert P.classify_critical(d).minima.tolist() == [0]


def test_odd_cycle_internal(P):
    topo = P.build_topology([2, 2])
    dirs = P.DirectionField(np.array([1, 2, 0, 3], np.uint64), np.zeros(4, np.uint64))
    with pytest.raises(P.Error) as e:
        P.compute_labels(topo, dirs)
    assert e.value.kind() == P.ErrKind.internal


def test_detect_golden_and_kinds(P, golden, oracle_lib):
    meta, arr = golden
    for case in meta["detect"]:
        p = f"detect/{case['name']}/"
        topo = P.build_topology(case["dims"])
        rep = P.detect_false_critical(topo, arr[p + "f"], arr[p + "g"])
        for k, lst in enumerate([rep.fp_max, rep.fp_min, rep.fn_max, rep.fn_min]):
            assert np.array_equal(lst, arr[p + f"list{k}"])
    from paper_2406_09423_b200 import inputs as I
    for dims in ([96, 80], [20, 18, 16]):
        topo = P.build_topology(dims)
        f = I.generate("gaussian-mixture", dims, 3)
        xi = I.resolve_rel(f, 1e-2)
        fh = I.compress_base(dims, f, xi)
        rep = P.detect_false_critical(topo, f, fh)
        want = oracle_lib.detect_false_critical(dims, f, fh)
        for got, w in zip([rep.fp_max, rep.fp_min, rep.fn_max, rep.fn_min], want):
            assert np.array_equal(got, w)
        for kind in range(4):
            assert np.array_equal(P.detect_kind(topo, f, fh, kind),
                                  oracle_lib.detect_kind(dims, f, fh, kind))


def test_lower_step_golden(P, golden, oracle_lib):
    meta, arr = golden
    for case in meta["lower_step"]:
        dt = np.dtype(case["dtype"])
        trace = arr[f"ls/{case['name']}/trace"]
        f = np.array([case["f"]], dt)
        g = trace[:1].copy()
        for want in trace[1:]:
            g, moved = P.lower_step(g, f, case["xi"])
            assert moved[0] and g.tobytes() == np.array([want], dt).tobytes(), case["name"]
        _, moved = P.lower_step(g, f, case["xi"])
        assert not moved[0]
        fl = P.representable_floor(f, case["xi"])
        assert fl.tobytes() == arr[f"ls/{case['name']}/floor"].tobytes()
    # random bulk check against the oracle's scalar restatement
    rng = np.random.default_rng(3)
    for dt in (np.float32, np.float64):
        f = (rng.standard_normal(4096) * 10).astype(dt)
        xi = 0.37
        g = (f.astype(np.float64) + rng.uniform(-xi, xi, 4096)).astype(dt)
        out, moved = P.lower_step(g, f, xi)
        for i in range(0, 4096, 37):
            m, want = oracle_lib.lower_step(g[i], f[i], xi, dt)
            assert m == moved[i] and dt(want).tobytes() == out[i].tobytes()


# ------------------------------------------------------------------ derive_edits
def test_derive_golden_cases(P, golden, oracle_lib):
    meta, arr = golden
    for case in meta["derive"]:
        p = f"derive/{case['name']}/"
        topo = P.build_topology(case["dims"])
        f, fh, xi = arr[p + "f"], arr[p + "fhat"], case["xi"]
        st = P.EditStats()
        edits = P.derive_edits(topo, f, fh, xi, P.DeriveOptions(), st)
        jac = oracle_lib.derive_edits(case["dims"], f, fh, xi, schedule=O.JACOBI)
        # bit-exact vs the Jacobi oracle
        assert np.array_equal(edits.indices, jac.indices), case["name"]
        assert edits.values.tobytes() == jac.values.tobytes(), case["name"]
        assert stats_dict(st) == {k: jac.stats[k] for k in STAT_KEYS}, case["name"]
        # tolerance vs the serial reference
        ref_touched = case["stats"]["touched"]
        assert abs(st.touched - ref_touched) <= max(4, int(1e-4 * ref_touched)), case["name"]
        g = P.apply_edits(topo, fh, edits)
        check_postconditions(P, topo, f, g, xi)
        assert np.all(edits.values < fh[edits.indices])


CONFIG_CASES = [
    ("gaussian-mixture", [512, 512], 0, 1e-3, np.float32),   # C1
    ("random-smooth", [177, 95, 48], 0, 1e-3, np.float32),   # C2
    ("trig", [177, 95, 48], 0, 1e-4, np.float32),             # C2 (trig, 1e-4)
    ("gaussian-mixture", [360, 240], 0, 1e-4, np.float32),   # C5 shape, reduced
    ("gaussian-mixture", [48, 40, 24], 2, 1e-3, np.float64),
    # the bench workload's generator (C4 is 1024^3): big FPmin batches, parked
    # items and fallbacks inside the persistent subloop
    ("multi-scale", [96, 96, 48], 0, 1e-3, np.float32),
]


@pytest.mark.parametrize("kind,dims,seed,rel,dt", CONFIG_CASES)
def test_derive_configs_vs_oracle(P, oracle_lib, kind, dims, seed, rel, dt):
    from paper_2406_09423_b200 import inputs as I
    topo = P.build_topology(dims)
    f = I.generate(kind, dims, seed, dt)
    xi = I.resolve_rel(f, rel)
    fh = I.compress_base(dims, f, xi)
    cap = 100000
    st = P.EditStats()
    edits = P.derive_edits(topo, f, fh, xi, P.DeriveOptions(subloop_cap=cap), st)
    jac = oracle_lib.derive_edits(dims, f, fh, xi, subloop_cap=cap, schedule=O.JACOBI)
    assert np.array_equal(edits.indices, jac.indices)
    assert edits.values.tobytes() == jac.values.tobytes()
    assert stats_dict(st) == {k: jac.stats[k] for k in STAT_KEYS}
    check_postconditions(P, topo, f, P.apply_edits(topo, fh, edits), xi)


def test_on_batch_snapshots_match_oracle(P, oracle_lib):
    from paper_2406_09423_b200 import inputs as I
    dims = [40, 36]
    f = I.generate("trig", dims, 5, np.float64)
    xi = I.resolve_rel(f, 1e-2)
    fh = I.compress_base(dims, f, xi)
    topo = P.build_topology(dims)
    snaps = []
    P.derive_edits(topo, f, fh, xi, P.DeriveOptions(on_batch=snaps.append))
    jac = oracle_lib.derive_edits(dims, f, fh, xi, schedule=O.JACOBI, record_batches=True)
    assert len(snaps) == len(jac.batches) > 0
    prev = fh
    for got, want in zip(snaps, jac.batches):
        assert got.tobytes() == want.tobytes()
        assert np.all(got <= prev) and np.all(got > f - xi)  # test_edit_engine.cpp:244-251
        prev = got


def test_on_batch_snapshots_multiscale_3d(P, oracle_lib):
    """Per-batch g on a 3D multi-scale field (FPmin-heavy: parked items are merged
    back on every kernel exit in on_batch mode, and before each fallback)."""
    from paper_2406_09423_b200 import inputs as I
    dims = [24, 20, 12]
    f = I.generate("multi-scale", dims, 3, np.float32)
    xi = I.resolve_rel(f, 1e-3)
    fh = I.compress_base(dims, f, xi)
    topo = P.build_topology(dims)
    snaps = []
    st = P.EditStats()
    P.derive_edits(topo, f, fh, xi, P.DeriveOptions(on_batch=snaps.append, subloop_cap=100000), st)
    jac = oracle_lib.derive_edits(dims, f, fh, xi, subloop_cap=100000, schedule=O.JACOBI,
                                  record_batches=True)
    assert st.sub_iterations[1] > 0
    assert len(snaps) == len(jac.batches) > 0
    for got, want in zip(snaps, jac.batches):
        assert got.tobytes() == want.tobytes()


def test_derive_identity_and_errors(P):
    from paper_2406_09423_b200 import inputs as I
    dims = [12, 12]
    topo = P.build_topology(dims)
    f = I.generate("gaussian-mixture", dims, 7, np.float64)
    st = P.EditStats()
    assert P.derive_edits(topo, f, f, 0.01, None, st).empty()
    assert st.outer_iterations == 1  # test_edit_engine.cpp:187-196
    fh = f.copy()
    fh[10] += 1.0
    with pytest.raises(P.Error) as e:  # test_edit_engine.cpp:256-272
        P.derive_edits(topo, f, fh, 0.01)
    assert e.value.kind() == P.ErrKind.bound_violation
    st = P.EditStats()
    P.derive_edits(topo, f, fh, 1.0, P.DeriveOptions(force=True), st)
    with pytest.raises(P.Error) as e:
        P.derive_edits(topo, f, f, 0.0)
    assert e.value.kind() == P.ErrKind.usage
    bad = f.copy()
    bad[3] = np.nan
    with pytest.raises(P.Error) as e:
        P.derive_edits(topo, bad, f, 0.01)
    assert e.value.kind() == P.ErrKind.io


def test_caps_raise_non_convergence(P, oracle_lib):
    from paper_2406_09423_b200 import inputs as I
    dims = [16, 16]  # test_edit_engine.cpp:274-295
    f = I.generate("random-smooth", dims, 4, np.float64)
    xi = I.resolve_rel(f, 2e-2)
    fh = I.compress_base(dims, f, xi)
    topo = P.build_topology(dims)
    with pytest.raises(P.Error) as e:
        P.derive_edits(topo, f, fh, xi, P.DeriveOptions(outer_cap=0))
    assert e.value.kind() == P.ErrKind.non_convergence
    # subloop cap: the oracle and the GPU must fail the same way
    with pytest.raises(O.CheckerError) as eo:
        oracle_lib.derive_edits(dims, f, fh, xi, subloop_cap=1, schedule=O.JACOBI)
    with pytest.raises(P.Error) as e:
        P.derive_edits(topo, f, fh, xi, P.DeriveOptions(subloop_cap=1))
    assert e.value.kind() == P.ErrKind.non_convergence and eo.value.code == 5
    assert e.value.msg == eo.value.msg


def test_device_entry_point_matches_host(P):
    import torch
    from paper_2406_09423_b200 import inputs as I
    dims = [177, 95, 48]
    f = I.generate("random-smooth", dims, 0)
    xi = I.resolve_rel(f, 1e-3)
    fh = I.compress_base(dims, f, xi)
    topo = P.build_topology(dims)
    host = P.derive_edits(topo, f, fh, xi)
    df = torch.from_numpy(f).cuda()
    dfh = torch.from_numpy(fh).cuda()
    n = topo.vertex_count
    di = torch.empty(n, dtype=torch.int64, device="cuda")
    dv = torch.empty(n, dtype=torch.float32, device="cuda")
    count, st = P.derive_edits_device(topo, df.data_ptr(), dfh.data_ptr(), xi, di.data_ptr(),
                                      dv.data_ptr(), n, np.float32,
                                      stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert count == host.size()
    assert np.array_equal(di[:count].cpu().numpy().astype(np.uint64), host.indices)
    assert dv[:count].cpu().numpy().tobytes() == host.values.tobytes()
    # fhat on the device is untouched (the engine edits its own copy)
    assert dfh.cpu().numpy().tobytes() == fh.tobytes()


def test_profile_class_mask(P):
    """DeriveOptions.profile: True times every class, profile_mask(...) only the named ones."""
    from paper_2406_09423_b200 import inputs as I
    dims = [64, 48, 24]
    f = I.generate("random-smooth", dims, 1, np.float32)
    xi = I.resolve_rel(f, 1e-3)
    fh = I.compress_base(dims, f, xi)
    topo = P.build_topology(dims)
    full, only = P.EditStats(), P.EditStats()
    a = P.derive_edits(topo, f, fh, xi, P.DeriveOptions(profile=True), full)
    b = P.derive_edits(topo, f, fh, xi, P.DeriveOptions(profile=P.profile_mask("directions")), only)
    assert np.array_equal(a.indices, b.indices) and a.values.tobytes() == b.values.tobytes()
    kf, ko = full.kernel_profile(), only.kernel_profile()
    assert sum(1 for v in kf.values() if v["ms"] > 0) >= 3
    assert ko["directions"]["ms"] > 0
    assert all(v["ms"] == 0 for k, v in ko.items() if k != "directions")
    assert ko["directions"]["launches"] == kf["directions"]["launches"]

"""Parity of the R-batch targets and of real correction states (not only inputs).

* R-batch target sets (run_r_loop's collect_mismatched + find_troublemaker +
  claim, edit_engine.cpp:336-352) from the engine's tiled pass AND its sparse
  Up(X) pass, against the unmodified reference (oracle/_ref) on the golden
  troublemaker KATs (test_edit_engine.cpp:138-185) and on g snapshots taken
  inside real corrections (DeriveOptions.on_batch_mode = "phases": after every
  C pass and every R iteration).
* Per-kernel parity on those snapshots: directions (mss.cpp:11-30), the
  false-critical report (edit_engine.cpp:134-158), labels (mss.cpp:84-97).
* The C2 error-bound sweep (BASELINE configs[1]: rel 1e-4 .. 1e-2, random-smooth
  and trig): bit-exact against the Jacobi oracle, EditStats against the
  reference within the stated tolerance.
* on_batch exceptions abort the correction and propagate (edit_engine.cpp:275).
"""
import numpy as np
import pytest

import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]

STAT_KEYS = ("outer_iterations", "c_passes", "sub_iterations", "r_iterations",
             "effective_edits", "touched")


@pytest.fixture(scope="module")
def P(mssz):
    if mssz.library().mssz_cu_device_count() == 0:
        pytest.fail("no CUDA device visible to the GPU test suite")
    return mssz


def touched_tolerance(ref_touched: int) -> int:
    """|touched - ref| <= max(4, 1e-4 * ref)."""
    return max(4, int(1e-4 * ref_touched))


def check_r_targets(P, ref_lib, dims, f, g, modes=("tiled", "sparse")):
    """GPU R-batch targets == the reference's (both behind the R gate: a pair with
    false critical points has no R batch, edit_engine.cpp:338)."""
    topo = P.build_topology(dims)
    want, false_cp, sources, _mism = ref_lib.r_targets(dims, f, g)
    paths = []
    for mode in modes:
        got = P.r_targets(topo, f, g, mode)
        assert got.false_critical == false_cp
        assert np.array_equal(got.targets, want), (mode, got.targets.size, want.size)
        assert got.sources == sources, mode
        paths.append(got.path)
    if false_cp:
        assert want.size == 0
    return want, paths


def check_kernels(P, ref_lib, dims, f, g):
    """Directions, false-critical report and labels of a snapshot vs the reference."""
    topo = P.build_topology(dims)
    d = P.compute_directions(topo, g)
    a, b = ref_lib.compute_directions(dims, g, threads=0)
    assert np.array_equal(d.asc, a) and np.array_equal(d.desc, b)
    rep = P.detect_false_critical(topo, f, g)
    want = ref_lib.detect_false_critical(dims, f, g)
    for got, w in zip([rep.fp_max, rep.fp_min, rep.fn_max, rep.fn_min], want):
        assert np.array_equal(got, w)
    lab = P.compute_labels(topo, d)
    M, m = ref_lib.compute_labels(dims, a, b, threads=0)
    assert np.array_equal(lab.max_label, M) and np.array_equal(lab.min_label, m)


# --------------------------------------------------------------- troublemaker KATs
def test_troublemaker_kats_r_targets(P, golden, ref_lib):
    """test_edit_engine.cpp:138-185: the golden (v_i, v_t) of the walk from v = 4 is
    one of the batch's targets, and the whole target set equals the reference's."""
    meta, arr = golden
    for case in meta["troublemaker"]:
        f = arr[f"tm/{case['name']}/f"]
        g = arr[f"tm/{case['name']}/g"]
        want, paths = check_r_targets(P, ref_lib, case["dims"], f, g)
        assert case["vt"] in want.tolist(), case["name"]


# --------------------------------------------------------------- snapshots
SNAPSHOT_CASES = [
    ("multi-scale", [96, 96, 48], 0, 1e-3, np.float32),
    ("random-smooth", [177, 95, 48], 0, 1e-2, np.float32),
    ("gaussian-mixture", [512, 512], 0, 1e-3, np.float32),
    ("trig", [64, 48, 40], 1, 1e-2, np.float64),
]


@pytest.mark.parametrize("kind,dims,seed,rel,dt", SNAPSHOT_CASES)
def test_snapshots_r_targets_and_kernels(P, ref_lib, kind, dims, seed, rel, dt):
    from paper_2406_09423_b200 import inputs as I
    topo = P.build_topology(dims)
    f = I.generate(kind, dims, seed, dt)
    xi = I.resolve_rel(f, rel)
    fh = I.compress_base(dims, f, xi)
    snaps, kinds = [], []

    def keep(g):
        snaps.append(g)
        kinds.append(P.batch_phase()[0])

    st = P.EditStats()
    P.derive_edits(topo, f, fh, xi, P.DeriveOptions(subloop_cap=100000, on_batch=keep,
                                                    on_batch_mode="phases"), st)
    # one snapshot per C pass and per R iteration
    assert len(snaps) == st.c_passes + st.r_iterations
    picks = sorted({0, 1, len(snaps) // 2, len(snaps) - 2, len(snaps) - 1} & set(range(len(snaps))))
    # the states every R iteration starts from: after the C loop (the last C
    # pass before an R iteration) and after each R iteration
    picks += [i for i in range(len(snaps) - 1) if kinds[i] == "c_pass" and kinds[i + 1] == "r_iteration"]
    nonempty = 0
    for i in sorted(set(picks)):
        g = snaps[i]
        want, _ = check_r_targets(P, ref_lib, dims, f, g)
        nonempty += want.size > 0
        check_kernels(P, ref_lib, dims, f, g)
    assert nonempty > 0  # at least one picked state has a real R batch


def test_phase_snapshots_are_batch_states(P):
    """Every phase snapshot is the state after some per-batch snapshot (same run)."""
    from paper_2406_09423_b200 import inputs as I
    dims = [40, 36, 12]
    f = I.generate("random-smooth", dims, 2, np.float32)
    xi = I.resolve_rel(f, 1e-2)
    fh = I.compress_base(dims, f, xi)
    topo = P.build_topology(dims)
    every, phases = [], []
    e1 = P.derive_edits(topo, f, fh, xi, P.DeriveOptions(on_batch=every.append))
    e2 = P.derive_edits(topo, f, fh, xi, P.DeriveOptions(on_batch=phases.append,
                                                         on_batch_mode="phases"))
    assert np.array_equal(e1.indices, e2.indices) and e1.values.tobytes() == e2.values.tobytes()
    seen = {s.tobytes() for s in every} | {fh.tobytes()}
    assert phases and all(p.tobytes() in seen for p in phases)
    assert phases[-1].tobytes() == P.apply_edits(topo, fh, e2).tobytes()


def test_on_batch_exception_propagates(P):
    """An exception raised by on_batch aborts derive_edits and reaches the caller."""
    from paper_2406_09423_b200 import inputs as I
    dims = [64, 48]
    f = I.generate("gaussian-mixture", dims, 1, np.float32)
    xi = I.resolve_rel(f, 1e-2)
    fh = I.compress_base(dims, f, xi)
    topo = P.build_topology(dims)
    calls = []

    class Stop(Exception):
        pass

    def cb(g):
        calls.append(1)
        if len(calls) == 2:
            raise Stop("second batch")

    with pytest.raises(Stop):
        P.derive_edits(topo, f, fh, xi, P.DeriveOptions(on_batch=cb))
    assert len(calls) == 2
    # the engine is reusable afterwards and still bit-exact
    a = P.derive_edits(topo, f, fh, xi)
    b = P.derive_edits(topo, f, fh, xi, P.DeriveOptions(on_batch=lambda g: None))
    assert np.array_equal(a.indices, b.indices) and a.values.tobytes() == b.values.tobytes()


# --------------------------------------------------------------- C2 error-bound sweep
SWEEP = [(k, rel) for k in ("random-smooth", "trig") for rel in (1e-4, 1e-3, 1e-2)]


@pytest.mark.parametrize("kind,rel", SWEEP)
def test_c2_error_bound_sweep(P, oracle_lib, ref_lib, kind, rel):
    """BASELINE configs[1] (177x95x48, rel 1e-4..1e-2) at the reference's default caps."""
    from paper_2406_09423_b200 import inputs as I
    dims = [177, 95, 48]
    topo = P.build_topology(dims)
    f = I.generate(kind, dims, 0)
    xi = I.resolve_rel(f, rel)
    fh = I.compress_base(dims, f, xi)
    st = P.EditStats()
    edits = P.derive_edits(topo, f, fh, xi, P.DeriveOptions(), st)
    jac = oracle_lib.derive_edits(dims, f, fh, xi, schedule=O.JACOBI)
    assert np.array_equal(edits.indices, jac.indices)
    assert edits.values.tobytes() == jac.values.tobytes()
    assert {k: getattr(st, k) for k in STAT_KEYS} == {k: jac.stats[k] for k in STAT_KEYS}
    ref = ref_lib.derive_edits(dims, f, fh, xi, threads=0)
    assert abs(st.touched - ref.stats["touched"]) <= touched_tolerance(ref.stats["touched"])
    g = P.apply_edits(topo, fh, edits)
    assert np.all(np.abs(g.astype(np.float64) - f.astype(np.float64)) <= xi)
    assert P.segmentation(topo, g) == P.segmentation(topo, f)


# --------------------------------------------------------------- apply_edits semantics
def test_apply_edits_order_and_range(P):
    """apply_edits (edit_engine.cpp:437-450): in-order application (last value wins
    for a repeated index); an out-of-range index raises corrupt_archive."""
    topo = P.build_topology([8, 8])
    fh = np.arange(64, dtype=np.float32)
    sorted_dup = P.EditSet(np.array([3, 3, 3, 9, 20, 20], np.uint64),
                           np.array([1, 2, 3, 4, 5, 6], np.float32))
    g = P.apply_edits(topo, fh, sorted_dup)
    assert g[3] == 3 and g[9] == 4 and g[20] == 6
    unsorted_dup = P.EditSet(np.array([20, 3, 9, 3, 20, 3], np.uint64),
                             np.array([1, 2, 3, 4, 5, 6], np.float32))
    g = P.apply_edits(topo, fh, unsorted_dup)
    assert g[3] == 6 and g[9] == 3 and g[20] == 5
    bad = P.EditSet(np.array([1, 64], np.uint64), np.array([0, 0], np.float32))
    with pytest.raises(P.Error) as e:
        P.apply_edits(topo, fh, bad)
    assert e.value.kind() == P.ErrKind.corrupt_archive


def test_batch_phase_reports_snapshot_kind(P):
    """mssz_cu_batch_phase inside on_batch: C passes then R iterations per outer iteration."""
    from paper_2406_09423_b200 import inputs as I
    dims = [48, 40, 16]
    f = I.generate("random-smooth", dims, 3, np.float32)
    xi = I.resolve_rel(f, 1e-2)
    fh = I.compress_base(dims, f, xi)
    topo = P.build_topology(dims)
    seen = []
    st = P.EditStats()
    P.derive_edits(topo, f, fh, xi, P.DeriveOptions(on_batch=lambda g: seen.append(P.batch_phase()),
                                                    on_batch_mode="phases"), st)
    assert sum(k == "c_pass" for k, _, _ in seen) == st.c_passes
    assert sum(k == "r_iteration" for k, _, _ in seen) == st.r_iterations
    assert max(o for _, o, _ in seen) == st.outer_iterations
    every = []
    P.derive_edits(topo, f, fh, xi, P.DeriveOptions(on_batch=lambda g: every.append(P.batch_phase())))
    assert sum(k == "batch" for k, _, _ in every) == sum(st.sub_iterations)
    assert sum(k == "r_iteration" for k, _, _ in every) == st.r_iterations


def test_skipped_subloops_are_empty(P, oracle_lib, monkeypatch):
    """ADVICE: a subloop skipped as provably empty (code epoch unchanged) is
    re-checked by a full detection sweep under MSSZ_CHECK_SKIPS; the run must
    still be bit-exact with the Jacobi oracle and must have skipped some."""
    from paper_2406_09423_b200 import inputs as I
    monkeypatch.setenv("MSSZ_CHECK_SKIPS", "1")
    dims = [96, 96, 48]
    f = I.generate("multi-scale", dims, 0, np.float32)
    xi = I.resolve_rel(f, 1e-3)
    fh = I.compress_base(dims, f, xi)
    topo = P.build_topology(dims)
    st = P.EditStats()
    e = P.derive_edits(topo, f, fh, xi, P.DeriveOptions(subloop_cap=100000), st)
    jac = oracle_lib.derive_edits(dims, f, fh, xi, subloop_cap=100000, schedule=O.JACOBI)
    assert st.skipped_subloops > 0
    assert np.array_equal(e.indices, jac.indices) and e.values.tobytes() == jac.values.tobytes()
    assert {k: getattr(st, k) for k in STAT_KEYS} == {k: jac.stats[k] for k in STAT_KEYS}

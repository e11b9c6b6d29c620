"""z-slab sharding on one GPU: P virtual ranks (host threads, the
in-process transport) must reproduce the single-device engine bit-for-bit --
edit set, values and every EditStats counter -- which itself matches the
oracle's Jacobi schedule (test_gpu_parity.py).  The multi-process NCCL path runs
the same SlabEngine with a different Transport."""
import numpy as np
import pytest

import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]

STAT_KEYS = ("outer_iterations", "c_passes", "sub_iterations", "r_iterations",
             "effective_edits", "touched", "input_bound_violations")


@pytest.fixture(scope="module")
def P(mssz):
    if mssz.library().mssz_cu_device_count() == 0:
        pytest.fail("no CUDA device visible to the GPU test suite")
    return mssz


def stats_dict(st):
    return {k: getattr(st, k) for k in STAT_KEYS}


CASES = [
    ("random-smooth", [177, 95, 48], 0, 1e-3, np.float32, (1, 2, 3, 5, 8)),   # C2
    ("trig", [177, 95, 48], 0, 1e-4, np.float32, (2, 4)),                     # C2 trig, 1e-4
    ("multi-scale", [64, 64, 64], 0, 1e-3, np.float32, (2, 4, 8)),            # C4 shape, reduced
    ("gaussian-mixture", [48, 40, 24], 2, 1e-3, np.float64, (2, 3, 12)),      # f64, 2-plane slabs
    ("random-smooth", [40, 30, 20], 3, 1e-2, np.float32, (2, 4)),             # large batches
]


@pytest.mark.parametrize("kind,dims,seed,rel,dt,slabs", CASES)
def test_slabs_match_single_device(P, kind, dims, seed, rel, dt, slabs):
    from paper_2406_09423_b200 import inputs as I
    topo = P.build_topology(dims)
    f = I.generate(kind, dims, seed, dt)
    xi = I.resolve_rel(f, rel)
    fh = I.compress_base(dims, f, xi)
    opts = P.DeriveOptions(subloop_cap=100000)
    st1 = P.EditStats()
    one = P.derive_edits(topo, f, fh, xi, opts, st1)
    for p in slabs:
        st = P.EditStats()
        got = P.derive_edits_slabs(topo, f, fh, xi, p, opts, st)
        assert np.array_equal(got.indices, one.indices), p
        assert got.values.tobytes() == one.values.tobytes(), p
        assert stats_dict(st) == stats_dict(st1), p


def test_slabs_match_oracle_small(P, oracle_lib):
    from paper_2406_09423_b200 import inputs as I
    dims = [20, 18, 16]
    f = I.generate("trig", dims, 5, np.float64)
    xi = I.resolve_rel(f, 1e-2)
    fh = I.compress_base(dims, f, xi)
    topo = P.build_topology(dims)
    jac = oracle_lib.derive_edits(dims, f, fh, xi, subloop_cap=100000, schedule=O.JACOBI)
    for p in (2, 4, 8):
        st = P.EditStats()
        got = P.derive_edits_slabs(topo, f, fh, xi, p, P.DeriveOptions(subloop_cap=100000), st)
        assert np.array_equal(got.indices, jac.indices)
        assert got.values.tobytes() == jac.values.tobytes()
        assert {k: getattr(st, k) for k in STAT_KEYS[:-1]} == {k: jac.stats[k] for k in STAT_KEYS[:-1]}


def test_slab_errors_match_single_device(P):
    from paper_2406_09423_b200 import inputs as I
    dims = [16, 16, 12]
    topo = P.build_topology(dims)
    f = I.generate("random-smooth", dims, 4, np.float64)
    xi = I.resolve_rel(f, 2e-2)
    fh = I.compress_base(dims, f, xi)
    for opts in (P.DeriveOptions(outer_cap=0), P.DeriveOptions(subloop_cap=1)):
        with pytest.raises(P.Error) as e1:
            P.derive_edits(topo, f, fh, xi, opts)
        with pytest.raises(P.Error) as e2:
            P.derive_edits_slabs(topo, f, fh, xi, 3, opts)
        assert e1.value.kind() == e2.value.kind() == P.ErrKind.non_convergence
        assert e1.value.msg == e2.value.msg
    bad = fh.copy()
    bad[7 * 256 + 5] += 1.0
    with pytest.raises(P.Error) as e:
        P.derive_edits_slabs(topo, f, bad, xi, 2)
    assert e.value.kind() == P.ErrKind.bound_violation
    with pytest.raises(P.Error) as e:
        P.derive_edits_slabs(topo, f, fh, 0.0, 2)
    assert e.value.kind() == P.ErrKind.usage
    with pytest.raises(P.Error) as e:  # slabs need >= 2 planes
        P.derive_edits_slabs(topo, f, fh, xi, 7)
    assert e.value.kind() == P.ErrKind.usage
    nan = f.copy()
    nan[-1] = np.nan
    with pytest.raises(P.Error) as e:
        P.derive_edits_slabs(topo, nan, fh, xi, 2)
    assert e.value.kind() == P.ErrKind.io
    assert P.derive_edits_slabs(topo, f, f, xi, 3).empty()


def test_slab_comm_single_rank(P):
    """The NCCL transport end to end with one rank (the only NCCL shape one GPU allows)."""
    from paper_2406_09423_b200 import inputs as I
    dims = [64, 48, 32]
    f = I.generate("multi-scale", dims, 1, np.float32)
    xi = I.resolve_rel(f, 1e-3)
    fh = I.compress_base(dims, f, xi)
    topo = P.build_topology(dims)
    st1 = P.EditStats()
    one = P.derive_edits(topo, f, fh, xi, P.DeriveOptions(subloop_cap=100000), st1)
    comm = P.SlabComm(P.SlabComm.unique_id(), 1, 0, 0)
    st = P.EditStats()
    got, off = comm.derive_edits(dims, f, fh, xi, P.DeriveOptions(subloop_cap=100000), st)
    comm.close()
    assert off == 0
    assert np.array_equal(got.indices, one.indices)
    assert got.values.tobytes() == one.values.tobytes()
    assert stats_dict(st) == stats_dict(st1)


@pytest.mark.parametrize("kind,dims,seed,rel,dt,slabs", [
    ("random-smooth", [40, 30, 20], 3, 1e-2, np.float32, (1, 2, 4)),
    ("multi-scale", [48, 40, 32], 0, 1e-3, np.float32, (3, 8)),
])
def test_slabs_global_ids_beyond_u32(P, monkeypatch, kind, dims, seed, rel, dt, slabs):
    """Global ids are u64 in the sharded engine (the reference caps grids at 2^40,
    grid.cpp:19, not 2^32).  MSSZ_SLAB_Z_BIAS places the field that many planes
    deep in a larger virtual grid, so every boundary edit, label-table entry and
    resolved label carries a global id >= 2^32; any truncation to 32 bits would
    break the table lookups and label comparisons."""
    from paper_2406_09423_b200 import inputs as I
    topo = P.build_topology(dims)
    f = I.generate(kind, dims, seed, dt)
    xi = I.resolve_rel(f, rel)
    fh = I.compress_base(dims, f, xi)
    opts = P.DeriveOptions(subloop_cap=100000)
    st1 = P.EditStats()
    one = P.derive_edits(topo, f, fh, xi, opts, st1)
    xy = dims[0] * dims[1]
    monkeypatch.setenv("MSSZ_SLAB_Z_BIAS", str((1 << 32) // xy + 7))
    for p in slabs:
        st = P.EditStats()
        got = P.derive_edits_slabs(topo, f, fh, xi, p, opts, st)
        assert np.array_equal(got.indices, one.indices), p
        assert got.values.tobytes() == one.values.tobytes(), p
        assert stats_dict(st) == stats_dict(st1), p


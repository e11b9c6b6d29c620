"""Edit-set encoding on the GPU against the reference's own
encode_edits (edit_codec.cpp:188-222, compiled into oracle/_ref): byte-identical
payloads for both backends, including multi-byte varints, long runs (> 65535,
the RLE chunk cap), the RLE marker byte itself, and the empty set."""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]


@pytest.fixture(scope="module")
def P(mssz):
    if mssz.library().mssz_cu_device_count() == 0:
        pytest.fail("no CUDA device visible to the GPU test suite")
    return mssz


def edit_sets():
    rng = np.random.default_rng(11)
    yield "empty", np.array([], np.uint64), np.array([], np.float32)
    yield "one", np.array([7], np.uint64), np.array([1.5], np.float32)
    # small gaps (1-byte varints), long equal runs and the RLE marker (delta 245 -> byte 0xF5)
    d = np.concatenate([np.ones(70000, np.uint64), np.full(3, 245, np.uint64),
                        rng.integers(1, 9, 5000).astype(np.uint64), np.full(65535 * 2 + 3, 2, np.uint64),
                        np.array([2, 2, 2, 3, 0xF5, 0xF5], np.uint64)])
    idx = np.cumsum(d) - 1
    yield "runs", idx.astype(np.uint64), rng.random(idx.size).astype(np.float32)
    # large gaps: multi-byte varints up to 2^40
    d = rng.integers(1, 1 << 40, 3000, dtype=np.uint64)
    idx = np.cumsum(d)
    yield "wide", idx.astype(np.uint64), rng.standard_normal(idx.size)
    # a realistic edit set: sorted random subset of a 2^24 grid
    idx = np.unique(rng.integers(0, 1 << 24, 400000)).astype(np.uint64)
    yield "subset", idx, rng.standard_normal(idx.size).astype(np.float32)


@pytest.mark.parametrize("codec", [0, 1])
def test_encode_edits_byte_identical(P, ref_lib, codec):
    for name, idx, val in edit_sets():
        got = P.encode_edits(P.EditSet(idx, val), codec)
        want = ref_lib.encode_edits(idx, val, codec)
        assert got == want, (name, codec, len(got), len(want))


def test_encode_edits_from_derive(P, ref_lib):
    from paper_2406_09423_b200 import inputs as I
    dims = [96, 80, 40]
    f = I.generate("multi-scale", dims, 3)
    xi = I.resolve_rel(f, 1e-3)
    fh = I.compress_base(dims, f, xi)
    edits = P.derive_edits(P.build_topology(dims), f, fh, xi, P.DeriveOptions(subloop_cap=100000))
    assert edits.size() > 1000
    for codec in (0, 1):
        assert P.encode_edits(edits, codec) == ref_lib.encode_edits(edits.indices, edits.values, codec)


def test_encode_edits_errors(P):
    with pytest.raises(P.Error) as e:  # edit_codec.cpp:31-33
        P.encode_edits(P.EditSet(np.array([5, 5], np.uint64), np.zeros(2, np.float32)))
    assert e.value.kind() == P.ErrKind.usage
    with pytest.raises(P.Error) as e:  # parse_backend (edit_codec.cpp:22-25)
        P.encode_edits(P.EditSet(np.array([1], np.uint64), np.zeros(1, np.float32)), codec=2)
    assert e.value.kind() == P.ErrKind.corrupt_archive

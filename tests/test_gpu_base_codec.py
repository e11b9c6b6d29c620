"""GPU base codec against the reference's compress_base
reconstruction (restated bit-exactly in csrc/inputs.cpp and pinned against the
reference by tests/test_inputs.py): reconstruction bit-identical, escape count
identical, and decompress(symbols, literals) == the reconstruction."""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]


@pytest.fixture(scope="module")
def P(mssz):
    if mssz.library().mssz_cu_device_count() == 0:
        pytest.fail("no CUDA device visible to the GPU test suite")
    return mssz


@pytest.mark.parametrize("kind,dims,rel,dt", [
    ("gaussian-mixture", [512, 512], 1e-3, np.float32),       # C1
    ("random-smooth", [177, 95, 48], 1e-3, np.float32),       # C2
    ("trig", [177, 95, 48], 1e-4, np.float32),
    ("multi-scale", [64, 64, 64], 1e-3, np.float32),
    ("gaussian-mixture", [33, 29, 17], 1e-2, np.float64),
    ("random-smooth", [360, 240], 1e-4, np.float32),          # C5 shape, reduced
    ("trig", [17, 3, 2], 1e-2, np.float64),
    ("gaussian-mixture", [40, 36], 1e-7, np.float64),          # escapes (residual beyond the radius)
])
def test_base_codec_matches_reference(P, kind, dims, rel, dt):
    from paper_2406_09423_b200 import inputs as I
    topo = P.build_topology(dims)
    f = I.generate(kind, dims, 5, dt)
    xi = I.resolve_rel(f, rel)
    want = I.compress_base(dims, f, xi)
    recon, sym, lits = P.compress_base(topo, f, xi)
    assert recon.tobytes() == want.tobytes()
    assert recon[sym == 0].tobytes() == f[sym == 0].tobytes()  # escapes keep the value
    back = P.decompress_base(topo, sym, lits, xi, dt)
    assert back.tobytes() == recon.tobytes()
    assert np.all(np.abs(recon.astype(np.float64) - f.astype(np.float64)) <= xi)


def test_base_codec_errors(P):
    topo = P.build_topology([8, 8])
    f = np.linspace(0, 1, 64)
    recon, sym, lits = P.compress_base(topo, f, 1e-3)
    with pytest.raises(P.Error) as e:  # literal count mismatch (base_codec.cpp:141-151)
        P.decompress_base(topo, np.zeros(64, np.uint32), lits, 1e-3, np.float64)
    assert e.value.kind() == P.ErrKind.corrupt_archive
    with pytest.raises(P.Error) as e:
        P.compress_base(topo, f, 0.0)
    assert e.value.kind() == P.ErrKind.usage
    bad = f.copy()
    bad[5] = np.inf
    with pytest.raises(P.Error) as e:
        P.compress_base(topo, bad, 1e-3)
    assert e.value.kind() == P.ErrKind.io

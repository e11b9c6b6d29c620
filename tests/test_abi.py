"""CPU: the C-ABI library loads, exports every symbol include/mssz_cuda.h declares,
and fails loudly (no CPU fallback) when no CUDA device is present."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "mssz_cuda.h")).read()
    names = set()
    for m in re.finditer(r"\b(mssz_cu_\w+?)(##SUF)?\(", text):
        if m.group(2):
            names.update({m.group(1) + "f32", m.group(1) + "f64"})
        else:
            names.add(m.group(1))
    names.discard("mssz_cu_")
    return names


def test_exports_match_header(mssz):
    lib = mssz.library()
    declared = header_symbols()
    assert declared == set(mssz.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name


def test_version_and_defaults(mssz):
    import ctypes as C
    lib = mssz.library()
    assert b"sm_100a" in lib.mssz_cu_version()
    o = mssz._Options()
    lib.mssz_cu_default_options(C.byref(o))
    assert (o.outer_cap, o.subloop_cap, o.r_cap, o.force, o.device) == (1000, 640, 100000, 0, -1)


def test_no_cpu_fallback(mssz):
    if mssz.library().mssz_cu_device_count() > 0:
        pytest.skip("a CUDA device is present")
    topo = mssz.build_topology([8, 8])
    f = np.zeros(64, np.float32)
    with pytest.raises(mssz.Error) as e:
        mssz.derive_edits(topo, f, f, 0.1)
    assert e.value.kind() == mssz.ErrKind.cuda
    with pytest.raises(mssz.Error):
        mssz.compute_directions(topo, f)


@pytest.mark.parametrize("dims", [[1, 4], [7], [2, 2, 2, 2], [1 << 21, 1 << 21, 4]])
def test_build_topology_usage_errors(mssz, dims):
    # test_grid.cpp:34-51
    with pytest.raises(mssz.Error) as e:
        mssz.build_topology(dims)
    assert e.value.kind() == mssz.ErrKind.usage


def test_topology_round_trip(mssz):
    t = mssz.build_topology([4, 5, 3])
    for v in range(t.vertex_count):
        assert t.index_of(*t.coords_of(v)) == v


def test_exported_sizes_in_ctypes(mssz):
    import ctypes as C
    # the ctypes mirrors must have the C layout: 3 u64 + 2 i32 + 2 pointers
    assert C.sizeof(mssz._Options) == 24 + 8 + 16 + 8
    assert C.sizeof(mssz._Stats) == 8 * 10 + 8 * 5 + 8 * 5 + 80 + 16 * 8 * 2

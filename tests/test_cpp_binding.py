"""The reference-signature C++ binding (include/mssz_b200.hpp) compiles, links
against the in-tree C-ABI library, fails loudly without a GPU (ErrKind 99) and
corrects a field on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def example(mssz, tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cpp") / "derive_example")
    libdir = os.path.dirname(mssz.CUDA_SO)
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "derive_example.cpp"), "-o", out,
           f"-L{libdir}", "-l:libmssz_b200.so", f"-Wl,-rpath,{libdir}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_cpp_example_fails_loudly_without_gpu(mssz, example):
    if mssz.library().mssz_cu_device_count() > 0:
        pytest.skip("GPU present")
    r = subprocess.run([example], capture_output=True, text=True)
    assert r.returncode == 99, (r.stdout, r.stderr)
    assert "no CUDA device" in r.stderr


@pytest.mark.gpu
def test_cpp_example_on_gpu(mssz, example, tmp_path, ref_lib):
    r = subprocess.run([example, str(tmp_path)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, (r.stdout, r.stderr)
    assert r.stdout.startswith("ok")
    # the payload the C++ binding produced equals the reference encoder's bytes
    import numpy as np
    idx = np.fromfile(tmp_path / "indices.u64", np.uint64)
    val = np.fromfile(tmp_path / "values.f32", np.float32)
    payload = (tmp_path / "payload.bin").read_bytes()
    assert idx.size > 0
    assert payload == ref_lib.encode_edits(idx, val, 1)

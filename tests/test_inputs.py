"""CPU: the parallel input producers (generators + base-codec reconstruction) are
bit-identical to the reference's (golden hashes; live reference when built)."""
import hashlib

import numpy as np
import pytest

from paper_2406_09423_b200 import inputs as I


def test_generator_and_codec_hashes(golden, mssz):
    meta, _ = golden
    for case in meta["hashes"]:
        dt = np.dtype(case["dtype"])
        f = I.generate(case["kind"], case["dims"], case["seed"], dt)
        assert hashlib.sha256(f.tobytes()).hexdigest() == case["f_sha256"], case
        xi = I.resolve_rel(f, case["rel"])
        assert xi == case["xi"]
        fh = I.compress_base(case["dims"], f, xi)
        assert hashlib.sha256(fh.tobytes()).hexdigest() == case["fhat_sha256"], case


def test_golden_derive_inputs_reproduce(golden, mssz):
    meta, arr = golden
    for case in meta["derive"]:
        if case["rel"] is None:
            continue
        dt = np.dtype(case["dtype"])
        f = I.generate(case["kind"], case["dims"], case["seed"], dt)
        assert f.tobytes() == arr[f"derive/{case['name']}/f"].tobytes()
        fh = I.compress_base(case["dims"], f, case["xi"])
        assert fh.tobytes() == arr[f"derive/{case['name']}/fhat"].tobytes()


@pytest.mark.parametrize("kind", ["gaussian-mixture", "trig", "random-smooth"])
@pytest.mark.parametrize("dims", [[33, 17], [9, 8, 7]])
def test_live_reference(ref_lib, mssz, kind, dims):
    for dt in (np.float32, np.float64):
        a = ref_lib.generate(kind, dims, 9, dt)
        b = I.generate(kind, dims, 9, dt)
        assert a.tobytes() == b.tobytes()
        xi = ref_lib.resolve_rel(dims, a, 1e-2)
        assert xi == I.resolve_rel(b, 1e-2)
        assert ref_lib.compress_base(dims, a, xi).tobytes() == I.compress_base(dims, b, xi).tobytes()


def test_multiscale_is_sum_in_double(mssz):
    dims = [10, 9, 8]
    f = I.generate("multi-scale", dims, 0, np.float64, a=0.2)
    gm = I.generate("gaussian-mixture", dims, 0, np.float64)
    rs = I.generate("random-smooth", dims, 1, np.float64)
    assert np.array_equal(f, gm + 0.2 * rs)

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as fp:
        meta = json.load(fp)
    arrays = dict(np.load(os.path.join(GOLDEN, "golden.npz")))
    return meta, arrays


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle as O
    if not os.path.exists(O.ORACLE_SO):
        O.build()
    return O.oracle()


@pytest.fixture(scope="session")
def ref_lib():
    import oracle as O
    if not O.have_ref():
        if os.path.isdir(O.REFERENCE_SRC):
            O.build()
        else:
            pytest.skip("reference library not built and /root/reference absent")
    return O.ref()


@pytest.fixture(scope="session")
def mssz():
    import paper_2406_09423_b200 as P
    P.build()
    return P

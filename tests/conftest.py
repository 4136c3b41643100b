import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "ref_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture(scope="session")
def ora():
    import oracle

    if not oracle.oracle_available():
        oracle.build(ref=False)
    return oracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle

    if not oracle.ref_available():
        if os.path.isdir("/root/reference/proj/core/src"):
            oracle.build(ref=True)
        else:
            pytest.skip("reference build (oracle/_ref) unavailable on this host")
    return oracle.Ref()


@pytest.fixture(scope="session")
def sk():
    import paper_2408_11235_b200 as sk

    return sk

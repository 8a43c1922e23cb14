import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(ROOT, "tests", "golden", "reference_vectors.npz"))


@pytest.fixture(scope="session")
def port():
    import oracle
    return oracle.load("port")


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference (oracle/_ref); skipped where it was never built."""
    import oracle
    if not (oracle.available("ref") or os.path.isdir(oracle.REF_SRC)):
        pytest.skip("oracle/_ref/libspeig_ref.so not available")
    return oracle.load("ref")


@pytest.fixture(scope="session")
def best_oracle():
    import oracle
    return oracle.best()


@pytest.fixture(scope="session")
def ctx():
    from paper_2409_15053_b200 import Context
    c = Context()
    yield c
    c.close()

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")


@pytest.fixture(scope="session")
def oracle():
    """Our C restatement of the reference path (test infrastructure)."""
    from oracle import Oracle, build
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        build(ref=True)
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    """The reference library itself, compiled from /root/reference (oracle/_ref)."""
    from oracle import Reference, build
    if not Reference.available() and os.path.isdir("/root/reference/proj"):
        build(ref=True)
    if not Reference.available():
        pytest.skip("oracle/_ref/libidkit_ref.so not built (reference sources absent)")
    return Reference()


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    d = np.linalg.norm(a - b)
    nb = np.linalg.norm(b)
    return d / nb if nb > 0 else d

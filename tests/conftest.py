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


# ---- parity records (profiles/parity_r02.json is copied from this file) ----------
_PARITY = {}


@pytest.fixture(scope="session")
def parity_record():
    """Tests add one dict per config; written to gpurun_out/parity_records.json
    at the end of the session (pivot equality, ||dZ||/||Z||, relative errors,
    reference wall time)."""
    return _PARITY


def pytest_sessionfinish(session, exitstatus):
    if not _PARITY:
        return
    import json
    import platform
    out = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out, exist_ok=True)
    path = os.path.join(out, "parity_records.json")
    old = {}
    try:
        with open(path) as f:
            old = json.load(f)
    except (OSError, ValueError):
        pass
    old.update(_PARITY)
    old["_host"] = {"nproc": os.cpu_count(), "cpu": _cpu_model(), "machine": platform.machine()}
    with open(path, "w") as f:
        json.dump(old, f, indent=1, sort_keys=True)


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"

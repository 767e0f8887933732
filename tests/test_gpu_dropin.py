"""The drop-in seen from the reference's side.

* idk_matmul_ref reproduces the reference's matmul (matrix.cpp:28-48) bit for
  bit, so the shim's IdResult::approx satisfies test_id.cpp:57-68's exact
  equality with matmul(select_columns(a, cols), z).
* The host entries return cols / Z / approx equal to the device path.
* oracle/_ref/acceptance_b200 -- the reference's own acceptance suite
  (tests/acceptance.cpp), compiled unchanged with src/id.cpp + src/qr.cpp
  replaced by integration/idkit_b200_shim.cpp over libidkit_b200.so (built by
  `make -C oracle dropin` where the reference sources exist; the binary travels
  with the repo) -- passes the criteria the reference itself passes here.
"""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def idk():
    import paper_2105_07076_b200 as idk
    return idk


def dev(a):
    import torch
    return torch.from_numpy(np.asfortranarray(a, dtype=np.float64)).cuda()


@pytest.mark.parametrize("m,k,n", [(7, 5, 9), (784, 190, 1000), (33, 64, 1)])
def test_matmul_ref_is_bit_identical_to_reference(idk, ref, m, k, n):
    rng = np.random.default_rng(m + k + n)
    a = rng.standard_normal((m, k))
    b = rng.standard_normal((k, n))
    b[rng.random((k, n)) < 0.3] = 0.0           # the reference skips zero entries of b
    b[:, :min(k, n)][np.arange(min(k, n)), np.arange(min(k, n))] = 1.0
    c = idk.matmul_ref(dev(a), dev(b)).cpu().numpy()
    assert np.array_equal(c, ref.matmul(a, b))


@pytest.mark.parametrize("rid", [False, True])
def test_host_entries_return_reference_approx(idk, ref, rid):
    a = np.asfortranarray(ref.gaussian_matrix(60, 90, 3))
    m, n, k = 60, 90, 12
    ctx = idk.context(0)
    cols = np.empty(k, dtype=np.int64)
    z = np.empty((k, n), order="F")
    approx = np.empty((m, n), order="F")
    P = lambda x: x.ctypes.data_as(C.c_void_p)  # noqa: E731
    if rid:
        rc = ctx.lib.idk_optim_rid_host(ctx.h, P(a), m, n, k, 0.2, 77, P(cols), P(z), None, P(approx))
        rcols, rz, rapprox = ref.optim_rid(a, k, 0.2, 77)
    else:
        rc = ctx.lib.idk_optim_id_host(ctx.h, P(a), m, n, k, P(cols), P(z), None, P(approx))
        rcols, rz, rapprox = ref.optim_id(a, k)
    ctx.check(rc)
    assert np.array_equal(cols, rcols)
    assert np.linalg.norm(z - rz) <= 1e-10 * np.linalg.norm(rz)
    # approx is the reference's matmul of (A[:, cols], Z) bit for bit (test_id.cpp:57-68)
    assert np.array_equal(approx, ref.matmul(np.asfortranarray(a[:, cols]), z))


def test_reference_acceptance_suite_through_the_shim():
    exe = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/acceptance_b200 not built (needs the reference sources: make -C oracle dropin)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600, cwd=ROOT).stdout
    print(out)
    status = dict(re.findall(r"\[criterion (\d)\] (PASS|FAIL|SKIP)", out))
    # the criteria the reference passes in this environment (1 and 3 need absent datasets)
    for c in ("2", "4", "5", "6"):
        assert status.get(c) == "PASS", (c, out)
    assert status.get("1") == "SKIP" and status.get("3") == "SKIP"
    # criterion 7 (rand_id faster than det_id) is reported, not asserted: on the GPU both
    # are bound by the k dependent CPQR steps, see INTEGRATION.md
    assert "7" in status


def test_shim_dual_and_sketch_rid_from_the_reference_side():
    """integration/dropin_check.cpp: id_auto's dual without a host transpose and
    idkit::sketch_rid, checked with the reference's own Matrix helpers."""
    exe = os.path.join(ROOT, "oracle", "_ref", "dropin_check_b200")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/dropin_check_b200 not built (make -C oracle dropin)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300, cwd=ROOT)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count("PASS") == 6


@pytest.mark.parametrize("method", [0, 1])
@pytest.mark.parametrize("shape", [(90, 40), (40, 90)])
def test_id_auto_ref_host_matches_reference_id_auto(idk, ref, method, shape):
    """idk_id_auto_ref_host = idkit::id_auto (id.cpp:78-95) incl. approx, bit-identical
    approx given the same (C, Z) -- the tall case without a host transpose."""
    m, n = shape
    a = np.asfortranarray(ref.gaussian_matrix(m, n, 21))
    a[:, ::5] *= 3.0
    k = 8
    ctx = idk.context(0)
    zc = max(m, n)
    cols = np.empty(k, dtype=np.int64)
    z = np.empty((k, zc), order="F")
    approx = np.empty((m, n), order="F")
    tr = C.c_int(0)
    P = lambda x: x.ctypes.data_as(C.c_void_p)  # noqa: E731
    ctx.check(ctx.lib.idk_id_auto_ref_host(ctx.h, P(a), m, n, k, method, 31, 0.25, 0, P(cols), P(z), None,
                                           P(approx), C.byref(tr)))
    rcols, rz, rapprox, rtr = ref.id_auto(a, k, method == 1, seed=31, frac=0.25)
    assert bool(tr.value) == rtr == (m > n)
    assert np.array_equal(cols, rcols)
    assert np.linalg.norm(z - rz) <= 1e-10 * np.linalg.norm(rz)
    mat = np.asfortranarray(a.T) if rtr else a
    prod = ref.matmul(np.asfortranarray(mat[:, cols]), z)
    assert np.array_equal(approx, np.asfortranarray(prod.T) if rtr else prod)

"""Edge shapes and layouts through the C ABI, against the reference library
(oracle/_ref): single rows/columns, padded leading dimensions (strided views),
k at the limits of every kernel variant (k = min(m, n); k > 256 -> blocked
TRSM; k > 234 -> Bunch-Kaufman in L2), sketches taller than the matrix
(l = k + p > m) and the all-zero matrix (test_id.cpp:120-129's error class).
Tolerances as elsewhere: identical columns, ||dZ||_F/||Z||_F <= 1e-10.
"""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu
ZTOL = 1e-10


@pytest.fixture(scope="module")
def idk():
    import paper_2105_07076_b200 as idk
    return idk


def dev(a):
    import torch
    return torch.from_numpy(np.asfortranarray(a, dtype=np.float64)).cuda()


def host(t):
    return t.cpu().numpy()


def padded(a, extra=5):
    """a as a strided view of a larger column-major buffer (lda = m + extra)."""
    import torch
    m, n = a.shape
    big = torch.zeros((n, m + extra), dtype=torch.float64, device="cuda")
    big[:, :m] = torch.from_numpy(np.ascontiguousarray(a.T))
    v = big.t()[:m, :]
    assert v.stride() == (1, m + extra)
    return v


@pytest.mark.parametrize("m,n", [(1, 9), (9, 1), (1, 1)])
def test_single_row_or_column(idk, ref, m, n):
    a = ref.gaussian_matrix(m, n, 3)
    r = idk.id_auto(dev(a), 1, idk.DETERMINISTIC)
    rcols, rz, rapprox, rtr = ref.id_auto(a, 1, False)
    assert r.transposed == rtr
    assert np.array_equal(host(r.cols), rcols)
    assert rel(host(r.z), rz) <= ZTOL


@pytest.mark.parametrize("shape,k", [((40, 70), 9), ((70, 40), 9)])
def test_padded_leading_dimension(idk, ref, shape, k):
    a = ref.gaussian_matrix(shape[0], shape[1], 11)
    rcols, rz, _, rtr = ref.id_auto(a, k, False)
    r = idk.id_auto(padded(a), k, idk.DETERMINISTIC)
    assert np.array_equal(host(r.cols), rcols) and rel(host(r.z), rz) <= ZTOL
    # optim_rid and the sketch on the same strided view equal the packed input
    if shape[0] <= shape[1]:
        p1 = idk.optim_rid(padded(a), k, 0.5, 4)
        p2 = idk.optim_rid(dev(a), k, 0.5, 4)
        assert np.array_equal(host(p1.cols), host(p2.cols)) and np.array_equal(host(p1.z), host(p2.z))
        s1 = idk.sketch_rid(padded(a), k, 4, seed=6)
        s2 = idk.sketch_rid(dev(a), k, 4, seed=6)
        assert np.array_equal(host(s1.cols), host(s2.cols)) and np.array_equal(host(s1.z), host(s2.z))


def test_k_equals_min_dimension(idk, ref):
    a = ref.gaussian_matrix(30, 45, 12)
    r = idk.optim_id(dev(a), 30)
    rcols, rz, _ = ref.optim_id(a, 30)
    assert np.array_equal(host(r.cols), rcols) and rel(host(r.z), rz) <= 1e-9
    err = np.linalg.norm(a - host(r.c) @ host(r.z)) / np.linalg.norm(a)
    assert err <= 1e-12


def test_large_k_blocked_trsm(idk, ref):
    """k = 280 > 256: the blocked (non-register) TRSM path."""
    a = ref.gaussian_matrix(300, 420, 13)
    r = idk.optim_id(dev(a), 280)
    rcols, rz, _ = ref.optim_id(a, 280)
    assert np.array_equal(host(r.cols), rcols)
    assert rel(host(r.z), rz) <= 1e-9


def test_large_k_ldlt_in_l2(idk, ref):
    """k = 250: the Bunch-Kaufman factor no longer fits packed in shared memory."""
    a = ref.gaussian_matrix(260, 600, 14)
    r = idk.optim_rid(dev(a), 250, 0.1, 21)
    rcols, rz, _ = ref.optim_rid(a, 250, 0.1, 21)
    assert np.array_equal(host(r.cols), rcols)
    assert rel(host(r.z), rz) <= 1e-9


def test_sketch_taller_than_matrix(idk, oracle):
    """l = k + p > m: Omega has more rows than A."""
    a = oracle.gaussian_matrix(20, 50, 15)
    k, p = 18, 10
    omega = oracle.omega_philox(k + p, 20, 16)
    r = idk.sketch_rid(dev(a), k, p, omega_mode=idk.OMEGA_VERBATIM, omega=dev(omega))
    ocols, oz, oc, _ = oracle.interp_decomp(a, k, omega)
    assert np.array_equal(host(r.cols), ocols)
    assert rel(host(r.z), oz) <= ZTOL


def test_zero_matrix_det_raises_not_posdef(idk, ref):
    a = np.zeros((8, 12))
    with pytest.raises(idk.NotPositiveDefiniteError):
        idk.optim_id(dev(a), 3)
    from oracle import NotPositiveDefiniteError as RefNPD
    with pytest.raises(RefNPD):
        ref.optim_id(a, 3)


def test_zero_matrix_qr_pivots_in_order(idk, ref):
    """All norms zero: every step pivots on the current position (qr.cpp:66-78)."""
    a = np.zeros((6, 10))
    f = idk.qr_column_pivoted(dev(a), 6)
    _, _, rperm = ref.qr_column_pivoted(a, 6)
    assert np.array_equal(host(f.perm), rperm)


@pytest.mark.parametrize("k", [1, 2, 31, 32, 33, 63, 64, 65, 96, 100, 127, 128, 129, 160, 224, 256, 257])
def test_z_solve_block_boundaries(idk, ref, monkeypatch, k):
    """The DMMA blocked Z solve (k <= 128: identity-padded 32-row blocks, 64
    right-hand sides per CTA) at every block and CTA boundary, against the
    reference and against the warp kernel it replaces (IDK_TRSM_DMMA=0)."""
    m, n = k + 7, 2 * k + 71  # n - k right-hand sides: not a multiple of 64
    a = ref.gaussian_matrix(m, n, 40 + k)
    a[:, ::5] *= 3.0
    rcols, rz, _, _ = ref.id_auto(a, k, False)
    r = idk.id_auto(dev(a), k, idk.DETERMINISTIC)
    assert np.array_equal(host(r.cols), rcols)
    assert rel(host(r.z), rz) <= ZTOL
    monkeypatch.setenv("IDK_TRSM_DMMA", "0")
    w = idk.id_auto(dev(a), k, idk.DETERMINISTIC)
    assert np.array_equal(host(w.cols), host(r.cols))
    assert rel(host(w.z), host(r.z)) <= 1e-12


@pytest.mark.parametrize("m,n,k,padded_ld", [(37, 50, 5, False), (64, 300, 17, True), (2000, 300, 120, False),
                                            (301, 77, 9, True), (2000, 40, 800, False)])
def test_select_columns_all_paths(idk, ref, m, n, k, padded_ld):
    """select_columns (matrix.cpp:121-130) through the vectorised column copy
    (even rows, 16-byte aligned), its scalar fallback (odd rows / padded ld) and
    the staged row gather of the dual: bit-exact."""
    import torch
    a = ref.gaussian_matrix(m, n, 5 + m)
    da = padded(a, extra=3) if padded_ld else dev(a)
    cols = np.random.default_rng(m + n).choice(n, size=min(k, n), replace=False)
    c = host(idk.select_columns(da, torch.from_numpy(cols).cuda()))
    assert np.array_equal(c, a[:, cols])
    rows = np.random.default_rng(m).choice(m, size=min(k, m), replace=False)
    cr = host(idk.select_columns(da, torch.from_numpy(rows).cuda(), rows_of_a=True))
    assert np.array_equal(cr, a[rows, :].T)

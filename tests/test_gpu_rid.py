"""GPU parity of the reference's own randomized ID, optim_rid (id.cpp:47-76),
through the C ABI (idk_optim_rid / idk_id_auto method 2) against the reference
library itself (oracle/_ref).  Mirrors test_id.cpp:49-118.

Tolerances: identical columns (the mt19937_64 sample and the CPQR pivots are
reproduced exactly); ||dZ||_F/||Z||_F <= 1e-10 on well-conditioned inputs.
Z solves the normal equations (R_k^T R_k) Z = C^T A, whose rounding error grows
with cond(R_k)^2 in both implementations, so the spectrum-decay case states its
bound as 1e-10 relative on the reconstruction error plus
||dZ||/||Z|| <= 64 eps cond(R_k)^2.
"""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu
ZTOL = 1e-10
EPS = np.finfo(np.float64).eps


@pytest.fixture(scope="module")
def idk():
    import paper_2105_07076_b200 as idk
    return idk


def dev(a):
    import torch
    return torch.from_numpy(np.asfortranarray(a, dtype=np.float64)).cuda()


def host(t):
    return t.cpu().numpy()


@pytest.mark.parametrize("m,n,k,frac,seed", [
    (14, 20, 6, 0.2, 3),      # test_id.cpp:57-68
    (18, 26, 8, 0.2, 1234),   # test_id.cpp:93-107
    (16, 16, 6, 0.2, 77),     # test_id.cpp:155-163
    (60, 200, 20, 0.5, 9),
    (120, 700, 40, 1.0, 21),
    (300, 1000, 200, 0.1, 5),  # k > 160: the LDL^T factor runs out of global memory
])
def test_optim_rid_vs_reference(idk, ref, m, n, k, frac, seed):
    a = ref.gaussian_matrix(m, n, seed + 100)
    r = idk.optim_rid(dev(a), k, frac, seed)
    rcols, rz, rapprox = ref.optim_rid(a, k, frac, seed)
    assert np.array_equal(host(r.cols), rcols)
    assert rel(host(r.z), rz) <= ZTOL
    assert np.array_equal(host(r.c), a[:, rcols])
    approx = host(r.c) @ host(r.z)
    assert rel(approx, rapprox) <= ZTOL


def test_optim_rid_spectrum_decay_vs_reference(idk, ref):
    """cfg2's matrix family (2000 x 2000, sigma_j = j^-2) at k = 100, frac 0.1."""
    from paper_2105_07076_b200.configs import make_np
    a = make_np("cfg2", seed=31)
    k, frac, seed = 100, 0.1, 31
    r = idk.optim_rid(dev(a), k, frac, seed)
    rcols, rz, rapprox = ref.optim_rid(a, k, frac, seed)
    assert np.array_equal(host(r.cols), rcols)
    c = a[:, rcols]
    s = np.linalg.svd(np.linalg.qr(c, mode="r"), compute_uv=False)
    kappa2 = (s[0] / s[-1]) ** 2
    dz = rel(host(r.z), rz)
    print(f"cfg2 optim_rid: ||dZ||/||Z|| = {dz:.3e}, cond(R_k)^2 = {kappa2:.3e}")
    assert dz <= max(ZTOL, 64 * EPS * kappa2)
    e = np.linalg.norm(a - c @ host(r.z)) / np.linalg.norm(a)
    re_ = np.linalg.norm(a - rapprox) / np.linalg.norm(a)
    assert abs(e - re_) <= ZTOL * re_


def test_full_sample_when_p_clamps_to_n(idk):
    """test_id.cpp:84-91: identity(10), k = 10 -> every column, exact."""
    a = np.eye(10)
    r = idk.optim_rid(dev(a), 10, 0.2, 17)
    assert sorted(host(r.cols).tolist()) == list(range(10))
    err = np.linalg.norm(a - host(r.c) @ host(r.z)) / np.linalg.norm(a)
    assert err <= 1e-10


def test_seed_reproducible(idk, ref):
    """test_id.cpp:93-107: same seed -> bit-identical, next seed -> new sample."""
    a = ref.gaussian_matrix(18, 26, 6)
    s1 = idk.optim_rid(dev(a), 8, 0.2, 1234)
    s2 = idk.optim_rid(dev(a), 8, 0.2, 1234)
    assert np.array_equal(host(s1.cols), host(s2.cols))
    assert np.array_equal(host(s1.z), host(s2.z))
    s3 = idk.optim_rid(dev(a), 8, 0.2, 1235)
    assert not np.array_equal(host(s1.cols), host(s3.cols))
    assert np.array_equal(host(s3.cols), ref.optim_rid(a, 8, 0.2, 1235)[0])


def test_rank_deficient_sample_is_singular(idk, ref):
    """test_id.cpp:109-118: two nonzero columns, any 3-column sample is singular."""
    a = np.zeros((4, 6))
    g = ref.gaussian_matrix(4, 2, 7)
    a[:, 0], a[:, 1] = g[:, 0], g[:, 1]
    with pytest.raises(idk.SingularMatrixError):
        idk.optim_rid(dev(a), 3, 0.0, 5)
    from oracle import SingularMatrixError as RefSingular
    with pytest.raises(RefSingular):
        ref.optim_rid(a, 3, 0.0, 5)


def test_invalid_arguments(idk, ref):
    """test_id.cpp:48-55."""
    a = dev(ref.gaussian_matrix(6, 9, 1))
    for k in (0, 7):
        with pytest.raises(idk.InvalidArgument):
            idk.optim_rid(a, k, 0.2, 1)
    with pytest.raises(idk.InvalidArgument):
        idk.optim_rid(a, 3, -0.5, 1)


@pytest.mark.parametrize("m,n", [(16, 16), (40, 12), (300, 90), (3000, 400)])
def test_id_auto_sampled_vs_reference(idk, ref, m, n):
    """id_auto(randomized) of the reference routes through optim_rid, tall inputs
    through A^T (id.cpp:78-95); method SAMPLED reproduces it, dual included."""
    a = ref.gaussian_matrix(m, n, m + n)
    k = 5
    r = idk.id_auto(dev(a), k, idk.SAMPLED, seed=77)
    rcols, rz, rapprox, rtr = ref.id_auto(a, k, True, seed=77, frac=0.2)
    assert r.transposed == rtr == (m > n)
    assert np.array_equal(host(r.cols), rcols)
    assert rel(host(r.z), rz) <= ZTOL
    if rtr:
        assert np.array_equal(host(r.c), a[rcols, :].T)
        approx = host(r.z).T @ a[rcols, :]
    else:
        approx = host(r.c) @ host(r.z)
    assert rel(approx, rapprox) <= ZTOL
    # the host-buffer entry gives the same result
    h = idk.id_auto(a, k, idk.SAMPLED, seed=77)
    assert np.array_equal(h.cols, rcols) and rel(h.z, rz) <= ZTOL


@pytest.mark.parametrize("m,n,k,frac,decay,seed", [
    (3000, 400, 30, 0.5, 6.0, 41),    # tall sample: p = 45, pivoted QR on the CholeskyQR3 factor
    (2500, 120, 40, 1.0, 9.0, 42),    # column norms down to 1e-9: the shifted first step matters
])
def test_optim_rid_tall_sample_vs_reference(idk, ref, m, n, k, frac, decay, seed):
    a = ref.gaussian_matrix(m, n, seed) * np.logspace(0, -decay, n)[None, :]
    a = np.asfortranarray(a)
    r = idk.optim_rid(dev(a), k, frac, seed)
    rcols, rz, rapprox = ref.optim_rid(a, k, frac, seed)
    assert np.array_equal(host(r.cols), rcols)
    c = a[:, rcols]
    s = np.linalg.svd(np.linalg.qr(c, mode="r"), compute_uv=False)
    kappa2 = (s[0] / s[-1]) ** 2
    assert rel(host(r.z), rz) <= max(ZTOL, 64 * EPS * kappa2)


def test_optim_rid_tall_sample_with_zero_columns(idk, ref):
    """An exactly zero sampled column keeps the reference's route (pivoted QR of A_S)."""
    a = np.asfortranarray(ref.gaussian_matrix(2000, 60, 43))
    a[:, ::3] = 0.0
    r = idk.optim_rid(dev(a), 8, 1.0, 44)
    rcols, rz, _ = ref.optim_rid(a, 8, 1.0, 44)
    assert np.array_equal(host(r.cols), rcols)
    assert rel(host(r.z), rz) <= ZTOL

"""Shapes that do not fit on chip (the reference factors any
shape; qr.cpp:42-46 validates only max_steps).  The resident CPQR cannot hold
these, so the streaming kernel runs with the matrix in HBM and -- when m
doubles no longer fit in shared memory (m > ~24k rows) -- its reflector in an
L2-resident buffer shared by all CTAs.  Compared with the reference library itself."""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def idk():
    import paper_2105_07076_b200 as idk
    return idk


def _dev(a):
    import torch
    return torch.from_numpy(np.asfortranarray(a)).cuda()


def _low_rank_tall(m, n, r, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, r)) @ (rng.standard_normal((r, n)) * np.exp(-np.arange(n) / 12.0))
    return np.asfortranarray(a + 1e-3 * rng.standard_normal((m, n)))


def test_qr_column_pivoted_100000_x_50(idk, ref):
    a = _low_rank_tall(100000, 50, 50, 1)
    ctx = idk.context(0)
    assert ctx.cpqr_plan(100000, 50, 50)["kind"] == "streaming"
    f = idk.qr_column_pivoted(_dev(a), 50)
    rq, rr, rperm = ref.qr_column_pivoted(a, 50)
    assert np.array_equal(f.perm.cpu().numpy(), rperm)
    assert rel(f.r.cpu().numpy(), rr) <= 1e-10
    assert rel(f.q.cpu().numpy(), rq) <= 1e-10


def test_optim_id_100000_x_50(idk, ref):
    a = _low_rank_tall(100000, 50, 30, 2)
    r = idk.optim_id(_dev(a), 20)
    rcols, rz, _ = ref.optim_id(a, 20)
    assert np.array_equal(r.cols.cpu().numpy(), rcols)
    assert rel(r.z.cpu().numpy(), rz) <= 1e-10
    assert np.array_equal(r.c.cpu().numpy(), a[:, rcols])


def test_qr_column_pivoted_30000_x_30000(idk, ref):
    """7.2 GB in HBM: 16 pivot steps of the streaming kernel against the reference."""
    import torch
    n = 30000
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    a = torch.randn((n, n), generator=g, device="cuda", dtype=torch.float64).t()  # column-major view
    a[:, ::7] *= 2.5
    f = idk.qr_column_pivoted(a, 16)
    ah = np.asfortranarray(a.cpu().numpy())
    del a
    torch.cuda.empty_cache()
    rq, rr, rperm = ref.qr_column_pivoted(ah, 16)
    assert np.array_equal(f.perm.cpu().numpy()[:16], rperm[:16])
    assert np.array_equal(f.perm.cpu().numpy(), rperm)
    assert rel(f.r.cpu().numpy(), rr) <= 1e-10
    assert rel(f.q.cpu().numpy(), rq) <= 1e-10


def test_optim_id_5000_x_3000_half_block_streaming(idk, ref):
    """120 MB: too large for the on-chip CPQR, columns long enough (>= 2048 rows) for the
    streaming kernel's half-block-per-column path with the reflector in shared memory."""
    rng = np.random.default_rng(7)
    m, n, k = 5000, 3000, 24
    a = rng.standard_normal((m, 40)) @ (rng.standard_normal((40, n)) * np.exp(-np.arange(n) / 300.0))
    a = np.asfortranarray(a + 1e-4 * rng.standard_normal((m, n)))
    ctx = idk.context(0)
    assert ctx.cpqr_plan(m, n, k)["kind"] == "streaming"
    r = idk.optim_id(_dev(a), k)
    rcols, rz, _ = ref.optim_id(a, k)
    assert np.array_equal(r.cols.cpu().numpy(), rcols)
    assert rel(r.z.cpu().numpy(), rz) <= 1e-10
    assert np.array_equal(r.c.cpu().numpy(), a[:, rcols])
    f = idk.qr_column_pivoted(_dev(a), k)
    rq, rr, rperm = ref.qr_column_pivoted(a, k)
    assert np.array_equal(f.perm.cpu().numpy(), rperm)
    assert rel(f.r.cpu().numpy(), rr) <= 1e-10
    assert rel(f.q.cpu().numpy(), rq) <= 1e-10

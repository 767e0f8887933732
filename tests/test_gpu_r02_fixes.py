"""Regression tests for the round-1 advisor findings.

* idk_id_from_sketch with a padded sketch (ldy > l) factors the right elements.
* idk_diagnostics rejects a column index outside Z like id.cpp:108-111.
* optim_rid on a tall sample taller than the on-chip CPQR budget (m > 25.6k
  rows) runs through the R0 route instead of failing the m x p fit check.
"""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def idk():
    import paper_2105_07076_b200 as idk
    return idk


def test_id_from_sketch_padded_ldy(idk, oracle):
    import torch
    rng = np.random.default_rng(3)
    l, n, k = 40, 700, 30
    y = rng.standard_normal((l, n)) * np.exp(-np.arange(n) / 90.0)
    store = torch.full((n, l + 24), float("nan"), dtype=torch.float64, device="cuda")
    store[:, :l] = torch.from_numpy(y.T).cuda()
    padded = store.t()[:l]  # l x n view, ld = l + 24
    assert padded.stride() == (1, l + 24)
    cols_p, z_p = idk.id_from_sketch(padded, k)
    cols_c, z_c = idk.id_from_sketch(torch.from_numpy(np.asfortranarray(y)).cuda(), k)
    assert torch.equal(cols_p, cols_c)
    assert torch.equal(z_p, z_c)
    ocols, oz, _, _ = oracle.interp_decomp(y, k, None, want_c=False)
    assert np.array_equal(cols_c.cpu().numpy(), ocols)
    assert rel(z_c.cpu().numpy(), oz) <= 1e-10


def test_diagnostics_rejects_bad_column(idk):
    import torch
    rng = np.random.default_rng(4)
    a = torch.from_numpy(np.asfortranarray(rng.standard_normal((50, 80)))).cuda()
    r = idk.optim_id(a, 10)
    r.cols[3] = 80  # outside Z's 80 columns
    with pytest.raises(idk.InvalidArgument):
        idk.diagnostics(a, r)


def test_optim_rid_very_tall_sample(idk, ref):
    rng = np.random.default_rng(5)
    m, n, k = 30000, 300, 12
    a = np.asfortranarray(rng.standard_normal((m, 40)) @ rng.standard_normal((40, n)))
    r = idk.optim_rid(a, k, 0.25, 77)
    rcols, rz, _ = ref.optim_rid(a, k, 0.25, 77)
    assert np.array_equal(r.cols, rcols)
    assert rel(r.z, rz) <= 1e-10

"""GPU parity at the BASELINE.json configurations.

cfg1/cfg2 run at full size against the reference library itself
(oracle/_ref); cfg3 on a sample of its 4096 matrices; cfg4/cfg5 at reduced
size (the CPU oracle would take minutes at 16384^2) with their spectra, plus
full-size property checks (identity block, literal columns, Eckart-Young floor,
run-to-run bit determinism, sketch vs an independent cuBLAS DGEMM).
Tolerances: identical columns; ||dZ||_F/||Z||_F <= 1e-10; relative error
within 1e-10 relative (BASELINE.json north_star).
"""
import numpy as np
import pytest

from conftest import rel
from paper_2105_07076_b200.configs import CONFIGS, make_np, make_torch, spectrum

pytestmark = pytest.mark.gpu
ZTOL = 1e-10


def dev(a):
    import torch
    return torch.from_numpy(np.asfortranarray(a, dtype=np.float64)).cuda()


def host(t):
    return t.cpu().numpy()


@pytest.fixture(scope="module")
def idk():
    import paper_2105_07076_b200 as idk
    return idk


def rel_err(a, c, z):
    return np.linalg.norm(a - c @ z) / np.linalg.norm(a)


def test_cfg1_full_size_vs_reference_optim_id(idk, ref):
    a = make_np("cfg1", seed=11)
    r = idk.optim_id(dev(a), 50)
    cols, z, c = host(r.cols), host(r.z), host(r.c)
    rcols, rz, rapprox = ref.optim_id(a, 50)
    assert np.array_equal(cols, rcols)
    assert rel(z, rz) <= ZTOL
    e, re_ = rel_err(a, c, z), np.linalg.norm(a - rapprox) / np.linalg.norm(a)
    assert abs(e - re_) <= ZTOL * re_


def test_cfg2_full_size_vs_reference_composition(idk, ref, oracle):
    a = make_np("cfg2", seed=12)
    k, p = 100, 10
    omega = ref.generate(1, k + p, 2000, 12)  # the reference's own generate(gaussian, l, m, seed)
    r = idk.sketch_rid(dev(a), k, p, omega_mode=idk.OMEGA_VERBATIM, omega=dev(omega))
    rcols, rz, rc = ref.sketch_id(a, k, omega)
    assert np.array_equal(host(r.cols), rcols)
    assert rel(host(r.z), rz) <= ZTOL
    assert np.array_equal(host(r.c), rc)
    # device Philox Omega against the oracle's Philox
    r2 = idk.sketch_rid(dev(a), k, p, seed=12)
    ocols, oz, oc, _ = oracle.interp_decomp(a, k, oracle.omega_philox(k + p, 2000, 12))
    assert np.array_equal(host(r2.cols), ocols)
    assert rel(host(r2.z), oz) <= ZTOL


@pytest.mark.parametrize("exact", [False, True])
def test_cfg3_sample_vs_reference(idk, ref, exact):
    import torch
    a = make_np("cfg3", seed=13, scale=96 / 4096)  # 96 of the 4096 matrices
    ctx = idk.context(0)
    ctx.set_batched_exact(exact)
    try:
        cols, z, c = idk.optim_id_batched(torch.from_numpy(a).cuda(), 16)
    finally:
        ctx.set_batched_exact(False)
    cols, z, c = host(cols), host(z), host(c)
    for b in range(a.shape[0]):
        ab = np.asfortranarray(a[b].T)
        rcols, rz, rc = ref.sketch_id(ab, 16, None)
        assert np.array_equal(cols[b], rcols)
        if exact:
            assert np.array_equal(z[b].T, rz)
        else:
            assert rel(z[b].T, rz) <= ZTOL
        assert np.array_equal(c[b].T, rc)
        if b < 8:  # the reference's optim_id (normal equations) agrees too
            ocols, oz, _ = ref.optim_id(ab, 16)
            assert np.array_equal(cols[b], ocols) and rel(z[b].T, oz) <= ZTOL


def test_cfg4_spectrum_scaled_vs_oracle(idk, oracle):
    """cfg4's spectrum at n = 2048 (the tightest Z margin)."""
    from paper_2105_07076_b200.configs import svd_matrix_np
    a = svd_matrix_np("cfg4", 2048, 2048, 14)
    k, p = 256, 16
    omega = oracle.omega_philox(k + p, 2048, 14)
    r = idk.sketch_rid(dev(a), k, p, omega_mode=idk.OMEGA_VERBATIM, omega=dev(omega))
    ocols, oz, oc, _ = oracle.interp_decomp(a, k, omega)
    assert np.array_equal(host(r.cols), ocols)
    dz = rel(host(r.z), oz)
    print(f"cfg4-spectrum n=2048: ||dZ||/||Z|| = {dz:.3e}")
    assert dz <= ZTOL
    assert np.array_equal(host(r.c), oc)
    e, oe = rel_err(a, host(r.c), host(r.z)), rel_err(a, oc, oz)
    assert abs(e - oe) <= ZTOL * oe


def test_cfg5_recipe_scaled_vs_oracle(idk, oracle):
    """cfg5's W H + noise recipe at 8192 x 512: the dual (m > n) runs on A^T."""
    from paper_2105_07076_b200.configs import nonneg_low_rank_np
    a = nonneg_low_rank_np(8192, 512, 64, 1e-6, 15)
    k, p = 64, 8
    r = idk.id_auto(dev(a), k, idk.RANDOMIZED, seed=15, p=p)
    assert r.transposed
    at = np.asfortranarray(a.T)
    ocols, oz, oc, _ = oracle.interp_decomp(at, k, oracle.omega_philox(k + p, 512, 15))
    assert np.array_equal(host(r.cols), ocols)
    assert rel(host(r.z), oz) <= ZTOL
    assert np.array_equal(host(r.c), oc)


@pytest.mark.parametrize("name", ["cfg4", "cfg5"])
def test_full_size_properties(idk, name):
    """Full BASELINE size: literal columns, exact identity block, error at the
    Eckart-Young floor, bit determinism, sketch vs cuBLAS DGEMM."""
    import torch
    cfg = CONFIGS[name]
    a = make_torch(name, seed=16)
    r1 = idk.id_auto(a, cfg.k, idk.RANDOMIZED, seed=16, p=cfg.p)
    r2 = idk.id_auto(a, cfg.k, idk.RANDOMIZED, seed=16, p=cfg.p)
    assert torch.equal(r1.cols, r2.cols) and torch.equal(r1.z, r2.z) and torch.equal(r1.c, r2.c)
    cols = r1.cols
    assert len(set(cols.tolist())) == cfg.k
    if r1.transposed:  # A ~= Z^T A[cols, :]
        assert torch.equal(r1.c, a[cols, :].t())
        approx = r1.z.t() @ a[cols, :]
    else:
        assert torch.equal(r1.c, a[:, cols])
        approx = r1.c @ r1.z
    zi = r1.z[:, cols]
    assert torch.equal(zi, torch.eye(cfg.k, dtype=zi.dtype, device=zi.device))
    err = float(torch.linalg.norm(a - approx) / torch.linalg.norm(a))
    del approx
    if name == "cfg4":
        s = spectrum("cfg4", cfg.m)
        floor = float(np.sqrt((s[cfg.k:] ** 2).sum() / (s ** 2).sum()))
        assert floor <= err <= 10 * floor, (err, floor)
    else:
        assert err <= 1e-5, err  # rank-64 W H + U[0, 1e-6] noise
    # the sketch against cuBLAS (test-only checker)
    om = idk.sketch_omega(cfg.l, cfg.n if r1.transposed else cfg.m, 16)
    y = idk.sketch(om, a, transposed=r1.transposed)
    y_ref = om @ (a.t() if r1.transposed else a)
    assert float(torch.linalg.norm(y - y_ref) / torch.linalg.norm(y_ref)) <= 1e-13

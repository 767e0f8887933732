"""GPU parity of the ID entry points against the reference (oracle/_ref) and the
C restatement (oracle/liboracle.so).

Mirrors /root/reference/proj/tests/test_id.cpp (cited per test), then checks
the north-star path: Gaussian sketch -> CPQR -> Z = [I | R11^-1 R12] P^T -> C.
Tolerances follow BASELINE.json north_star: identical column indices; Z and
the relative error within 1e-10 relative (fp64), Z measured normwise
(||dZ||_F / ||Z||_F).
"""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu

ZTOL = 1e-10


def dev(a):
    import torch
    return torch.from_numpy(np.asfortranarray(a, dtype=np.float64)).cuda()


def host(t):
    return None if t is None else t.cpu().numpy()


@pytest.fixture(scope="module")
def idk():
    import paper_2105_07076_b200 as idk
    return idk


@pytest.fixture(autouse=True, params=[0, 1, 2, 3],
                ids=["cpqr-auto", "cpqr-resident-grid", "cpqr-streaming", "cpqr-cluster-pull"])
def cpqr_mode(request, idk):
    """Every case runs on each CPQR kernel: cluster/resident (auto), resident grid, streaming."""
    ctx = idk.context(0)
    ctx.set_cpqr_mode(request.param)
    yield request.param
    ctx.set_cpqr_mode(0)


def rel_error(a, c, z):
    return np.linalg.norm(a - c @ z) / np.linalg.norm(a)


def run_det(idk, a, k):
    r = idk.optim_id(dev(a), k)
    return host(r.cols), host(r.z), host(r.c)


# ---- test_id.cpp mirrors ----------------------------------------------------------

def test_identity_full_rank(idk):  # test_id.cpp:13-28
    cols, z, c = run_det(idk, np.eye(5), 5)
    assert rel_error(np.eye(5), c, z) <= 1e-14
    assert np.all(np.minimum(np.abs(z), np.abs(z - 1)) <= 1e-12)
    np.testing.assert_allclose(z.sum(axis=1), 1.0)


def test_norm2_column_first(idk):  # test_id.cpp:30-46
    a = np.zeros((6, 3))
    a[0, 0] = 1.0
    a[0, 1] = 2.0
    a[1, 2] = 1.0
    cols, z, c = run_det(idk, a, 2)
    assert list(cols) == [1, 2]
    assert rel_error(a, c, z) <= 1e-12


def test_k_bounds(idk, oracle):  # test_id.cpp:48-55
    a = dev(oracle.gaussian_matrix(6, 9, 1))
    for k in (0, 7):
        with pytest.raises(idk.InvalidArgument):
            idk.optim_id(a, k)
        with pytest.raises(idk.InvalidArgument):
            idk.sketch_rid(a, k, 2, seed=1)
    with pytest.raises(idk.InvalidArgument):
        idk.id_auto(a, 0, idk.DETERMINISTIC)


def test_literal_columns(idk, oracle):  # test_id.cpp:57-68
    a = oracle.gaussian_matrix(14, 20, 2)
    for r in (idk.optim_id(dev(a), 6), idk.sketch_rid(dev(a), 6, 2, seed=3)):
        cols = host(r.cols)
        assert np.array_equal(host(r.c), a[:, cols])
        assert len(set(cols.tolist())) == 6 and cols.max() < 20


def test_det_z_solves_normal_equations(idk, oracle):  # test_id.cpp:70-76
    a = oracle.gaussian_matrix(15, 22, 4)
    cols, z, c = run_det(idk, a, 7)
    res = c.T @ (a - c @ z)
    assert np.linalg.norm(res) <= 1e-9 * np.linalg.norm(c) * np.linalg.norm(a)


def test_identity_block_deviation(idk, oracle):  # test_id.cpp:78-82
    a = oracle.gaussian_matrix(30, 24, 5)
    cols, z, c = run_det(idk, a, 10)
    assert np.max(np.abs(z[:, cols] - np.eye(10))) <= 1e-8


def test_bit_reproducible(idk, oracle):  # test_id.cpp:93-107
    a = dev(oracle.gaussian_matrix(18, 26, 6))
    r1, r2 = idk.optim_id(a, 8), idk.optim_id(a, 8)
    assert np.array_equal(host(r1.cols), host(r2.cols)) and np.array_equal(host(r1.z), host(r2.z))
    s1, s2 = idk.sketch_rid(a, 8, 3, seed=1234), idk.sketch_rid(a, 8, 3, seed=1234)
    assert np.array_equal(host(s1.cols), host(s2.cols)) and np.array_equal(host(s1.z), host(s2.z))


def test_rank_deficient_det_raises_not_posdef(idk, oracle):  # test_id.cpp:120-129
    g = oracle.gaussian_matrix(10, 2, 8)
    a = np.zeros((10, 12))
    a[:, 3] = g[:, 0]
    a[:, 9] = g[:, 1]
    with pytest.raises(idk.NotPositiveDefiniteError):
        idk.optim_id(dev(a), 3)


def test_rank_deficient_sketch_raises_singular(idk, oracle):  # test_id.cpp:109-118 (sketch analogue)
    g = oracle.gaussian_matrix(4, 2, 7)
    a = np.zeros((4, 6))
    a[:, 0] = g[:, 0]
    a[:, 1] = g[:, 1]
    with pytest.raises(idk.SingularMatrixError):
        idk.sketch_rid(dev(a), 3, 1, seed=5)


def test_id_auto_transposes_tall(idk, oracle):  # test_id.cpp:131-147
    a = oracle.gaussian_matrix(40, 12, 10)
    r = idk.id_auto(dev(a), 5, idk.DETERMINISTIC)
    assert r.transposed
    cols, z = host(r.cols), host(r.z)
    assert z.shape == (5, 40) and np.all(cols < 40)
    rows = a[cols, :]
    assert np.array_equal(host(r.c), rows.T)


def test_id_auto_shape_contract(idk, oracle):  # test_id.cpp:149-158
    a = oracle.gaussian_matrix(1000, 784, 16)
    r = idk.id_auto(dev(a), 50, idk.DETERMINISTIC)
    assert r.transposed and host(r.z).shape == (50, 1000)


def test_tall_low_rank_reconstructs_through_dual(idk, oracle):  # test_id.cpp:169-182
    base = oracle.gaussian_matrix(3, 8, 12)
    picks = np.random.default_rng(13).integers(0, 3, size=50)
    a = np.asfortranarray(base[picks, :])  # 50 x 8, rank 3: replicated rows
    r = idk.id_auto(dev(a), 3, idk.DETERMINISTIC)
    assert r.transposed
    cols, z = host(r.cols), host(r.z)
    approx = z.T @ a[cols, :]
    assert np.linalg.norm(a - approx) / np.linalg.norm(a) <= 1e-10


def test_full_rank_square_exact(idk, oracle):  # test_id.cpp:184-187
    a = oracle.gaussian_matrix(12, 12, 20)
    cols, z, c = run_det(idk, a, 12)
    assert rel_error(a, c, z) <= 1e-10


def test_errors_dominate_svd_and_shrink_with_k(idk, oracle, ref):  # test_id.cpp:189-201
    a = oracle.gaussian_matrix(35, 50, 14)
    prev = 2.0
    for k in (3, 6, 12, 20):
        floor = ref.truncated_svd_error(a, k)
        cols, z, c = run_det(idk, a, k)
        det = rel_error(a, c, z)
        r = idk.sketch_rid(dev(a), k, 4, seed=21)
        rnd = rel_error(a, host(r.c), host(r.z))
        assert det >= floor - 1e-10 and rnd >= floor - 1e-10
        assert det <= prev + 1e-12
        prev = det


# ---- parity against the reference on the same inputs ------------------------------

@pytest.mark.parametrize("m,n,k,seed", [(14, 20, 6, 2), (30, 24, 10, 5), (64, 256, 16, 9), (200, 300, 40, 3),
                                        (784, 1000, 190, 7)])
def test_det_matches_reference_optim_id(idk, ref, m, n, k, seed):
    a = ref.gaussian_matrix(m, n, seed)
    cols, z, c = run_det(idk, a, k)
    rcols, rz, rapprox = ref.optim_id(a, k)
    assert np.array_equal(cols, rcols)
    assert rel(z, rz) <= ZTOL
    err = rel_error(a, c, z)
    rerr = np.linalg.norm(a - rapprox) / np.linalg.norm(a)
    assert abs(err - rerr) <= ZTOL * rerr


@pytest.mark.parametrize("m,n,k,p,seed", [(20, 30, 5, 3, 1), (60, 90, 12, 4, 2), (300, 700, 40, 10, 3),
                                          (2000, 1500, 64, 8, 4), (128, 5000, 30, 6, 5)])
def test_sketch_matches_reference_composition(idk, ref, oracle, m, n, k, p, seed):
    """Verbatim Omega (the reference's own generate(gaussian)) -> identical cols, Z within 1e-10, C exact."""
    a = ref.gaussian_matrix(m, n, seed)
    a[:, ::5] *= 2.0
    omega = ref.generate(1, k + p, m, seed + 100)
    r = idk.sketch_rid(dev(a), k, p, omega_mode=idk.OMEGA_VERBATIM, omega=dev(omega))
    rcols, rz, rc = ref.sketch_id(a, k, omega)
    assert np.array_equal(host(r.cols), rcols)
    assert rel(host(r.z), rz) <= ZTOL
    assert np.array_equal(host(r.c), rc)


def test_sketch_mt19937_mode_equals_reference_generate(idk, ref):
    a = ref.gaussian_matrix(100, 300, 8)
    r = idk.sketch_rid(dev(a), 20, 5, seed=77, omega_mode=idk.OMEGA_MT19937)
    rcols, rz, _ = ref.sketch_id(a, 20, ref.generate(1, 25, 100, 77))
    assert np.array_equal(host(r.cols), rcols)
    assert rel(host(r.z), rz) <= ZTOL


def test_philox_omega_matches_oracle(idk, oracle):
    om = host(idk.sketch_omega(37, 501, 123456789))
    want = oracle.omega_philox(37, 501, 123456789)
    assert np.max(np.abs(om - want)) <= 1e-13
    r = idk.sketch_rid(dev(oracle.gaussian_matrix(60, 80, 3)), 10, 4, seed=99)
    r2 = idk.sketch_rid(dev(oracle.gaussian_matrix(60, 80, 3)), 10, 4, seed=99, omega_mode=idk.OMEGA_VERBATIM,
                        omega=dev(oracle.omega_philox(14, 60, 99)))
    assert np.array_equal(host(r.cols), host(r2.cols))
    assert rel(host(r.z), host(r2.z)) <= 1e-12


def test_sketch_gemm_matches_reference_matmul(idk, ref):
    for (l, m, n) in [(7, 33, 65), (110, 2000, 333), (272, 300, 129), (72, 1000, 4097)]:
        om = ref.generate(1, l, m, 5)
        a = ref.gaussian_matrix(m, n, 6)
        y = host(idk.sketch(dev(om), dev(a)))
        assert rel(y, ref.matmul(om, a)) <= 1e-13
        yt = host(idk.sketch(dev(om), dev(a.T), transposed=True))
        assert rel(yt, ref.matmul(om, a)) <= 1e-13


@pytest.mark.parametrize("l,m,n", [(1, 5, 7), (7, 33, 65), (17, 2001, 130), (110, 2000, 333), (272, 300, 129),
                                   (72, 1000, 4097), (130, 64, 64)])
def test_tma_sketch_bit_identical_to_cp_async_kernel(idk, ref, monkeypatch, l, m, n):
    """The TMA-fed DMMA GEMM (sketch_tma.cu: zero-filled boxes, swizzled
    fragments) and the cp.async kernel (IDK_GEMM_TMA=0) run the same DMMA
    sequence per output tile and the same split order: bit-identical Y, both
    layouts, also through a padded leading dimension."""
    import torch
    om = ref.generate(1, l, m, 5)
    a = ref.gaussian_matrix(m, n, 6)
    big = torch.zeros((n, m + 6), dtype=torch.float64, device="cuda")  # lda = m + 6 (even)
    big[:, :m] = torch.from_numpy(np.ascontiguousarray(a.T))
    a_pad = big.t()[:m, :]
    outs = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("IDK_GEMM_TMA", mode)
        outs[mode] = (host(idk.sketch(dev(om), dev(a))), host(idk.sketch(dev(om), dev(a.T), transposed=True)),
                      host(idk.sketch(dev(om), a_pad)))
    for x, y in zip(outs["1"], outs["0"]):
        assert np.array_equal(x, y)
    assert rel(outs["1"][0], ref.matmul(om, a)) <= 1e-13


def test_dual_sketch_matches_reference_on_transpose(idk, ref):
    """id_auto randomized on a tall A == sketch composition on A^T, without forming A^T on the GPU."""
    a = ref.gaussian_matrix(900, 120, 31)
    k, p = 16, 4
    omega = ref.generate(1, k + p, 120, 5)
    r = idk.sketch_rid(dev(a), k, p, omega_mode=idk.OMEGA_VERBATIM, omega=dev(omega), transposed=True)
    rcols, rz, rc = ref.sketch_id(np.asfortranarray(a.T), k, omega)
    assert np.array_equal(host(r.cols), rcols)
    assert rel(host(r.z), rz) <= ZTOL
    assert np.array_equal(host(r.c), rc)


def test_batched_bit_identical_to_reference_composition(idk, ref):
    import torch
    batch, m, n, k = 37, 64, 256, 16
    from paper_2105_07076_b200.configs import low_rank_batch_np
    a = low_rank_batch_np(batch, m, n, 16, 1e-4, 3)
    ctx = idk.context(0)
    ctx.set_batched_exact(True)
    try:
        cols, z, c = idk.optim_id_batched(torch.from_numpy(a).cuda(), k)
    finally:
        ctx.set_batched_exact(False)
    cols, z, c = host(cols), host(z), host(c)
    for b in range(batch):
        ab = np.asfortranarray(a[b].T)
        rcols, rz, rc = ref.sketch_id(ab, k, None)
        assert np.array_equal(cols[b], rcols)
        assert np.array_equal(z[b].T, rz), b
        assert np.array_equal(c[b].T, rc)
        if b < 5:
            ocols, oz, _ = ref.optim_id(ab, k)
            assert np.array_equal(cols[b], ocols)
            assert rel(z[b].T, oz) <= ZTOL


@pytest.mark.parametrize("batch,m,n,k,noise", [(300, 64, 256, 16, 1e-4), (57, 64, 256, 16, 1e-8), (40, 48, 200, 12, 1e-3),
                                               (33, 64, 128, 32, 1e-2), (20, 20, 60, 5, 1e-4)])
def test_batched_fast_matches_reference(idk, ref, batch, m, n, k, noise):
    """Throughput kernel (default): identical columns, Z within 1e-10, C exact."""
    import torch
    from paper_2105_07076_b200.configs import low_rank_batch_np
    a = low_rank_batch_np(batch, m, n, k, noise, 5)
    cols, z, c = idk.optim_id_batched(torch.from_numpy(a).cuda(), k)
    cols, z, c = host(cols), host(z), host(c)
    for b in range(batch):
        ab = np.asfortranarray(a[b].T)
        rcols, rz, rc = ref.sketch_id(ab, k, None)
        assert np.array_equal(cols[b], rcols), b
        assert rel(z[b].T, rz) <= ZTOL, b
        assert np.array_equal(c[b].T, rc), b


def test_batched_rank_deficient_raises(idk):
    import torch
    a = torch.zeros((3, 8, 6), dtype=torch.float64, device="cuda")
    a[:, 0, :] = 1.0
    with pytest.raises(idk.NotPositiveDefiniteError):
        idk.optim_id_batched(a, 2)


def test_host_entry_matches_device_entry(idk, oracle):
    a = oracle.gaussian_matrix(50, 70, 4)
    h = idk.id_auto(a, 9, idk.RANDOMIZED, seed=5, p=3)
    d = idk.id_auto(dev(a), 9, idk.RANDOMIZED, seed=5, p=3)
    assert np.array_equal(h.cols, host(d.cols)) and np.array_equal(h.z, host(d.z))
    assert np.array_equal(h.c, host(d.c))


@pytest.mark.parametrize("method", [0, 1])
def test_pipelined_host_entry_matches_single_calls(idk, oracle, method):
    mats = [oracle.gaussian_matrix(60, 90, s) for s in range(6)]
    mats = [np.asfortranarray(x) for x in mats]
    cols, zs, cs, tr = idk.id_auto_many(mats, 8, method, seed=3, p=4)
    assert not tr
    tall = [np.asfortranarray(oracle.gaussian_matrix(90, 60, s)) for s in range(3)]
    tcols, tzs, tcs, ttr = idk.id_auto_many(tall, 8, method, seed=3, p=4)
    assert ttr
    for x, c_, z_ in zip(tall, tcols, tzs):
        r = idk.id_auto(x, 8, method, seed=3, p=4)
        assert np.array_equal(c_, r.cols) and np.array_equal(z_, r.z)
    for x, c_, z_, cc in zip(mats, cols, zs, cs):
        r = idk.id_auto(x, 8, method, seed=3, p=4)
        assert np.array_equal(c_, r.cols) and np.array_equal(z_, r.z) and np.array_equal(cc, r.c)


def test_pipelined_host_entry_reports_failing_index(idk, oracle):
    good = oracle.gaussian_matrix(10, 12, 1)
    bad = np.zeros((10, 12))
    g = oracle.gaussian_matrix(10, 2, 8)
    bad[:, 3], bad[:, 9] = g[:, 0], g[:, 1]
    with pytest.raises(idk.NotPositiveDefiniteError, match="matrix 2"):
        idk.id_auto_many([good, good, bad, good], 3, idk.DETERMINISTIC)


@pytest.mark.parametrize("method", [0, 1, 2])
@pytest.mark.parametrize("shape,k", [((110, 4000), 100), ((60, 90), 8), ((90, 60), 8)])
def test_concurrent_batch_entry_matches_single_calls(idk, oracle, method, shape, k):
    """idk_id_auto_batch: 11 IDs over 4 lanes give the bit-identical results of
    single idk_id_auto calls (same kernels, same per-ID workspace layout)."""
    mats = [dev(oracle.gaussian_matrix(shape[0], shape[1], 40 + s)) for s in range(11)]
    seeds = [100 + s for s in range(11)]
    cols, zs, cs, tr = idk.id_auto_batch(mats, k, method, seeds=seeds, p=5, lanes=4)
    assert tr == (shape[0] > shape[1])
    for x, sd, c_, z_, cc in zip(mats, seeds, cols, zs, cs):
        r = idk.id_auto(x, k, method, seed=sd, p=5, oversampling_fraction=5 / k if method == 2 else None)
        assert np.array_equal(host(c_), host(r.cols))
        assert np.array_equal(host(z_), host(r.z))
        assert np.array_equal(host(cc), host(r.c))


def test_concurrent_batch_entry_reports_failing_index(idk, oracle):
    good = dev(oracle.gaussian_matrix(10, 12, 1))
    bad = np.zeros((10, 12))
    g = oracle.gaussian_matrix(10, 2, 8)
    bad[:, 3], bad[:, 9] = g[:, 0], g[:, 1]
    with pytest.raises(idk.NotPositiveDefiniteError, match="matrix 2"):
        idk.id_auto_batch([good, good, dev(bad), good], 3, idk.DETERMINISTIC, lanes=3)


@pytest.mark.parametrize("shape,k,method", [((40, 70), 9, 0), ((300, 500), 40, 1), ((900, 120), 16, 1), ((120, 90), 7, 0)])
def test_diagnostics_and_approx_match_reference(idk, ref, shape, k, method):
    """id.cpp:97-122 on the device (fused residual) vs the reference's diagnostics."""
    a = ref.gaussian_matrix(shape[0], shape[1], 21)
    r = idk.id_auto(dev(a), k, method, seed=4, p=3)
    d = idk.diagnostics(dev(a), r)
    ap = host(idk.approx(r))
    cols, z = host(r.cols), host(r.z)
    rd = ref.diagnostics(a, cols, z, ap)
    assert abs(d["relative_error"] - rd["relative_error"]) <= 1e-12 * max(rd["relative_error"], 1e-300)
    assert d["max_abs_z"] == rd["max_abs_z"]
    assert abs(d["identity_deviation"] - rd["identity_deviation"]) <= 1e-15
    assert d["entry_bound_satisfied"] == rd["entry_bound_satisfied"]
    if r.transposed:
        want = z.T @ a[cols, :]
    else:
        want = a[:, cols] @ z
    assert rel(ap, want) <= 1e-13


@pytest.mark.parametrize("chunk,grouped", [("1", "1"), ("3", "1"), ("32", "1"), ("4", "0"), ("4", "")])
def test_grouped_sketch_batch_matches_single_calls(idk, oracle, monkeypatch, chunk, grouped):
    """The grouped sketch path of idk_id_auto_batch (one Omega launch + one DMMA
    GEMM per chunk of IDs on a low-priority stream, CPQR on the lanes) is
    bit-identical to single idk_id_auto calls for any chunk size, tall or wide."""
    monkeypatch.setenv("IDK_BATCH_CHUNK", chunk)
    monkeypatch.setenv("IDK_BATCH_GROUPED", grouped)
    for shape, k in (((110, 2100), 30), ((700, 90), 12)):
        mats = [dev(oracle.gaussian_matrix(shape[0], shape[1], 70 + s)) for s in range(7)]
        seeds = [300 + s for s in range(7)]
        cols, zs, cs, tr = idk.id_auto_batch(mats, k, idk.RANDOMIZED, seeds=seeds, p=6, lanes=3)
        assert tr == (shape[0] > shape[1])
        for x, sd, c_, z_, cc in zip(mats, seeds, cols, zs, cs):
            r = idk.id_auto(x, k, idk.RANDOMIZED, seed=sd, p=6)
            assert np.array_equal(host(c_), host(r.cols))
            assert np.array_equal(host(z_), host(r.z))
            assert np.array_equal(host(cc), host(r.c))


def test_batched_host_entry_matches_device_entry(idk, oracle):
    """idk_optim_id_batched_host (chunks of 2 x num_SMs matrices through a
    3-deep upload / factor / download pipeline) returns exactly the device
    entry's results, across chunk boundaries; a rank-deficient matrix in a
    later chunk is reported with its batch index."""
    import torch
    from paper_2105_07076_b200.configs import make_np
    a = make_np("cfg3", seed=21, scale=700 / 4096)  # (700, n, m): 3 chunks on a 148-SM B200
    cols_h, z_h, c_h = idk.optim_id_batched(a, 16)
    cols_d, z_d, c_d = idk.optim_id_batched(torch.from_numpy(a).cuda(), 16)
    assert np.array_equal(cols_h, host(cols_d))
    assert np.array_equal(z_h, host(z_d))
    assert np.array_equal(c_h, host(c_d))
    bad = a.copy()
    bad[650] = 0.0
    with pytest.raises(idk.NotPositiveDefiniteError, match="matrix 650"):
        idk.optim_id_batched(bad, 16)


def test_batched_kernel_variants_agree(tmp_path):
    """IDK_BATCHED_GROUP selects the batched ID kernel when the library first runs one: the
    default (two threads per column, batched_group.cu) and 0 (one thread per column,
    batched_fast.cu) must pick the same columns and agree on Z within rounding."""
    import os
    import subprocess
    import sys
    script = tmp_path / "run_batched.py"
    script.write_text(
        "import sys, numpy as np, torch\n"
        "sys.path.insert(0, %r)\n"
        "import paper_2105_07076_b200 as idk\n"
        "from paper_2105_07076_b200.configs import low_rank_batch_np\n"
        "a = low_rank_batch_np(150, 64, 256, 16, 1e-4, 11)\n"
        "cols, z, c = idk.optim_id_batched(torch.from_numpy(a).cuda(), 16)\n"
        "np.savez(sys.argv[1], cols=cols.cpu().numpy(), z=z.cpu().numpy(), c=c.cpu().numpy())\n"
        % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    out = {}
    for g in ("0", "2"):
        env = dict(os.environ, IDK_BATCHED_GROUP=g)
        path = tmp_path / f"out{g}.npz"
        subprocess.run([sys.executable, str(script), str(path)], check=True, env=env, timeout=600)
        out[g] = np.load(path)
    assert np.array_equal(out["0"]["cols"], out["2"]["cols"])
    assert np.array_equal(out["0"]["c"], out["2"]["c"])
    assert rel(out["0"]["z"], out["2"]["z"]) <= 1e-12

"""GPU: the sharded stages (sketch of a column block, id_from_sketch on the
gathered sketch, owner gathers) reproduce the single-GPU ID bit for bit --
emulating G ranks on one device by running each rank's stages in turn."""
import numpy as np
import pytest
import torch

from paper_2105_07076_b200.sharded import CudaStages, column_range

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.asfortranarray(a, dtype=np.float64)).cuda()


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("transposed", [False, True])
def test_emulated_ranks_match_single_gpu(oracle, world, transposed):
    import paper_2105_07076_b200 as idk
    st = CudaStages()
    if transposed:
        a = oracle.gaussian_matrix(3000, 120, 4)  # tall: M = A^T is 120 x 3000
        m, n = 120, 3000
    else:
        a = oracle.gaussian_matrix(300, 2500, 4)
        m, n = 300, 2500
    a[::7] *= 2.0
    k, p, seed = 24, 6, 99
    ref = idk.sketch_rid(dev(a), k, p, seed=seed, transposed=transposed)
    rcols, rz, rc = ref.cols.cpu().numpy(), ref.z.cpu().numpy(), ref.c.cpu().numpy()
    omega = st.omega(k + p, m, seed, dev(a))
    blocks = []
    for r in range(world):
        b, e = column_range(n, world, r)
        local = dev(a[b:e, :]) if transposed else dev(a[:, b:e])
        blocks.append(st.sketch(omega, local, transposed))
    y_all = torch.cat([blk.t() for blk in blocks], dim=0).t()  # l x n column-major
    c_sum = np.zeros((m, k))
    for r in range(world):
        b, e = column_range(n, world, r)
        cols, z_local = st.factor(y_all.clone(), k, b, e)  # factor overwrites Y
        cols = cols.cpu().numpy()
        assert np.array_equal(cols, rcols)
        assert np.array_equal(z_local.cpu().numpy(), rz[:, b:e])
        own = (cols >= b) & (cols < e)
        if own.any():
            local = dev(a[b:e, :]) if transposed else dev(a[:, b:e])
            part = st.gather(local, torch.as_tensor(cols[own] - b).cuda(), transposed).cpu().numpy()
            c_sum[:, own] += part
    assert np.array_equal(c_sum, rc)


def test_single_rank_sharded_api(oracle):
    import paper_2105_07076_b200 as idk
    from paper_2105_07076_b200 import sharded
    a = dev(oracle.gaussian_matrix(200, 900, 2))
    cols, z, c = sharded.sketch_rid_sharded(a, 900, 20, 5, seed=3)
    ref = idk.sketch_rid(a, 20, 5, seed=3)
    assert torch.equal(cols, ref.cols) and torch.equal(z, ref.z) and torch.equal(c, ref.c)


def test_id_from_sketch_rejects_bad_range(oracle):
    import paper_2105_07076_b200 as idk
    y = dev(oracle.gaussian_matrix(30, 100, 1))
    with pytest.raises(idk.InvalidArgument):
        idk.id_from_sketch(y, 10, 50, 120)


@pytest.mark.parametrize("transposed", [False, True])
def test_c_abi_id_sharded_one_rank(oracle, transposed):
    """idk_id_sharded without a communicator (one rank) equals idk_sketch_rid bit for bit."""
    import paper_2105_07076_b200 as idk
    if transposed:
        a = dev(oracle.gaussian_matrix(2600, 150, 6))
        m, n = 150, 2600
    else:
        a = dev(oracle.gaussian_matrix(180, 3100, 6))
        m, n = 180, 3100
    cols, z, c = idk.id_sharded(a, m, n, 30, 8, seed=21, transposed=transposed)
    ref = idk.sketch_rid(a, 30, 8, seed=21, transposed=transposed)
    assert torch.equal(cols, ref.cols) and torch.equal(z, ref.z) and torch.equal(c, ref.c)


def test_c_abi_id_sharded_one_rank_nccl_comm(oracle):
    """The same through an NCCL communicator of size 1 (idk_nccl_unique_id + idk_comm_init)."""
    import paper_2105_07076_b200 as idk
    a = dev(oracle.gaussian_matrix(160, 2000, 8))
    ctx = idk.context(0)
    ctx.comm_init(1, 0, idk.nccl_unique_id())
    try:
        cols, z, c = idk.id_sharded(a, 160, 2000, 25, 5, seed=4)
    finally:
        ctx.comm_destroy()
    ref = idk.sketch_rid(a, 25, 5, seed=4)
    assert torch.equal(cols, ref.cols) and torch.equal(z, ref.z) and torch.equal(c, ref.c)


@pytest.mark.parametrize("transposed", [False, True])
def test_sketch_fanout_writes_every_destination_bit_identical(oracle, transposed):
    """The fused sketch + all-gather of the peer mode (idk_sketch_fanout): one
    rank's block lands in every destination buffer (here three local buffers
    standing in for three ranks' NVLink-mapped Y), bit-identical to the same
    columns of the unsharded sketch (the split-K count of the full n)."""
    import ctypes as C
    import paper_2105_07076_b200 as idk
    if transposed:
        a = dev(oracle.gaussian_matrix(9000, 150, 12))  # M = A^T: 150 x 9000
        m, n = 150, 9000
    else:
        a = dev(oracle.gaussian_matrix(2400, 7000, 12))
        m, n = 2400, 7000
    l, world = 40, 3
    om = idk.sketch_omega(l, m, 5)
    y_full = idk.sketch(om, a, transposed=transposed)
    w = -(-n // world)
    ctx = idk.context(0)
    ctx.bind_stream()
    bufs = [torch.full((world * w, l), float("nan"), dtype=torch.float64, device="cuda") for _ in range(world)]
    for r in range(world):
        b, e = column_range(n, world, r)
        local = (a[b:e, :] if transposed else a[:, b:e]).t().contiguous().t()
        dst = (C.c_void_p * world)(*[C.c_void_p(bf.data_ptr() + 8 * l * b) for bf in bufs])
        ctx.check(ctx.lib.idk_sketch_fanout(ctx.h, C.c_void_p(om.data_ptr()), l, C.c_void_p(local.data_ptr()), m, e - b,
                                            local.stride(1), 1 if transposed else 0, dst, world, l, n))
    for bf in bufs:
        assert torch.equal(bf[:n].t(), y_full)

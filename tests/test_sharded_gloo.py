"""Multi-rank host logic of paper_2105_07076_b200.sharded under gloo on CPU
(world_size 2 and 3), with oracle-backed stages: the assembled (cols, Z, C)
must be bit-identical to the single-process composition on the full matrix
(column blocks of Omega*A are exactly the columns of the full product)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2105_07076_b200.sharded import column_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from cpu_stages import OracleStages, _t
        from oracle import Oracle
        from paper_2105_07076_b200 import sharded
        o = Oracle()
        if case in ("wide", "tall", "narrow"):
            m, n, k, p = {"wide": (40, 97, 8, 3), "tall": (101, 30, 7, 2), "narrow": (30, 9, 4, 2)}[case]
            a = o.gaussian_matrix(m, n, 5)
            a[:, ::4] *= 3.0
            if case == "wide":  # a dominant column holding -0.0 entries: C must keep their sign
                a[:, 9] *= 50.0
                a[:4, 9] = -0.0
            elif case == "tall":
                a[17, :] *= 50.0
                a[17, :3] = -0.0
            if case in ("wide", "narrow"):
                b, e = column_range(n, world, rank)
                local = _t(a[:, b:e])
                cols, z_local, c = sharded.sketch_rid_sharded(local, n, k, p, seed=11, stages=OracleStages())
                assert z_local.shape == (k, e - b)
                ntot = n
            else:  # M = A^T (30 x 101); rank owns rows [b, e) of A = columns of M
                b, e = column_range(m, world, rank)
                local = _t(a[b:e, :])
                cols, z_local, c = sharded.sketch_rid_sharded(local, m, k, p, seed=11, transposed=True,
                                                              stages=OracleStages())
                ntot = m
            z = sharded.gather_result(cols, z_local, ntot)
            if rank == 0:
                np.savez(os.path.join(out_dir, f"{case}.npz"), cols=cols.numpy(), z=z.numpy(), c=c.numpy(), a=a)
        else:  # batched partition
            from paper_2105_07076_b200.configs import low_rank_batch_np
            a = torch.from_numpy(low_rank_batch_np(7, 12, 20, 3, 1e-4, 2))
            bgn, end, cols, z, c = sharded.optim_id_batched_sharded(a, 3, stages=OracleStages())
            np.savez(os.path.join(out_dir, f"batched_{rank}.npz"), begin=bgn, end=end, cols=cols.numpy(),
                     z=z.numpy(), c=c.numpy(), a=a.numpy())
    finally:
        dist.destroy_process_group()


def _run(world, case, tmp_path):
    mp.spawn(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True)


def test_column_range_covers_exactly():
    from paper_2105_07076_b200 import idkit
    for n in (1, 5, 97, 16384, 65536):
        for world in (1, 2, 3, 4, 8):
            spans = [column_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            w = -(-n // world)
            assert all(b == min(r * w, n) and e - b <= w for r, (b, e) in enumerate(spans))
            # the C ABI's split (idk_shard_range) is the same
            assert spans == [idkit.shard_range(n, world, r) for r in range(world)]


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("case", ["wide", "tall"])
def test_sharded_sketch_matches_single_process(world, case, tmp_path, oracle):
    _run(world, case, tmp_path)
    d = np.load(tmp_path / f"{case}.npz")
    a = d["a"]
    k, p = (8, 3) if case == "wide" else (7, 2)
    mat = a if case == "wide" else np.asfortranarray(a.T)
    om = oracle.omega_philox(k + p, mat.shape[0], 11)
    cols, z, c, _ = oracle.interp_decomp(mat, k, om)
    assert np.array_equal(d["cols"], cols)
    assert np.array_equal(d["z"], z)
    assert np.array_equal(d["c"], c)
    assert np.array_equal(np.signbit(d["c"]), np.signbit(c))  # -0.0 survives (no SUM all-reduce)
    assert np.signbit(d["c"]).any()


def test_sharded_with_an_empty_rank(tmp_path, oracle):
    """9 columns over 4 ranks: blocks of 3, the last rank owns none but still
    takes part in the all-gather and the broadcasts."""
    _run(4, "narrow", tmp_path)
    d = np.load(tmp_path / "narrow.npz")
    om = oracle.omega_philox(6, 30, 11)
    cols, z, c, _ = oracle.interp_decomp(d["a"], 4, om)
    assert np.array_equal(d["cols"], cols) and np.array_equal(d["z"], z) and np.array_equal(d["c"], c)


def test_batched_partition_by_matrix(tmp_path, oracle):
    _run(2, "batched", tmp_path)
    seen = []
    for r in range(2):
        d = np.load(tmp_path / f"batched_{r}.npz")
        a = d["a"]
        for j, b in enumerate(range(int(d["begin"]), int(d["end"]))):
            ab = np.asfortranarray(a[b].T)
            cols, z, c, _ = oracle.interp_decomp(ab, 3)
            assert np.array_equal(d["cols"][j], cols)
            assert np.array_equal(d["z"][j].T, z)
            seen.append(b)
    assert sorted(seen) == list(range(7))

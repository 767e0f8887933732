"""The multi-rank C-ABI sharded path (idk_id_sharded) with 2, 3, 4 and 8
processes on one GPU (SURVEY.md section 4 asks for G = 1, 2, 4, 8 on one box): the ranks meet over gloo through idk_set_host_collectives (NCCL does
not allow two ranks on one device), and -- in peer mode -- map each other's Y
buffers by CUDA IPC, so the fused sketch + all-gather (each rank's split-K
reduction storing into every rank's Y) runs across processes.  No kernel waits
on another process: the barriers are host-side.  Every rank's (cols, Z block,
C) must equal the single-process idk_sketch_rid bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, transposed, p2p, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if not p2p:
        os.environ["IDK_SHARD_P2P"] = "0"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import paper_2105_07076_b200 as idk
        from paper_2105_07076_b200 import sharded
        torch.cuda.set_device(0)
        g = torch.Generator(device="cuda")
        g.manual_seed(7)
        if transposed:
            a = torch.randn((5000, 120), generator=g, device="cuda", dtype=torch.float64).t().contiguous().t()
            m, n = 120, 5000
        else:
            a = torch.randn((200, 4100), generator=g, device="cuda", dtype=torch.float64).t().contiguous().t()
            m, n = 200, 4100
        a[:, ::5] *= 3.0 if not transposed else 1.0
        k, p, seed = 24, 8, 31
        ref = idk.sketch_rid(a, k, p, seed=seed, transposed=transposed)
        ctx = sharded.host_collectives_setup(0)
        b, e = sharded.column_range(n, world, rank)
        local = (a[b:e, :] if transposed else a[:, b:e]).t().contiguous().t()
        res = {}
        for it in range(2):  # twice: the second call reuses the mapped peer buffers
            cols, z, c = idk.id_sharded(local, m, n, k, p, seed=seed, transposed=transposed)
            res[it] = (torch.equal(cols, ref.cols), torch.equal(z, ref.z[:, b:e]), torch.equal(c, ref.c))
        mode = ctx.lib.idk_shard_peer_mode(ctx.h)
        np.save(os.path.join(out_dir, f"r{rank}.npy"), np.array([all(res[0]), all(res[1]), mode == (1 if p2p else -1)]))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,transposed,p2p", [(2, False, True), (2, True, True), (2, False, False),
                                                  (2, True, False), (3, False, True), (3, True, False),
                                                  (4, False, True), (4, True, True), (8, False, True)])
def test_c_abi_sharded_multi_process(tmp_path, world, transposed, p2p):
    mp.spawn(_worker, args=(world, _free_port(), transposed, p2p, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        ok = np.load(tmp_path / f"r{r}.npy")
        assert ok.all(), (r, ok)

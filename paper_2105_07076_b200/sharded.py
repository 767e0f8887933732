"""Multi-GPU ID: one process per GPU.

SURVEY.md 8(e):
  * cfg3 (batched small IDs): partition by matrix, no collective.
  * cfg4 (wide A) / cfg5 (tall A, id_auto dual): the decomposed matrix M is
    sharded by column blocks (for cfg5: row blocks of the stored A), ceil-sized
    so rank r's block starts at column r*w (w = ceil(n / world)).  Each rank
      1. draws the same Omega (counter-based RNG: identical on every rank),
      2. sketches its block straight into its slot of the full Y buffer,
      3. all-gathers Y in place (one all_gather_into_tensor / ncclAllGather,
         35-38 MB at cfg4/cfg5),
      4. runs the deterministic CPQR of Y itself (bit-identical on every rank,
         so every rank agrees on the pivots without a broadcast),
      5. solves Z only for its own columns,
      6. gathers the pivot columns it owns; each owner broadcasts them, so C is
         assembled exactly (no reduction, -0.0 stays -0.0).

Two front ends share the split:
  * ``id_sharded_nccl``: the whole chain inside one C-ABI call
    (``idk_id_sharded`` over the library's own NCCL communicator,
    ``nccl_setup`` bootstraps it through torch.distributed) -- the product path.
  * ``sketch_rid_sharded``: the same chain with torch.distributed collectives
    and injectable stages, so the host logic is testable with gloo on CPU
    (tests/cpu_stages.py supplies oracle-backed stages).
There is no CPU path for the computation in this module.
"""
from __future__ import annotations

from typing import Optional, Tuple

import torch
import torch.distributed as dist


def column_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Columns [begin, end) of rank `rank`: ceil-sized contiguous blocks
    (w = ceil(n / world)), the split of idk_shard_range, so rank r's block
    starts at column r * w of the gathered Y."""
    w = -(-n // world)
    begin = min(rank * w, n)
    return begin, min(begin + w, n)


def world_rank(group=None) -> Tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def fortran_empty(rows: int, cols: int, like: torch.Tensor) -> torch.Tensor:
    return torch.empty((cols, rows), dtype=like.dtype, device=like.device).t()


class CudaStages:
    """The ID stages on this rank's GPU, through the C ABI."""

    def __init__(self):
        from . import idkit
        self.idk = idkit

    def omega(self, l: int, m: int, seed: int, like: torch.Tensor) -> torch.Tensor:
        return self.idk.sketch_omega(l, m, seed, device=like.device.index or 0)

    def sketch(self, omega: torch.Tensor, a_local: torch.Tensor, transposed: bool) -> torch.Tensor:
        return self.idk.sketch(omega, a_local, transposed=transposed)

    def factor(self, y: torch.Tensor, k: int, c_begin: int, c_end: int):
        return self.idk.id_from_sketch(y, k, c_begin, c_end)

    def gather(self, a_local: torch.Tensor, idx: torch.Tensor, rows_of_a: bool) -> torch.Tensor:
        return self.idk.select_columns(a_local, idx, rows_of_a=rows_of_a)

    def batched(self, a_local: torch.Tensor, k: int):
        return self.idk.optim_id_batched(a_local, k)


def sketch_rid_sharded(a_local: torch.Tensor, n_total: int, k: int, p: int, seed: int = 0,
                       transposed: bool = False, group=None, stages=None):
    """Column-sharded Gaussian-sketch RID (torch.distributed collectives).

    a_local: this rank's block of M's columns column_range(n_total, world, rank)
             (column-major m x n_r), or, with transposed=True, this rank's row
             block of the stored tall A (n_r x m, column-major), i.e. the same
             columns of M = A^T.
    Returns (cols, z_local, c): cols (k,) global column ids of M (row ids of A when
    transposed), z_local (k x n_r) = Z[:, begin:end], c (m x k) on every rank.
    """
    stages = stages or CudaStages()
    world, rank = world_rank(group)
    begin, end = column_range(n_total, world, rank)
    w = -(-n_total // world)
    m = a_local.shape[1] if transposed else a_local.shape[0]
    n_r = a_local.shape[0] if transposed else a_local.shape[1]
    if n_r != end - begin:
        raise ValueError(f"rank {rank}: local block has {n_r} columns, expected {end - begin}")
    l = k + p
    omega = stages.omega(l, m, seed, a_local)
    # Y (l x world*w, column-major) is stored as (world*w, l) rows: rank r's slot is rows [r*w, (r+1)*w)
    y_store = torch.empty((world * w, l), dtype=a_local.dtype, device=a_local.device)
    if n_r > 0:
        y_store[begin:end] = stages.sketch(omega, a_local, transposed).t()
    if world > 1:
        slot = y_store[rank * w:(rank + 1) * w]
        dist.all_gather_into_tensor(y_store.view(-1), slot.reshape(-1), group=group)
    y = y_store[:n_total].t()                                     # l x n, ld = l
    cols, z_local = stages.factor(y, k, begin, end)
    c_store = torch.empty((k, m), dtype=a_local.dtype, device=a_local.device)  # (k, m) rows = C's columns
    own = (cols >= begin) & (cols < end)
    if bool(own.any()):
        c_store[own] = stages.gather(a_local, cols[own] - begin, transposed).t()
    if world > 1:
        owner = torch.div(cols, w, rounding_mode="floor")
        for r in range(world):  # each owner broadcasts its columns: exact, no reduction
            sel = torch.nonzero(owner == r).flatten()
            if sel.numel() == 0:
                continue
            blk = c_store[sel].contiguous()
            dist.broadcast(blk, src=r, group=group)
            c_store[sel] = blk
    return cols, z_local, c_store.t()


def nccl_setup(device: int, group=None):
    """Give this rank's C-ABI context an NCCL communicator over the ranks of the
    torch.distributed group (rank 0's ncclUniqueId travels by broadcast_object_list)."""
    from . import idkit
    world, rank = world_rank(group)
    ctx = idkit.context(device)
    if world == 1:
        return ctx
    uid = [idkit.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0, group=group)
    ctx.comm_init(world, rank, uid[0])
    return ctx


def host_collectives_setup(device: int, group=None):
    """Give this rank's C-ABI context host collectives over the torch.distributed
    group (any backend, e.g. gloo on CPU) instead of NCCL: the transport for
    setups without NCCL, and how the multi-rank C-ABI path is tested with
    several processes on one GPU (tests/test_gpu_sharded_capi.py)."""
    import ctypes as C
    from . import idkit
    world, rank = world_rank(group)
    ctx = idkit.context(device)

    def allgather(send, recv, nbytes):
        src = torch.frombuffer((C.c_char * nbytes).from_address(send), dtype=torch.uint8).clone()
        out = torch.empty(world * nbytes, dtype=torch.uint8)
        dist.all_gather_into_tensor(out, src, group=group)
        C.memmove(recv, out.data_ptr(), world * nbytes)

    def broadcast(buf, nbytes, root):
        t = torch.frombuffer((C.c_char * nbytes).from_address(buf), dtype=torch.uint8).clone()
        dist.broadcast(t, src=root, group=group)
        C.memmove(buf, t.data_ptr(), nbytes)

    def barrier():
        dist.barrier(group=group)

    ctx.set_host_collectives(world, rank, allgather, broadcast, barrier)
    return ctx


def id_sharded_nccl(a_local: torch.Tensor, n_total: int, k: int, p: int, seed: int = 0, transposed: bool = False):
    """The product path: sketch -> in-place ncclAllGather(Y) -> replicated CPQR ->
    local Z -> owner broadcasts of C, all inside idk_id_sharded (call nccl_setup once)."""
    from . import idkit
    m = a_local.shape[1] if transposed else a_local.shape[0]
    return idkit.id_sharded(a_local, m, n_total, k, p, seed=seed, transposed=transposed)


def batched_partition(batch: int, world: int, rank: int) -> Tuple[int, int]:
    return column_range(batch, world, rank)


def optim_id_batched_sharded(a: torch.Tensor, k: int, group=None, stages=None, already_local: bool = False):
    """cfg3: partition the (batch, n, m) stack by matrix; no collective.
    Returns (begin, end, cols, z, c) for this rank's matrices."""
    stages = stages or CudaStages()
    world, rank = world_rank(group)
    if already_local:
        begin, end, local = 0, a.shape[0], a
    else:
        begin, end = batched_partition(a.shape[0], world, rank)
        local = a[begin:end].contiguous()
    cols, z, c = stages.batched(local, k)
    return begin, end, cols, z, c


def gather_result(cols: torch.Tensor, z_local: torch.Tensor, n_total: int, group=None) -> Optional[torch.Tensor]:
    """Assemble the full Z (k x n) on every rank (tests / small problems only)."""
    world, rank = world_rank(group)
    if world == 1:
        return z_local
    k = z_local.shape[0]
    widths = [column_range(n_total, world, r) for r in range(world)]
    wmax = max(e - b for b, e in widths)
    send = torch.zeros((wmax, k), dtype=z_local.dtype, device=z_local.device)
    send[: z_local.shape[1]] = z_local.t()
    recv = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(recv, send, group=group)
    return torch.cat([recv[r][: e - b] for r, (b, e) in enumerate(widths)], dim=0).t()

"""Multi-GPU ID: one process per GPU, torch.distributed for the plumbing.

SURVEY.md 8(e):
  * cfg3 (batched small IDs): partition by matrix, no collective.
  * cfg4 (wide A) / cfg5 (tall A, id_auto dual): A is sharded by column blocks
    of the decomposed matrix M (for cfg5: row blocks of the stored A).  Each rank
      1. draws the same Omega (counter-based RNG: identical on every rank),
      2. sketches its block, Y_r = Omega M_r (local DMMA GEMM, no communication),
      3. all-gathers the small sketch Y (l x n, 35-38 MB at cfg4/cfg5),
      4. runs the deterministic CPQR of Y itself (bit-identical on every rank,
         so every rank agrees on the pivots without a broadcast),
      5. solves Z only for its own columns (idk_id_from_sketch),
      6. gathers the selected columns/rows of A it owns; one all-reduce
         assembles C (exact: every entry has a single non-zero contributor).
The compute stages are the C-ABI kernels (CudaStages); there is no CPU path in
this module.  `stages` is injectable so the host logic is testable with gloo
on CPU (tests/cpu_stages.py supplies the oracle-backed stages).
"""
from __future__ import annotations

from typing import Optional, Tuple

import torch
import torch.distributed as dist


def column_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Balanced contiguous split of n columns over `world` ranks."""
    base, extra = divmod(n, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


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
    """Column-sharded Gaussian-sketch RID.

    a_local: this rank's block of M's columns [begin, end) (column-major m x n_r),
             or, with transposed=True, this rank's row block of the stored tall A
             (n_r x m, column-major), i.e. the same columns of M = A^T.
    Returns (cols, z_local, c): cols (k,) global column ids of M (row ids of A when
    transposed), z_local (k x n_r) = Z[:, begin:end], c (m x k) replicated.
    """
    stages = stages or CudaStages()
    world, rank = world_rank(group)
    begin, end = column_range(n_total, world, rank)
    m = a_local.shape[1] if transposed else a_local.shape[0]
    n_r = a_local.shape[0] if transposed else a_local.shape[1]
    if n_r != end - begin:
        raise ValueError(f"rank {rank}: local block has {n_r} columns, expected {end - begin}")
    l = k + p
    omega = stages.omega(l, m, seed, a_local)
    y_local = stages.sketch(omega, a_local, transposed)          # l x n_r, column-major
    y = _all_gather_columns(y_local, n_total, world, group)       # l x n, column-major
    cols, z_local = stages.factor(y, k, begin, end)
    own = (cols >= begin) & (cols < end)
    c = torch.zeros((k, m), dtype=a_local.dtype, device=a_local.device).t()
    if bool(own.any()):
        idx = (cols[own] - begin)
        c[:, own] = stages.gather(a_local, idx, transposed)
    if world > 1:
        c_rows = c.t().contiguous()  # (k, m) storage == column-major m x k
        dist.all_reduce(c_rows, op=dist.ReduceOp.SUM, group=group)
        c = c_rows.t()
    return cols, z_local, c


def _all_gather_columns(y_local: torch.Tensor, n_total: int, world: int, group) -> torch.Tensor:
    """Concatenate column-major l x n_r blocks from every rank into l x n_total."""
    if world == 1:
        return y_local
    l = y_local.shape[0]
    widths = [column_range(n_total, world, r) for r in range(world)]
    wmax = max(e - b for b, e in widths)
    send = torch.zeros((wmax, l), dtype=y_local.dtype, device=y_local.device)
    send[: y_local.shape[1]] = y_local.t()
    recv = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(recv, send, group=group)
    full = torch.cat([recv[r][: e - b] for r, (b, e) in enumerate(widths)], dim=0)  # (n, l) rows
    return full.t()


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

"""paper_2105_07076_b200 -- B200-native interpolative decomposition (ID) path.

Drop-in for the hot path of the reference library idkit (arXiv 2105.07076,
"Optim ID / Optim RID"): Gaussian sketch -> column-pivoted Householder QR ->
Z = [I | R11^-1 R12] P^T -> C = A[:, cols], as hand-written sm_100a kernels
behind the C ABI in include/idkit_b200.h.  `idkit` is the Python mirror of the
reference's C++ API; `sharded` is the multi-GPU (torch.distributed) layer.
"""
from .idkit import (DETERMINISTIC, OMEGA_MT19937, OMEGA_PHILOX, OMEGA_VERBATIM, RANDOMIZED, SAMPLED, Context, CudaError,
                    IdkitError, IdResult, InvalidArgument, NotPositiveDefiniteError, PivotedQr, SingularMatrixError,
                    approx, context, diagnostics, id_sharded, nccl_unique_id, shard_range, matmul_ref, id_auto, id_auto_batch, id_auto_many, id_from_sketch, optim_id, optim_id_batched, optim_rid, qr_column_pivoted, select_columns, sketch,
                    sketch_omega, sketch_rid)

__all__ = [
    "DETERMINISTIC", "RANDOMIZED", "SAMPLED", "OMEGA_PHILOX", "OMEGA_MT19937", "OMEGA_VERBATIM", "Context", "CudaError",
    "IdkitError", "IdResult", "InvalidArgument", "NotPositiveDefiniteError", "PivotedQr", "SingularMatrixError",
    "approx", "context", "diagnostics", "id_sharded", "nccl_unique_id", "shard_range", "matmul_ref", "id_auto", "id_auto_batch", "id_auto_many", "id_from_sketch", "optim_id", "optim_id_batched", "optim_rid", "qr_column_pivoted", "select_columns", "sketch",
    "sketch_omega", "sketch_rid",
]

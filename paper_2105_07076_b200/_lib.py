"""ctypes binding of libidkit_b200.so (the C ABI in include/idkit_b200.h).

Loading fails loudly: there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IDK_LIB_PATH") or os.path.join(PKG, "libidkit_b200.so")  # override: A/B of tuning builds

# Every symbol include/idkit_b200.h declares, with its ctypes signature.
_P = C.c_void_p
_I64 = C.c_int64
SIGNATURES = {
    "idk_abi_version": (C.c_int, []),
    "idk_create": (C.c_int, [C.POINTER(_P), C.c_int]),
    "idk_destroy": (C.c_int, [_P]),
    "idk_set_stream": (C.c_int, [_P, _P]),
    "idk_last_error": (C.c_char_p, [_P]),
    "idk_status_string": (C.c_char_p, [C.c_int]),
    "idk_kernel_launches": (C.c_int64, [_P]),
    "idk_set_profiling": (C.c_int, [_P, C.c_int]),
    "idk_set_cpqr_mode": (C.c_int, [_P, C.c_int]),
    "idk_set_batched_exact": (C.c_int, [_P, C.c_int]),
    "idk_set_sketch_order": (C.c_int, [_P, C.c_int]),
    "idk_debug_cpqr_trace": (C.c_int, [_P, _P]),
    "idk_cpqr_plan": (C.c_int, [_P, _I64, _I64, _I64, C.POINTER(C.c_int64)]),
    "idk_stage_times": (C.c_int, [_P, C.POINTER(C.c_double), C.c_int]),
    "idk_optim_id": (C.c_int, [_P, _P, _I64, _I64, _I64, _I64, _P, _P, _P]),
    "idk_sketch_rid": (C.c_int, [_P, _P, _I64, _I64, _I64, C.c_int, _I64, _I64, C.c_uint64, C.c_int, _P, _P, _P, _P]),
    "idk_id_auto_batch": (C.c_int, [_P, _I64, _P, _I64, _I64, _I64, _I64, C.c_int, _P, _I64, C.c_int, _P, _P, _P,
                                    C.POINTER(C.c_int)]),
    "idk_set_concurrency": (C.c_int, [_P, C.c_int]),
    "idk_qr_column_pivoted_host": (C.c_int, [_P, _P, _I64, _I64, _I64, _P, _P, _P]),
    "idk_optim_id_host": (C.c_int, [_P, _P, _I64, _I64, _I64, _P, _P, _P, _P]),
    "idk_optim_rid_host": (C.c_int, [_P, _P, _I64, _I64, _I64, C.c_double, C.c_uint64, _P, _P, _P, _P]),
    "idk_id_auto_ref_host": (C.c_int, [_P, _P, _I64, _I64, _I64, C.c_int, C.c_uint64, C.c_double, _I64, _P, _P, _P,
                                       _P, C.POINTER(C.c_int)]),
    "idk_matmul_ref": (C.c_int, [_P, _P, _I64, _I64, _I64, _P, _I64, _I64, _P, _I64]),
    "idk_optim_rid": (C.c_int, [_P, _P, _I64, _I64, _I64, C.c_int, _I64, C.c_double, C.c_uint64, _P, _P, _P]),
    "idk_id_auto": (C.c_int, [_P, _P, _I64, _I64, _I64, _I64, C.c_int, C.c_uint64, _I64, C.c_int, _P, _P, _P, _P,
                              C.POINTER(C.c_int)]),
    "idk_optim_id_batched": (C.c_int, [_P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _P, _P, _P]),
    "idk_optim_id_batched_host": (C.c_int, [_P, _P, _I64, _I64, _I64, _I64, _P, _P, _P]),
    "idk_id_from_sketch": (C.c_int, [_P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _P, _P]),
    "idk_sketch_omega": (C.c_int, [_P, _I64, _I64, C.c_uint64, _P]),
    "idk_sketch": (C.c_int, [_P, _P, _I64, _P, _I64, _I64, _I64, C.c_int, _P, _I64]),
    "idk_qr_column_pivoted": (C.c_int, [_P, _P, _I64, _I64, _I64, _I64, _P, _P, _P]),
    "idk_select_columns": (C.c_int, [_P, _P, _I64, _I64, _I64, _P, _I64, C.c_int, _P]),
    "idk_approx": (C.c_int, [_P, _P, _I64, _I64, _P, _I64, _P, _I64]),
    "idk_diagnostics": (C.c_int, [_P, _P, _I64, _I64, _I64, C.c_int, _P, _I64, _P, _P, C.POINTER(C.c_double)]),
    "idk_id_auto_host_many": (C.c_int, [_P, _I64, _P, _I64, _I64, _I64, C.c_int, C.c_uint64, _I64, C.c_int, _P, _P, _P,
                                        C.POINTER(C.c_int)]),
    "idk_shard_range": (C.c_int, [_I64, C.c_int, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "idk_nccl_unique_id": (C.c_int, [_P]),
    "idk_comm_init": (C.c_int, [_P, C.c_int, C.c_int, _P]),
    "idk_set_nccl_comm": (C.c_int, [_P, _P]),
    "idk_comm_destroy": (C.c_int, [_P]),
    "idk_set_host_collectives": (C.c_int, [_P, C.c_int, C.c_int, _P]),
    "idk_shard_peer_mode": (C.c_int, [_P]),
    "idk_sketch_fanout": (C.c_int, [_P, _P, _I64, _P, _I64, _I64, _I64, C.c_int, _P, C.c_int, _I64, _I64]),
    "idk_id_sharded": (C.c_int, [_P, _P, _I64, _I64, _I64, C.c_int, _I64, _I64, C.c_uint64, C.c_int, _P, _P, _P, _P]),
    "idk_id_auto_host": (C.c_int, [_P, _P, _I64, _I64, _I64, C.c_int, C.c_uint64, _I64, C.c_int, _P, _P, _P,
                                   C.POINTER(C.c_int)]),
}

_lock = threading.Lock()
_lib = None


class IdkitLibraryMissing(ImportError):
    pass


def load(path: str | None = None):
    """Load (once) and type the C-ABI library; raise if it is absent."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise IdkitLibraryMissing(
                f"{p} not built: run `python -m paper_2105_07076_b200.build` (nvcc, sm_100a). "
                "There is no CPU fallback.")
        lib = C.CDLL(p)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.idk_abi_version() != 1:
            raise IdkitLibraryMissing(f"{p}: unexpected ABI version {lib.idk_abi_version()}")
        if path is None:
            _lib = lib
        return lib

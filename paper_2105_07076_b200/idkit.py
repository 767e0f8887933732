"""Host-side mirror of the reference's ID interface (proj/include/idkit/id.hpp,
qr.hpp, matrix.hpp) over the B200 C ABI.

Same names, argument meaning and error behaviour as the reference:

  reference (C++)                                 here
  ----------------------------------------------  ---------------------------------------------
  IdResult optim_id(const Matrix&, k)   id.hpp:40  optim_id(a, k)
  (sketch RID composed from the reference API)   sketch_rid(a, k, p, seed, omega_mode, omega)
  IdResult id_auto(a, k, method, seed, frac)      id_auto(a, k, method, seed, p=...)
  PivotedQr qr_column_pivoted(a, steps) qr.hpp:34 qr_column_pivoted(a, steps)
  Matrix select_columns(a, cols)    matrix.hpp:76 select_columns(a, cols)
  std::invalid_argument                           InvalidArgument (a ValueError)
  SingularMatrixError / NotPositiveDefiniteError  same names

Matrices are torch CUDA fp64 tensors in column-major layout (shape (m, n),
strides (1, lda)) -- the idkit::Matrix storage contract -- or numpy arrays,
which are routed through the host-buffer entry (copies inside the call).
Results come back on the same side they went in.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib

OMEGA_PHILOX, OMEGA_MT19937, OMEGA_VERBATIM = 0, 1, 2
DETERMINISTIC, RANDOMIZED, SAMPLED = 0, 1, 2  # SAMPLED: the reference's column-sampling optim_rid


class IdkitError(RuntimeError):
    pass


class InvalidArgument(IdkitError, ValueError):
    """std::invalid_argument in the reference (id.cpp:14-18, qr.cpp:45-46)."""


class SingularMatrixError(IdkitError):
    """idkit::SingularMatrixError (errors.hpp:9-13)."""


class NotPositiveDefiniteError(IdkitError):
    """idkit::NotPositiveDefiniteError (errors.hpp:15-19)."""


class CudaError(IdkitError):
    pass


_ERRORS = {1: InvalidArgument, 2: SingularMatrixError, 3: NotPositiveDefiniteError, 4: CudaError,
           5: CudaError, 6: CudaError}


@dataclass
class IdResult:
    """id.hpp:17-22.  `approx` is not materialised (next row);
    `c` is C = A[:, cols] (rows of A when transposed)."""
    cols: object
    z: object
    c: Optional[object] = None
    transposed: bool = False


@dataclass
class PivotedQr:
    """qr.hpp:16-21."""
    q: object
    r: object
    perm: object
    steps: int


class Context:
    """One idk_handle bound to a device; one per thread (handles are not shared)."""

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        h = C.c_void_p()
        rc = self.lib.idk_create(C.byref(h), device)
        if rc != 0:
            raise CudaError(f"idk_create(device={device}) failed: {self.lib.idk_status_string(rc).decode()} "
                            "(no usable sm_100 GPU; there is no CPU fallback)")
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            self.lib.idk_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc: int):
        if rc != 0:
            msg = self.lib.idk_last_error(self.h).decode()
            raise _ERRORS.get(rc, IdkitError)(msg)

    def bind_stream(self):
        import torch
        s = torch.cuda.current_stream(self.device).cuda_stream
        self.lib.idk_set_stream(self.h, C.c_void_p(s))

    @property
    def kernel_launches(self) -> int:
        return int(self.lib.idk_kernel_launches(self.h))

    STAGES = ("prep", "sketch", "cpqr", "solve", "gather")
    CPQR_AUTO, CPQR_RESIDENT_GRID, CPQR_STREAMING, CPQR_CLUSTER_PULL = 0, 1, 2, 3

    def set_cpqr_mode(self, mode: int):
        self.check(self.lib.idk_set_cpqr_mode(self.h, mode))

    SKETCH_DMMA, SKETCH_REFERENCE_ORDER = 0, 1

    def set_sketch_order(self, order: int):
        """IDK_SKETCH_DMMA (default) or IDK_SKETCH_REFERENCE_ORDER (Y bit-identical to the
        reference's matmul, matrix.cpp:28-48; slow -- bit-compatibility checks)."""
        self.check(self.lib.idk_set_sketch_order(self.h, order))

    def set_batched_exact(self, exact: bool = True):
        self.check(self.lib.idk_set_batched_exact(self.h, 1 if exact else 0))

    def cpqr_plan(self, m: int, n: int, k: int) -> dict:
        out = (C.c_int64 * 8)()
        self.check(self.lib.idk_cpqr_plan(self.h, m, n, k, out))
        kinds = {1: "cluster", 2: "resident-grid", 3: "streaming", 4: "cluster-pull"}
        keys = ("kind", "ctas", "cols_per_cta", "threads_per_col", "reg_rows", "smem_rows", "threads", "smem")
        d = dict(zip(keys, list(out)))
        d["kind"] = kinds[d["kind"]]
        return d

    def set_profiling(self, enable: bool = True):
        self.check(self.lib.idk_set_profiling(self.h, 1 if enable else 0))

    def stage_times(self) -> dict:
        buf = (C.c_double * 5)()
        n = self.lib.idk_stage_times(self.h, buf, 5)
        return {self.STAGES[i]: buf[i] for i in range(n)}

    # ---- multi-GPU: the handle's NCCL communicator (idk_comm_init) ----
    def comm_init(self, nranks: int, rank: int, unique_id: bytes):
        if len(unique_id) != 128:
            raise InvalidArgument("an ncclUniqueId is 128 bytes")
        buf = C.create_string_buffer(unique_id, 128)
        self.check(self.lib.idk_comm_init(self.h, nranks, rank, buf))
        self.nranks, self.rank = nranks, rank

    # idk_host_collectives callbacks: allgather(ctx, send, recv, bytes), broadcast(ctx, buf, bytes, root), barrier(ctx)
    _AG = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64)
    _BC = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int)
    _BR = C.CFUNCTYPE(C.c_int, C.c_void_p)

    class _HostColl(C.Structure):
        _fields_ = [("ctx", C.c_void_p), ("allgather", C.c_void_p), ("broadcast", C.c_void_p), ("barrier", C.c_void_p)]

    def set_host_collectives(self, nranks: int, rank: int, allgather, broadcast, barrier):
        """A caller transport instead of NCCL (idk_set_host_collectives): Python
        callables over host buffers -- allgather(send_addr, recv_addr, nbytes),
        broadcast(buf_addr, nbytes, root), barrier(); raise to fail."""
        def wrap(fn):
            def cb(*args):
                try:
                    fn(*args[1:])
                    return 0
                except Exception:  # noqa: BLE001 -- reported to the library as a failed collective
                    return 1
            return cb
        self._hc_refs = (self._AG(wrap(allgather)), self._BC(wrap(broadcast)), self._BR(wrap(barrier)))
        st = self._HostColl(None, C.cast(self._hc_refs[0], C.c_void_p), C.cast(self._hc_refs[1], C.c_void_p),
                            C.cast(self._hc_refs[2], C.c_void_p))
        self._hc_struct = st
        self.check(self.lib.idk_set_host_collectives(self.h, nranks, rank, C.byref(st)))
        self.nranks, self.rank = nranks, rank

    def comm_destroy(self):
        self.check(self.lib.idk_comm_destroy(self.h))
        self.nranks, self.rank = 1, 0


_tls = threading.local()


def context(device: int = 0) -> Context:
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


# ---- layout helpers -----------------------------------------------------------

def is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def fortran(t):
    """Column-major view/copy of a 2-D fp64 CUDA tensor: strides (1, ld)."""
    import torch
    if t.dtype != torch.float64:
        raise InvalidArgument("matrices are fp64 (idkit::Matrix stores double)")
    if t.dim() != 2:
        raise InvalidArgument("expected a 2-D matrix")
    if (t.stride(0) == 1 or t.shape[0] <= 1) and (t.shape[1] <= 1 or t.stride(1) >= max(1, t.shape[0])):
        return t
    return t.t().contiguous().t()


def empty_f(m: int, n: int, device):
    import torch
    return torch.empty((n, m), dtype=torch.float64, device=device).t()


def _ld(t) -> int:
    # a single column has no meaningful column stride (torch may report 1)
    return max(int(t.stride(1)), 1) if t.shape[1] > 1 else max(int(t.shape[0]), 1)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


# ---- the ID path ----------------------------------------------------------------

def optim_id(a, k: int, want_c: bool = True) -> IdResult:
    """Deterministic ID (id.hpp:40).  Z in the interpolation form [I | R11^-1 R12] P^T."""
    import torch
    if not is_torch(a):
        r = optim_id(torch.from_numpy(np.asfortranarray(a, dtype=np.float64)).cuda(), k, want_c)
        return IdResult(r.cols.cpu().numpy(), r.z.cpu().numpy(), None if r.c is None else r.c.cpu().numpy(), False)
    a = fortran(a)
    m, n = a.shape
    ctx = context(a.device.index or 0)
    ctx.bind_stream()
    cols = torch.empty(max(k, 0), dtype=torch.int64, device=a.device)
    z = empty_f(max(k, 0), n, a.device)
    c = empty_f(m, max(k, 0), a.device) if want_c else None
    ctx.check(ctx.lib.idk_optim_id(ctx.h, _ptr(a), m, n, _ld(a), k, _ptr(cols), _ptr(z), _ptr(c)))
    return IdResult(cols, z, c, False)


def sketch_rid(a, k: int, p: int, seed: int = 0, omega_mode: int = OMEGA_PHILOX, omega=None,
               transposed: bool = False, want_c: bool = True) -> IdResult:
    """Gaussian-sketch RID.  `a` is M (m x n) or, with transposed=True, the stored
    n x m matrix whose transpose is decomposed (id_auto dual without A^T)."""
    import torch
    a = fortran(a)
    if transposed:
        n, m = a.shape
    else:
        m, n = a.shape
    ctx = context(a.device.index or 0)
    ctx.bind_stream()
    om = fortran(omega) if omega is not None else None
    if omega_mode == OMEGA_VERBATIM and (om is None or om.shape != (k + p, m) or _ld(om) != k + p):
        raise InvalidArgument("verbatim omega must be a packed (k+p) x m fp64 CUDA matrix")
    cols = torch.empty(max(k, 0), dtype=torch.int64, device=a.device)
    z = empty_f(max(k, 0), n, a.device)
    c = empty_f(m, max(k, 0), a.device) if want_c else None
    ctx.check(ctx.lib.idk_sketch_rid(ctx.h, _ptr(a), m, n, _ld(a), 1 if transposed else 0, k, p, seed,
                                     omega_mode, _ptr(om), _ptr(cols), _ptr(z), _ptr(c)))
    return IdResult(cols, z, c, transposed)


def optim_rid(a, k: int, oversampling_fraction: float = 0.2, seed: int = 0, transposed: bool = False,
              want_c: bool = True) -> IdResult:
    """The reference's randomized ID (id.hpp:47-50, id.cpp:47-76): column sampling
    (mt19937_64, bit-identical sample) -> CPQR of A[:, S] -> Bunch-Kaufman solve
    of (R_k^T R_k) Z = C^T A.  Singular sample -> SingularMatrixError."""
    import torch
    if not is_torch(a):
        r = optim_rid(torch.from_numpy(np.asfortranarray(a, dtype=np.float64)).cuda(), k, oversampling_fraction,
                      seed, transposed, want_c)
        return IdResult(r.cols.cpu().numpy(), r.z.cpu().numpy(), None if r.c is None else r.c.cpu().numpy(),
                        transposed)
    a = fortran(a)
    n, m = a.shape if transposed else a.shape[::-1]
    ctx = context(a.device.index or 0)
    ctx.bind_stream()
    cols = torch.empty(max(k, 0), dtype=torch.int64, device=a.device)
    z = empty_f(max(k, 0), n, a.device)
    c = empty_f(m, max(k, 0), a.device) if want_c else None
    ctx.check(ctx.lib.idk_optim_rid(ctx.h, _ptr(a), m, n, _ld(a), 1 if transposed else 0, k,
                                    float(oversampling_fraction), seed, _ptr(cols), _ptr(z), _ptr(c)))
    return IdResult(cols, z, c, transposed)


def _sampled_extra(k: int, frac: float) -> int:
    if not frac >= 0.0:
        raise InvalidArgument("optim_rid: oversampling_fraction must be non-negative")
    return int(float(frac) * float(k))  # size_t(fraction * k), id.cpp:54


def id_auto(a, k: int, method: int = DETERMINISTIC, seed: int = 0, p: int = 0,
            omega_mode: int = OMEGA_PHILOX, want_c: bool = True, oversampling_fraction: float = None) -> IdResult:
    """id.hpp:55-56: tall inputs (m > n) are decomposed through their transpose.
    `p` is the sketch oversampling (rows of Omega = k + p) for method=RANDOMIZED;
    method=SAMPLED runs the reference's optim_rid with `oversampling_fraction`
    (default 0.2, id.hpp:56)."""
    if method == SAMPLED:
        p = _sampled_extra(k, 0.2 if oversampling_fraction is None else oversampling_fraction)
    m, n = a.shape
    tall = m > n
    zc = m if tall else n
    crow = n if tall else m
    if is_torch(a):
        import torch
        a = fortran(a)
        ctx = context(a.device.index or 0)
        ctx.bind_stream()
        cols = torch.empty(max(k, 0), dtype=torch.int64, device=a.device)
        z = empty_f(max(k, 0), zc, a.device)
        c = empty_f(crow, max(k, 0), a.device) if want_c else None
        tr = C.c_int(0)
        ctx.check(ctx.lib.idk_id_auto(ctx.h, _ptr(a), m, n, _ld(a), k, method, seed, p, omega_mode, None,
                                      _ptr(cols), _ptr(z), _ptr(c), C.byref(tr)))
        return IdResult(cols, z, c, bool(tr.value))
    a = np.asfortranarray(a, dtype=np.float64)
    ctx = context(0)
    cols = np.empty(max(k, 0), dtype=np.int64)
    z = np.empty((max(k, 0), zc), order="F")
    c = np.empty((crow, max(k, 0)), order="F") if want_c else None
    tr = C.c_int(0)
    ctx.check(ctx.lib.idk_id_auto_host(ctx.h, a.ctypes.data_as(C.c_void_p), m, n, k, method, seed, p, omega_mode,
                                       cols.ctypes.data_as(C.c_void_p), z.ctypes.data_as(C.c_void_p),
                                       c.ctypes.data_as(C.c_void_p) if c is not None else None, C.byref(tr)))
    return IdResult(cols, z, c, bool(tr.value))


def id_auto_many(mats, k: int, method: int = DETERMINISTIC, seed: int = 0, p: int = 0,
                 omega_mode: int = OMEGA_PHILOX, want_c: bool = True, out=None):
    """Pipelined host entry: IDs of several host matrices (same shape); uploads,
    compute and downloads overlap on separate streams.  Pass pinned, column-major
    numpy arrays for asynchronous copies.  `out` (optional) = preallocated
    (cols, z, c) lists to write into.  Returns (cols list, z list, c list, transposed)."""
    mats = [np.asfortranarray(x, dtype=np.float64) for x in mats]
    cnt = len(mats)
    m, n = mats[0].shape
    if any(x.shape != (m, n) for x in mats):
        raise InvalidArgument("id_auto_many: all matrices must have the same shape")
    tall = m > n
    zc, crow = (m, n) if tall else (n, m)
    if out is None:
        cols = [np.empty(k, dtype=np.int64) for _ in range(cnt)]
        zs = [np.empty((k, zc), order="F") for _ in range(cnt)]
        cs = [np.empty((crow, k), order="F") for _ in range(cnt)] if want_c else None
    else:
        cols, zs, cs = out
    P = C.c_void_p * max(cnt, 1)
    pa = P(*[x.ctypes.data for x in mats])
    pcol = P(*[x.ctypes.data for x in cols])
    pz = P(*[x.ctypes.data for x in zs])
    pc = P(*[x.ctypes.data for x in cs]) if cs is not None else None
    ctx = context(0)
    ctx.bind_stream()
    tr = C.c_int(0)
    ctx.check(ctx.lib.idk_id_auto_host_many(ctx.h, cnt, pa, m, n, k, method, seed, p, omega_mode, pcol, pz, pc,
                                            C.byref(tr)))
    return cols, zs, cs, bool(tr.value)


def id_auto_batch(mats, k: int, method: int = DETERMINISTIC, seeds=None, p: int = 0,
                  omega_mode: int = OMEGA_PHILOX, want_c: bool = True, out=None, lanes: int = None):
    """Concurrent device entry (idk_id_auto_batch): IDs of several same-shape
    fp64 CUDA matrices, spread over `lanes` streams so one ID's CPQR overlaps
    the others' GEMMs.  `seeds`: one per matrix (default 0).  `p`: sketch
    oversampling (RANDOMIZED) or extra sampled columns floor(fraction*k)
    (SAMPLED), as in the C ABI.  `out` (optional) =
    preallocated (cols, z, c) lists.  Returns (cols, z, c, transposed)."""
    import torch
    mats = [fortran(x) for x in mats]
    cnt = len(mats)
    m, n = mats[0].shape
    if any(tuple(x.shape) != (m, n) or _ld(x) != _ld(mats[0]) for x in mats):
        raise InvalidArgument("id_auto_batch: all matrices must have the same shape and leading dimension")
    tall = m > n
    zc, crow = (m, n) if tall else (n, m)
    dev = mats[0].device
    if out is None:
        cols = [torch.empty(k, dtype=torch.int64, device=dev) for _ in range(cnt)]
        zs = [empty_f(k, zc, dev) for _ in range(cnt)]
        cs = [empty_f(crow, k, dev) for _ in range(cnt)] if want_c else None
    else:
        cols, zs, cs = out
    P = C.c_void_p * max(cnt, 1)
    ctx = context(dev.index or 0)
    ctx.bind_stream()
    if lanes is not None:
        ctx.check(ctx.lib.idk_set_concurrency(ctx.h, lanes))
    sd = (C.c_uint64 * max(cnt, 1))(*(list(seeds) if seeds is not None else [0] * cnt))
    tr = C.c_int(0)
    ctx.check(ctx.lib.idk_id_auto_batch(ctx.h, cnt, P(*[x.data_ptr() for x in mats]), m, n, _ld(mats[0]), k, method,
                                        sd, p, omega_mode, P(*[x.data_ptr() for x in cols]),
                                        P(*[x.data_ptr() for x in zs]),
                                        P(*[x.data_ptr() for x in cs]) if cs is not None else None, C.byref(tr)))
    return cols, zs, cs, bool(tr.value)


def matmul_ref(a, b):
    """idkit::matmul (matrix.cpp:28-48) on the device in the reference's exact
    arithmetic (summation order, zero skipping, no FMA): bit-identical to the
    CPU reference.  a, b: fp64 CUDA matrices."""
    a, b = fortran(a), fortran(b)
    m, k = a.shape
    if b.shape[0] != k:
        raise InvalidArgument(f"matmul: inner dimensions disagree ({k} vs {b.shape[0]})")
    n = b.shape[1]
    c = empty_f(m, n, a.device)
    ctx = context(a.device.index or 0)
    ctx.bind_stream()
    ctx.check(ctx.lib.idk_matmul_ref(ctx.h, _ptr(a), m, k, _ld(a), _ptr(b), n, _ld(b), _ptr(c), max(m, 1)))
    return c


def optim_id_batched(a, k: int, want_c: bool = True):
    """BASELINE cfg3: `a` is a (batch, n, m) contiguous CUDA tensor holding
    batch column-major m x n matrices (i.e. a[b].t() is matrix b).
    Returns cols (batch, k), z (batch, n, k) [= Z_b^T row-major], c (batch, k, m).
    A numpy array (or CPU tensor) of the same layout runs through the pipelined
    host entry (idk_optim_id_batched_host) and returns numpy arrays."""
    import torch
    if not is_torch(a) or a.device.type == "cpu":
        import numpy as np
        ah = a.numpy() if is_torch(a) else np.asarray(a)
        if ah.ndim != 3 or ah.dtype != np.float64:
            raise InvalidArgument("batched input must be a (batch, n, m) fp64 array")
        ah = np.ascontiguousarray(ah)
        batch, n, m = ah.shape
        ctx = context(0)
        cols = np.empty((batch, max(k, 0)), dtype=np.int64)
        z = np.empty((batch, n, max(k, 0)), dtype=np.float64)
        c = np.empty((batch, max(k, 0), m), dtype=np.float64) if want_c else None
        ctx.check(ctx.lib.idk_optim_id_batched_host(ctx.h, ah.ctypes.data, batch, m, n, k, cols.ctypes.data,
                                                    z.ctypes.data, c.ctypes.data if want_c else None))
        return cols, z, c
    if a.dim() != 3 or not a.is_contiguous() or a.dtype != torch.float64:
        raise InvalidArgument("batched input must be a contiguous (batch, n, m) fp64 tensor")
    batch, n, m = a.shape
    ctx = context(a.device.index or 0)
    ctx.bind_stream()
    cols = torch.empty((batch, max(k, 0)), dtype=torch.int64, device=a.device)
    z = torch.empty((batch, n, max(k, 0)), dtype=torch.float64, device=a.device)
    c = torch.empty((batch, max(k, 0), m), dtype=torch.float64, device=a.device) if want_c else None
    ctx.check(ctx.lib.idk_optim_id_batched(ctx.h, _ptr(a), batch, m, n, m, m * n, k, _ptr(cols), _ptr(z),
                                           _ptr(c)))
    return cols, z, c


def id_from_sketch(y, k: int, c_begin: int = 0, c_end: Optional[int] = None):
    """Factor an (all-gathered) sketch Y in place and solve Z for columns
    [c_begin, c_end).  Returns (cols, z_local)."""
    import torch
    y = fortran(y)
    l, n = y.shape
    c_end = n if c_end is None else c_end
    ctx = context(y.device.index or 0)
    ctx.bind_stream()
    cols = torch.empty(max(k, 0), dtype=torch.int64, device=y.device)
    z = empty_f(max(k, 0), max(c_end - c_begin, 0), y.device)
    ctx.check(ctx.lib.idk_id_from_sketch(ctx.h, _ptr(y), l, n, _ld(y), k, c_begin, c_end, _ptr(cols),
                                         _ptr(z) if c_end > c_begin else None))
    return cols, z


def approx(r: IdResult):
    """IdResult::approx (id.hpp:17-22) on the device: C Z, or (C Z)^T for the dual."""
    import torch
    c, z = fortran(r.c), fortran(r.z)
    mr, k = c.shape
    n = z.shape[1]
    ctx = context(c.device.index or 0)
    ctx.bind_stream()
    out = empty_f(mr, n, c.device)
    ctx.check(ctx.lib.idk_approx(ctx.h, _ptr(c), mr, k, _ptr(z), n, _ptr(out), mr))
    return out.t() if r.transposed else out


def diagnostics(a, r: IdResult) -> dict:
    """idkit::diagnostics (id.hpp:60): relative error, max |Z|, identity
    deviation, |Z| <= 2 flag -- on the device, approx never materialised."""
    a = fortran(a)
    m, n = a.shape
    z = fortran(r.z)
    cols = r.cols.contiguous()
    k = cols.numel()
    ctx = context(a.device.index or 0)
    ctx.bind_stream()
    out = (C.c_double * 4)()
    cptr = _ptr(fortran(r.c)) if r.c is not None else None
    ctx.check(ctx.lib.idk_diagnostics(ctx.h, _ptr(a), m, n, _ld(a), 1 if r.transposed else 0, _ptr(cols), k,
                                      _ptr(z), cptr, out))
    return {"relative_error": out[0], "max_abs_z": out[1], "identity_deviation": out[2],
            "entry_bound_satisfied": bool(out[3])}


# ---- multi-GPU (C ABI: idk_shard_range / idk_comm_init / idk_id_sharded) ------------

def shard_range(n: int, nranks: int, rank: int):
    """Columns [begin, end) of an n-column matrix owned by `rank` (ceil-sized blocks)."""
    lib = _lib.load()
    b, e = C.c_int64(), C.c_int64()
    if lib.idk_shard_range(n, nranks, rank, C.byref(b), C.byref(e)) != 0:
        raise InvalidArgument("shard_range: bad arguments")
    return b.value, e.value


def nccl_unique_id() -> bytes:
    lib = _lib.load()
    buf = C.create_string_buffer(128)
    rc = lib.idk_nccl_unique_id(buf)
    if rc != 0:
        raise CudaError("idk_nccl_unique_id failed (libnccl.so.2 not loadable?)")
    return buf.raw


def id_sharded(a_local, m: int, n: int, k: int, p: int, seed: int = 0, transposed: bool = False,
               omega_mode: int = OMEGA_PHILOX, omega=None, want_c: bool = True):
    """Column-sharded sketch RID through the C ABI (idk_id_sharded) on this
    rank's context (comm_init first for more than one rank).  a_local: this
    rank's columns of M (m x n_r), or with transposed=True the stored row block
    (n_r x m) of the tall A.  Returns (cols, z_local (k x n_r), c (m x k))."""
    import torch
    dev = a_local.device
    ctx = context(dev.index or 0)
    ctx.bind_stream()
    a_local = fortran(a_local)
    nranks, rank = getattr(ctx, "nranks", 1), getattr(ctx, "rank", 0)
    b, e = shard_range(n, nranks, rank)
    nr = e - b
    if (a_local.shape[0] if transposed else a_local.shape[1]) != nr:
        raise InvalidArgument(f"rank {rank}: local block has the wrong width (expected {nr} columns of M)")
    om = fortran(omega) if omega is not None else None
    cols = torch.empty(max(k, 0), dtype=torch.int64, device=dev)
    z = empty_f(max(k, 0), nr, dev)
    c = empty_f(m, max(k, 0), dev) if want_c else None
    ctx.check(ctx.lib.idk_id_sharded(ctx.h, _ptr(a_local) if nr > 0 else None, m, n, _ld(a_local) if nr > 0 else 1,
                                     1 if transposed else 0, k, p, seed, omega_mode, _ptr(om), _ptr(cols),
                                     _ptr(z) if nr > 0 else None, _ptr(c)))
    return cols, z, c


# ---- stages / primitives ----------------------------------------------------------

def sketch_omega(l: int, m: int, seed: int, device=0):
    import torch
    ctx = context(device)
    ctx.bind_stream()
    om = empty_f(l, m, torch.device("cuda", device))
    ctx.check(ctx.lib.idk_sketch_omega(ctx.h, l, m, seed, _ptr(om)))
    return om


def sketch(omega, a, transposed: bool = False):
    """Y = Omega * M (matrix.cpp:28-48 on the DMMA pipe)."""
    omega = fortran(omega)
    a = fortran(a)
    l, m = omega.shape
    n = a.shape[0] if transposed else a.shape[1]
    ctx = context(a.device.index or 0)
    ctx.bind_stream()
    y = empty_f(l, n, a.device)
    ctx.check(ctx.lib.idk_sketch(ctx.h, _ptr(omega), l, _ptr(a), m, n, _ld(a), 1 if transposed else 0, _ptr(y), l))
    return y


def qr_column_pivoted(a, steps: int, want_q: bool = True) -> PivotedQr:
    """qr.hpp:34."""
    import torch
    a = fortran(a)
    m, n = a.shape
    ctx = context(a.device.index or 0)
    ctx.bind_stream()
    q = empty_f(m, max(steps, 0), a.device) if want_q else None
    r = empty_f(max(steps, 0), n, a.device)
    perm = torch.empty(n, dtype=torch.int64, device=a.device)
    ctx.check(ctx.lib.idk_qr_column_pivoted(ctx.h, _ptr(a), m, n, _ld(a), steps, _ptr(q), _ptr(r), _ptr(perm)))
    return PivotedQr(q, r, perm, steps)


def select_columns(a, cols, rows_of_a: bool = False):
    """matrix.hpp:76 (rows_of_a: the dual's row gather)."""
    import torch
    a = fortran(a)
    m, n = a.shape
    cols = torch.as_tensor(cols, dtype=torch.int64, device=a.device).contiguous()
    ctx = context(a.device.index or 0)
    ctx.bind_stream()
    out = empty_f(n if rows_of_a else m, cols.numel(), a.device)
    ctx.check(ctx.lib.idk_select_columns(ctx.h, _ptr(a), m, n, _ld(a), _ptr(cols), cols.numel(),
                                         1 if rows_of_a else 0, _ptr(out)))
    return out

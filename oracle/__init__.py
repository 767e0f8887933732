"""TEST INFRASTRUCTURE ONLY -- ctypes front-ends for the parity checkers.

* ``Oracle``   -> oracle/liboracle.so, our C restatement of the reference path
                  (idk_oracle.c; every function cites the reference file:line).
* ``Reference`` -> oracle/_ref/libidkit_ref.so, the unmodified reference sources
                  compiled in place by oracle/Makefile (only where
                  /root/reference exists; the .so then travels with the repo).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this package.  The product package
``paper_2105_07076_b200`` never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/proj"

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    pass


class InvalidArgument(OracleError, ValueError):
    pass


class SingularMatrixError(OracleError):
    pass


class NotPositiveDefiniteError(OracleError):
    pass


_CODES = {1: InvalidArgument, 2: SingularMatrixError, 3: NotPositiveDefiniteError}


def build(ref: bool = True, dropin: bool = False) -> None:
    """Compile liboracle.so (and oracle/_ref when the reference is present;
    `dropin` adds the reference's acceptance suite on both libraries)."""
    targets = ["all"]
    if ref and os.path.isdir(REF_SRC):
        targets.append("ref")
        if dropin:
            targets.append("dropin")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _f64(a):
    return np.asfortranarray(a, dtype=np.float64)


def _ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(C.c_void_p)


class _Lib:
    prefix = ""
    err_fn = ""

    def __init__(self, path):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle{' ref' if 'ref' in path else ''}`")
        self.lib = C.CDLL(path)
        getattr(self.lib, self.err_fn).restype = C.c_char_p

    def _check(self, rc):
        if rc != 0:
            msg = getattr(self.lib, self.err_fn)().decode()
            raise _CODES.get(rc, OracleError)(msg)


class Oracle(_Lib):
    """Our CPU restatement (liboracle.so)."""

    err_fn = "idko_last_error"

    def __init__(self, path=None):
        super().__init__(path or os.path.join(HERE, "liboracle.so"))
        L = self.lib
        L.idko_mix_seed.restype = C.c_uint64
        L.idko_mix_seed.argtypes = [C.c_uint64, C.c_char_p]

    def mix_seed(self, base, label):
        return int(self.lib.idko_mix_seed(C.c_uint64(base), label.encode()))

    def generate(self, kind, rows, cols, seed):
        out = np.empty((rows, cols), order="F")
        self._check(self.lib.idko_generate(C.c_int(kind), C.c_int64(rows), C.c_int64(cols),
                                           C.c_uint64(seed), _ptr(out)))
        return out

    def gaussian_matrix(self, m, n, seed):
        return self.generate(1, m, n, seed)

    def omega_philox(self, l, m, seed):
        out = np.empty((l, m), order="F")
        self.lib.idko_omega_philox(C.c_int64(l), C.c_int64(m), C.c_uint64(seed), _ptr(out))
        return out

    def sample_without_replacement(self, population, count, seed):
        out = np.empty(count, dtype=np.int64)
        self._check(self.lib.idko_sample_without_replacement(C.c_int64(population), C.c_int64(count),
                                                             C.c_uint64(seed), _ptr(out)))
        return out

    def matmul(self, a, b):
        a, b = _f64(a), _f64(b)
        out = np.empty((a.shape[0], b.shape[1]), order="F")
        self.lib.idko_matmul(_ptr(a), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]), _ptr(b),
                             C.c_int64(b.shape[1]), _ptr(out))
        return out

    def qr_column_pivoted(self, a, steps, want_q=True):
        a = _f64(a)
        m, n = a.shape
        q = np.empty((m, steps), order="F") if want_q else None
        r = np.empty((steps, n), order="F")
        perm = np.empty(n, dtype=np.int64)
        taus = np.empty(max(steps, 1))
        self._check(self.lib.idko_qr_column_pivoted(_ptr(a), C.c_int64(m), C.c_int64(n),
                                                    C.c_int64(steps), _ptr(q), _ptr(r), _ptr(perm),
                                                    _ptr(taus), None))
        return q, r, perm

    def solve_triangular(self, t, b, upper=True):
        t = _f64(t)
        x = np.array(b, dtype=np.float64, order="F", copy=True)
        self._check(self.lib.idko_solve_triangular(_ptr(t), C.c_int64(t.shape[0]), _ptr(x),
                                                   C.c_int64(x.shape[1]), C.c_int(1 if upper else 0)))
        return x

    def solve_posdef(self, s, b):
        s = _f64(s)
        x = np.array(b, dtype=np.float64, order="F", copy=True)
        self._check(self.lib.idko_solve_posdef(_ptr(s), C.c_int64(s.shape[0]), _ptr(x),
                                               C.c_int64(x.shape[1])))
        return x

    def solve_symmetric_indefinite(self, s, b):
        s = _f64(s)
        x = np.array(b, dtype=np.float64, order="F", copy=True)
        self._check(self.lib.idko_solve_symmetric_indefinite(_ptr(s), C.c_int64(s.shape[0]), _ptr(x),
                                                             C.c_int64(x.shape[1])))
        return x

    def optim_id(self, a, k, want_approx=True):
        a = _f64(a)
        m, n = a.shape
        cols = np.empty(k, dtype=np.int64)
        z = np.empty((k, n), order="F")
        approx = np.empty((m, n), order="F") if want_approx else None
        self._check(self.lib.idko_optim_id(_ptr(a), C.c_int64(m), C.c_int64(n), C.c_int64(k),
                                           _ptr(cols), _ptr(z), _ptr(approx)))
        return cols, z, approx

    def optim_rid(self, a, k, frac, seed, want_approx=True):
        a = _f64(a)
        m, n = a.shape
        cols = np.empty(k, dtype=np.int64)
        z = np.empty((k, n), order="F")
        approx = np.empty((m, n), order="F") if want_approx else None
        self._check(self.lib.idko_optim_rid(_ptr(a), C.c_int64(m), C.c_int64(n), C.c_int64(k),
                                            C.c_double(frac), C.c_uint64(seed), _ptr(cols), _ptr(z),
                                            _ptr(approx)))
        return cols, z, approx

    def interp_decomp(self, a, k, omega=None, want_c=True, want_approx=False):
        """North-star ID: optional sketch, CPQR, TRSM form of Z, gather."""
        a = _f64(a)
        m, n = a.shape
        om = _f64(omega) if omega is not None else None
        l = om.shape[0] if om is not None else 0
        cols = np.empty(k, dtype=np.int64)
        z = np.empty((k, n), order="F")
        c = np.empty((m, k), order="F") if want_c else None
        approx = np.empty((m, n), order="F") if want_approx else None
        self._check(self.lib.idko_interp_decomp(_ptr(a), C.c_int64(m), C.c_int64(n), C.c_int64(k),
                                                _ptr(om), C.c_int64(l), _ptr(cols), _ptr(z), _ptr(c),
                                                _ptr(approx)))
        return cols, z, c, approx

    def id_auto(self, a, k, method, seed=0, frac=0.2, p=0, omega_mode=0, want_approx=True):
        a = _f64(a)
        m, n = a.shape
        cols = np.empty(k, dtype=np.int64)
        z = np.empty((k, max(m, n)), order="F")
        approx = np.empty((m, n), order="F") if want_approx else None
        tr = C.c_int(0)
        self._check(self.lib.idko_id_auto(_ptr(a), C.c_int64(m), C.c_int64(n), C.c_int64(k),
                                          C.c_int(method), C.c_uint64(seed), C.c_double(frac),
                                          C.c_int64(p), C.c_int(omega_mode), _ptr(cols), _ptr(z),
                                          _ptr(approx), C.byref(tr)))
        zc = m if tr.value else n
        return cols, np.asfortranarray(z[:, :zc]), approx, bool(tr.value)

    def diagnostics(self, a, cols, z, approx):
        a, z, approx = _f64(a), _f64(z), _f64(approx)
        cols = np.ascontiguousarray(cols, dtype=np.int64)
        out = np.empty(4)
        self._check(self.lib.idko_diagnostics(_ptr(a), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]),
                                              _ptr(cols), C.c_int64(len(cols)), _ptr(z),
                                              C.c_int64(z.shape[1]), _ptr(approx), _ptr(out)))
        return {"relative_error": out[0], "max_abs_z": out[1], "identity_deviation": out[2],
                "entry_bound_satisfied": bool(out[3])}


class Reference(_Lib):
    """The reference library itself (oracle/_ref/libidkit_ref.so)."""

    err_fn = "ref_last_error"

    def __init__(self, path=None):
        super().__init__(path or os.path.join(HERE, "_ref", "libidkit_ref.so"))
        self.lib.ref_mix_seed.restype = C.c_uint64
        self.lib.ref_mix_seed.argtypes = [C.c_uint64, C.c_char_p]

    @staticmethod
    def available(path=None):
        return os.path.exists(path or os.path.join(HERE, "_ref", "libidkit_ref.so"))

    def mix_seed(self, base, label):
        return int(self.lib.ref_mix_seed(C.c_uint64(base), label.encode()))

    def generate(self, kind, rows, cols, seed):
        out = np.empty((rows, cols), order="F")
        self._check(self.lib.ref_generate(C.c_int(kind), C.c_int64(rows), C.c_int64(cols),
                                          C.c_uint64(seed), _ptr(out)))
        return out

    def gaussian_matrix(self, m, n, seed):
        out = np.empty((m, n), order="F")
        self._check(self.lib.ref_gaussian_matrix(C.c_int64(m), C.c_int64(n), C.c_uint64(seed), _ptr(out)))
        return out

    def sample_without_replacement(self, population, count, seed):
        out = np.empty(count, dtype=np.int64)
        self._check(self.lib.ref_sample_without_replacement(C.c_int64(population), C.c_int64(count),
                                                            C.c_uint64(seed), _ptr(out)))
        return out

    def matmul(self, a, b):
        a, b = _f64(a), _f64(b)
        out = np.empty((a.shape[0], b.shape[1]), order="F")
        self._check(self.lib.ref_matmul(_ptr(a), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]), _ptr(b),
                                        C.c_int64(b.shape[1]), _ptr(out)))
        return out

    def qr_column_pivoted(self, a, steps):
        a = _f64(a)
        m, n = a.shape
        q = np.empty((m, steps), order="F")
        r = np.empty((steps, n), order="F")
        perm = np.empty(n, dtype=np.int64)
        self._check(self.lib.ref_qr_column_pivoted(_ptr(a), C.c_int64(m), C.c_int64(n), C.c_int64(steps),
                                                   _ptr(q), _ptr(r), _ptr(perm)))
        return q, r, perm

    def solve_triangular(self, t, b, upper=True):
        t, b = _f64(t), _f64(b)
        x = np.empty_like(b, order="F")
        self._check(self.lib.ref_solve_triangular(_ptr(t), C.c_int64(t.shape[0]), _ptr(b),
                                                  C.c_int64(b.shape[1]), C.c_int(1 if upper else 0), _ptr(x)))
        return x

    def solve_posdef(self, s, b):
        s, b = _f64(s), _f64(b)
        x = np.empty_like(b, order="F")
        self._check(self.lib.ref_solve_posdef(_ptr(s), C.c_int64(s.shape[0]), _ptr(b),
                                              C.c_int64(b.shape[1]), _ptr(x)))
        return x

    def solve_symmetric_indefinite(self, s, b):
        s, b = _f64(s), _f64(b)
        x = np.empty_like(b, order="F")
        self._check(self.lib.ref_solve_symmetric_indefinite(_ptr(s), C.c_int64(s.shape[0]), _ptr(b),
                                                            C.c_int64(b.shape[1]), _ptr(x)))
        return x

    def optim_id(self, a, k):
        a = _f64(a)
        m, n = a.shape
        cols = np.empty(k, dtype=np.int64)
        z = np.empty((k, n), order="F")
        approx = np.empty((m, n), order="F")
        self._check(self.lib.ref_optim_id(_ptr(a), C.c_int64(m), C.c_int64(n), C.c_int64(k), _ptr(cols),
                                          _ptr(z), _ptr(approx)))
        return cols, z, approx

    def optim_rid(self, a, k, frac, seed):
        a = _f64(a)
        m, n = a.shape
        cols = np.empty(k, dtype=np.int64)
        z = np.empty((k, n), order="F")
        approx = np.empty((m, n), order="F")
        self._check(self.lib.ref_optim_rid(_ptr(a), C.c_int64(m), C.c_int64(n), C.c_int64(k),
                                           C.c_double(frac), C.c_uint64(seed), _ptr(cols), _ptr(z),
                                           _ptr(approx)))
        return cols, z, approx

    def id_auto(self, a, k, randomized, seed=0, frac=0.2):
        a = _f64(a)
        m, n = a.shape
        cols = np.empty(k, dtype=np.int64)
        z = np.empty((k, max(m, n)), order="F")
        approx = np.empty((m, n), order="F")
        tr = C.c_int(0)
        self._check(self.lib.ref_id_auto(_ptr(a), C.c_int64(m), C.c_int64(n), C.c_int64(k),
                                         C.c_int(1 if randomized else 0), C.c_uint64(seed), C.c_double(frac),
                                         _ptr(cols), _ptr(z), _ptr(approx), C.byref(tr)))
        zc = m if tr.value else n
        return cols, np.asfortranarray(z[:, :zc]), approx, bool(tr.value)

    def sketch_id(self, a, k, omega=None, want_c=True):
        a = _f64(a)
        m, n = a.shape
        om = _f64(omega) if omega is not None else None
        l = om.shape[0] if om is not None else 0
        cols = np.empty(k, dtype=np.int64)
        z = np.empty((k, n), order="F")
        c = np.empty((m, k), order="F") if want_c else None
        self._check(self.lib.ref_sketch_id(_ptr(a), C.c_int64(m), C.c_int64(n), C.c_int64(k), _ptr(om),
                                           C.c_int64(l), _ptr(cols), _ptr(z), _ptr(c)))
        return cols, z, c

    def sketch_id_mt(self, a, k, omega=None, l=None, seed=0, transposed=False, threads=None, want_c=True):
        """sketch_id on `threads` host threads (bit-identical to one thread: see
        ref_sketch_id_mt).  `a` is the stored matrix (column-major, any ld);
        transposed=True decomposes M = a^T (id_auto's dual).  omega=None ->
        the reference's generate(gaussian, l, m, seed) inside the timed region.
        Returns (cols, z, c, times) with times = {omega, matmul, qr, solve, select} s."""
        if not (a.flags["F_CONTIGUOUS"] and a.dtype == np.float64):
            a = _f64(a)
        lda = a.shape[0]
        m, n = (a.shape[1], a.shape[0]) if transposed else a.shape
        om = _f64(omega) if omega is not None else None
        ll = om.shape[0] if om is not None else int(l)
        threads = threads or (len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count())
        cols = np.empty(k, dtype=np.int64)
        z = np.empty((k, n), order="F")
        c = np.empty((m, k), order="F") if want_c else None
        t5 = np.zeros(5)
        self._check(self.lib.ref_sketch_id_mt(_ptr(a), C.c_int64(lda), C.c_int64(m), C.c_int64(n),
                                              C.c_int(1 if transposed else 0), C.c_int64(k), _ptr(om),
                                              C.c_int64(ll), C.c_uint64(seed), C.c_int(int(threads)), _ptr(cols),
                                              _ptr(z), _ptr(c), _ptr(t5)))
        names = ("omega", "matmul", "qr", "solve", "select")
        return cols, z, c, dict(zip(names, t5.tolist()))

    def optim_id_batch_mt(self, a, k, threads=None, want_approx=False):
        """optim_id over a (batch, n, m) stack (matrix b column-major = a[b].T) on threads."""
        a = np.ascontiguousarray(a, dtype=np.float64)
        batch, n, m = a.shape
        threads = threads or (len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count())
        cols = np.empty((batch, k), dtype=np.int64)
        z = np.empty((batch, n, k))  # z[b] = Z_b^T storage: Z_b (k x n) column-major
        approx = np.empty_like(a) if want_approx else None
        self._check(self.lib.ref_optim_id_batch_mt(_ptr(a), C.c_int64(batch), C.c_int64(m), C.c_int64(n),
                                                   C.c_int64(k), C.c_int(int(threads)), _ptr(cols), _ptr(z),
                                                   _ptr(approx)))
        return cols, z, approx

    def gram_schmidt_pivoted(self, a, steps):
        a = _f64(a)
        order = np.empty(steps, dtype=np.int64)
        norms = np.empty(steps)
        self._check(self.lib.ref_gram_schmidt_pivoted(_ptr(a), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]),
                                                      C.c_int64(steps), _ptr(order), _ptr(norms)))
        return order, norms

    def truncated_svd_error(self, a, k):
        a = _f64(a)
        out = C.c_double(0)
        self._check(self.lib.ref_truncated_svd_error(_ptr(a), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]),
                                                     C.c_int64(k), C.byref(out)))
        return out.value

    def diagnostics(self, a, cols, z, approx):
        a, z, approx = _f64(a), _f64(z), _f64(approx)
        cols = np.ascontiguousarray(cols, dtype=np.int64)
        out = np.empty(4)
        self._check(self.lib.ref_diagnostics(_ptr(a), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]),
                                             _ptr(cols), C.c_int64(len(cols)), _ptr(z), C.c_int64(z.shape[1]),
                                             _ptr(approx), _ptr(out)))
        return {"relative_error": out[0], "max_abs_z": out[1], "identity_deviation": out[2],
                "entry_bound_satisfied": bool(out[3])}

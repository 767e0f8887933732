"""TEST INFRASTRUCTURE: oracle-backed stand-ins for sharded.CudaStages, so the
multi-rank host logic (partitioning, all_gather of Y, local Z range, C
all-reduce) runs under gloo on CPU.  The product never uses these."""
import numpy as np
import torch

from oracle import Oracle


def _f(t):
    return np.asfortranarray(t.numpy())


def _t(a):
    a = np.asfortranarray(a)
    return torch.from_numpy(np.ascontiguousarray(a.T)).t()


class OracleStages:
    def __init__(self):
        self.o = Oracle()

    def omega(self, l, m, seed, like):
        return _t(self.o.omega_philox(l, m, seed))

    def sketch(self, omega, a_local, transposed):
        a = _f(a_local)
        mm = np.asfortranarray(a.T) if transposed else a
        return _t(self.o.matmul(_f(omega), mm))

    def factor(self, y, k, c_begin, c_end):
        cols, z, _, _ = self.o.interp_decomp(_f(y), k, None, want_c=False)
        return torch.from_numpy(cols), _t(z[:, c_begin:c_end])

    def gather(self, a_local, idx, rows_of_a):
        a = _f(a_local)
        idx = idx.numpy()
        return _t(a[idx, :].T if rows_of_a else a[:, idx])

    def batched(self, a_local, k):
        cols, zs, cs = [], [], []
        for b in range(a_local.shape[0]):
            ab = np.asfortranarray(a_local[b].numpy().T)
            c_, z_, cc, _ = self.o.interp_decomp(ab, k)
            cols.append(c_)
            zs.append(z_.T)
            cs.append(cc.T)
        return torch.from_numpy(np.stack(cols)), torch.from_numpy(np.stack(zs)), torch.from_numpy(np.stack(cs))

"""Synthetic inputs for the five BASELINE.json configurations.

No dataset is involved: BASELINE's configs are synthetic constructions, built
here from seeded generators (numpy on the host for tests, torch on the GPU for
the 2 GiB configs).  Shapes, spectra and distributions follow BASELINE.json;
SURVEY.md 8(d) lists them.  cfg3's "N(0, 1e-8)" noise is read as variance
1e-8 (standard deviation 1e-4); see DESIGN.md.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    m: int
    n: int
    k: int
    p: int            # sketch oversampling; -1 = deterministic ID (no sketch)
    batch: int = 1
    sharded: bool = False

    @property
    def randomized(self) -> bool:
        return self.p >= 0

    @property
    def l(self) -> int:  # noqa: E743 -- the survey's notation for k + p
        return self.k + max(self.p, 0)


CONFIGS = {
    "cfg1": Config("cfg1", 500, 1000, 50, -1),
    "cfg2": Config("cfg2", 2000, 4000, 100, 10),
    "cfg3": Config("cfg3", 64, 256, 16, -1, batch=4096, sharded=True),
    "cfg4": Config("cfg4", 16384, 16384, 256, 16, sharded=True),
    "cfg5": Config("cfg5", 65536, 4096, 64, 8, sharded=True),
}


def spectrum(name: str, r: int) -> np.ndarray:
    i = np.arange(r, dtype=np.float64)
    if name == "cfg1":
        return 10.0 ** (-i / 25.0)
    if name == "cfg2":
        return np.exp(-i / 30.0)
    if name == "cfg4":
        s = np.ones(r)
        t = i >= 128
        s[t] = (i[t] - 127.0) ** -2.0
        return s
    raise ValueError(name)


def _orthonormal(rng: np.random.Generator, m: int, r: int) -> np.ndarray:
    q, _ = np.linalg.qr(rng.standard_normal((m, r)))
    return q


def svd_matrix_np(name: str, m: int, n: int, seed: int) -> np.ndarray:
    """A = U diag(sigma) V^T with Gaussian-QR orthonormal U (m x r), V (n x r), r = min(m, n)."""
    rng = np.random.default_rng(seed)
    r = min(m, n)
    u = _orthonormal(rng, m, r)
    v = _orthonormal(rng, n, r)
    return np.asfortranarray((u * spectrum(name, r)) @ v.T)


def low_rank_batch_np(batch: int, m: int, n: int, rank: int, noise_std: float, seed: int) -> np.ndarray:
    """cfg3: batch x (G1 (m x rank) G2 (rank x n) + N(0, noise_std^2)); returns (batch, n, m):
    element [b, j, i] = A_b(i, j) (each matrix column-major)."""
    rng = np.random.default_rng(seed)
    g1 = rng.standard_normal((batch, m, rank))
    g2 = rng.standard_normal((batch, rank, n))
    a = g1 @ g2 + noise_std * rng.standard_normal((batch, m, n))
    return np.ascontiguousarray(np.transpose(a, (0, 2, 1)))


def nonneg_low_rank_np(m: int, n: int, rank: int, noise: float, seed: int) -> np.ndarray:
    """cfg5: W (m x rank) H (rank x n), U[0,1] entries, + U[0, noise]."""
    rng = np.random.default_rng(seed)
    w = rng.random((m, rank))
    h = rng.random((rank, n))
    return np.asfortranarray(w @ h + noise * rng.random((m, n)))


def make_np(name: str, seed: int = 20260601, scale: float = 1.0):
    """Host construction of a config (optionally shrunk by `scale` for tests)."""
    c = CONFIGS[name]
    if name in ("cfg1", "cfg2", "cfg4"):
        m, n = max(int(c.m * scale), c.l + 1), max(int(c.n * scale), c.l + 1)
        return svd_matrix_np(name, m, n, seed)
    if name == "cfg3":
        return low_rank_batch_np(max(int(c.batch * scale), 1), c.m, c.n, 16, 1e-4, seed)
    if name == "cfg5":
        return nonneg_low_rank_np(max(int(c.m * scale), 2 * c.n), max(int(c.n * scale), c.l + 1), 64, 1e-6, seed)
    raise ValueError(name)


# ---- device construction (bench: the 2 GiB configs) ------------------------------

def make_torch(name: str, seed: int = 20260601, device: str = "cuda"):
    """Same constructions with torch on the GPU (harness only, not the measured path).
    Returns a column-major (m, n) fp64 CUDA tensor, or (batch, n, m) for cfg3."""
    import torch
    c = CONFIGS[name]
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    dt = torch.float64
    if name in ("cfg1", "cfg2", "cfg4"):
        r = min(c.m, c.n)
        u, _ = torch.linalg.qr(torch.randn((c.m, r), generator=g, device=device, dtype=dt))
        v, _ = torch.linalg.qr(torch.randn((c.n, r), generator=g, device=device, dtype=dt))
        s = torch.from_numpy(spectrum(name, r)).to(device)
        a = (u * s) @ v.t()
        del u, v
        return a.t().contiguous().t()
    if name == "cfg3":
        g1 = torch.randn((c.batch, c.m, 16), generator=g, device=device, dtype=dt)
        g2 = torch.randn((c.batch, 16, c.n), generator=g, device=device, dtype=dt)
        a = g1 @ g2 + 1e-4 * torch.randn((c.batch, c.m, c.n), generator=g, device=device, dtype=dt)
        return a.transpose(1, 2).contiguous()
    if name == "cfg5":
        w = torch.rand((c.m, 64), generator=g, device=device, dtype=dt)
        h = torch.rand((64, c.n), generator=g, device=device, dtype=dt)
        a = torch.addmm(1e-6 * torch.rand((c.m, c.n), generator=g, device=device, dtype=dt), w, h)
        return a.t().contiguous().t()
    raise ValueError(name)

"""TEST INFRASTRUCTURE: a near-exactly rounded sketch Y = Omega M on the GPU,
independent of both the reference's sequential sum and our DMMA sum.

Error-free splitting (Ozaki scheme in fp64): every row of Omega and every
column of M is scaled by a power of two and cut into S slices of BETA bits, so
each slice entry is an integer multiple of 2^-(BETA*(t+1)) below 2^-(BETA*t).
With 2*BETA + log2(K) <= 53 every slice product Omega_s M_u is computed
EXACTLY by any fp64 GEMM (all partial sums are representable), here
torch.matmul (cuBLAS, test-only checker).  The S^2 exact products are then
summed smallest first, so Y is within a couple of ulps of the exact product
(the slices keep S*BETA = 76 bits below each row/column maximum).

Used to tell which of two fp64 solutions (ours, the reference's) is closer
to the exact one when they differ at the conditioning limit (cfg4).
"""
import torch

S = 4


def _split(x, dim, beta):
    """x = scale * sum_t slices[t]; scale per row (dim=1) or column (dim=0)."""
    amax = x.abs().amax(dim=dim, keepdim=True)
    e = torch.where(amax > 0, torch.floor(torch.log2(amax)) + 1, torch.zeros_like(amax))
    scale = torch.pow(2.0, e)
    r = x / scale  # exact: power-of-two scaling, |r| < 1
    slices = []
    for t in range(S):
        f = 2.0 ** (beta * (t + 1))
        q = torch.trunc(r * f) / f  # exact
        slices.append(q)
        r = r - q  # exact
    return scale, slices


def accurate_sketch(omega, m_mat):
    """omega (l x K), m_mat (K x n) fp64 CUDA tensors -> Y (l x n), ~1-2 ulp accurate."""
    K = omega.shape[1]
    beta = (53 - (K - 1).bit_length()) // 2
    so, os_ = _split(omega, 1, beta)
    sm, ms = _split(m_mat, 0, beta)
    y = torch.zeros((omega.shape[0], m_mat.shape[1]), dtype=torch.float64, device=omega.device)
    terms = sorted(((s, u) for s in range(S) for u in range(S)), key=lambda su: -(su[0] + su[1]))
    for s, u in terms:  # smallest products first
        y += os_[s] @ ms[u]
        if y.is_cuda:
            torch.cuda.synchronize()
    del os_, ms
    return (y * so) * sm

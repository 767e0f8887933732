// tsqr.cu -- R factor of a tall-skinny matrix for optim_rid's pivoted QR.
//
// optim_rid (id.cpp:47-76) factors the sampled columns A_S (m x p, m >> p)
// with qr_column_pivoted (qr.cpp:42-126).  Pivoted QR of A_S and of any R0 with
// A_S = Q0 R0 (Q0 orthonormal) pick the same pivots and produce the same R up
// to row signs in exact arithmetic, so for tall samples the pivoted QR runs on
// the p x p factor R0 instead of the m x p matrix (the on-chip kernels then fit
// a single cluster).  R0 comes from shifted CholeskyQR3 (Fukaya et al.,
// "Shifted Cholesky QR for computing the QR factorization of ill-conditioned
// matrices", SIAM J. Sci. Comput. 42 (2020)): a shifted Cholesky QR step
// followed by two plain ones; every Gram matrix is a DMMA GEMM, the p x p
// Choleskys and the triangular solves run here.  It is backward stable for
// condition numbers up to ~1e15.
#include <climits>

#include "common.cuh"

namespace idk {

namespace {

constexpr int kCholThreads = 512;

// G (p x p, ld p, column-major, symmetric) + shift*I -> lower Cholesky factor
// L written into Lf (p x p, ld p; entries above the diagonal zeroed).  Packed
// by columns in shared memory when it fits, else in place in Lf (L2).
// *status = index of the first non-positive pivot (untouched on success).
__global__ void __launch_bounds__(kCholThreads)
cholesky_kernel(const double* __restrict__ G, int p, const double* __restrict__ trace, double shift_factor,
                double* __restrict__ Lf, int* __restrict__ status, int switch_at) {
    extern __shared__ double sm[];
    const double shift = trace ? shift_factor * *trace : 0.0;
    const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = T >> 5;
    // the working triangle starts in Lf (L2) and moves on chip, packed by
    // columns, once the trailing part fits (switch_at = 0: from the start)
    int s0 = INT_MAX;
    auto colp = [&](int j) -> double* {
        if (j >= s0) {
            const int jj = j - s0, nn = p - s0;
            return sm + (jj * nn - jj * (jj - 1) / 2 - jj - s0);
        }
        return Lf + static_cast<int64_t>(j) * p;
    };
    for (int j = wid; j < p; j += nw) {
        double* cj = colp(j);
        for (int i = j + lane; i < p; i += 32)
            cj[i] = 0.5 * (G[static_cast<int64_t>(j) * p + i] + G[static_cast<int64_t>(i) * p + j]) + (i == j ? shift : 0.0);
    }
    __syncthreads();
    for (int kk = 0; kk < p; ++kk) {
        if (s0 == INT_MAX && kk >= switch_at) {
            const int nn = p - kk;
            for (int j = kk + wid; j < p; j += nw) {
                const int jj = j - kk;
                double* dst = sm + (jj * nn - jj * (jj - 1) / 2 - jj - kk);
                const double* src = Lf + static_cast<int64_t>(j) * p;
                for (int i = j + lane; i < p; i += 32) dst[i] = src[i];
            }
            __syncthreads();
            s0 = kk;
        }
        double* ck = colp(kk);
        const double d = ck[kk];
        if (!(d > 0.0)) {
            if (tid == 0) *status = kk;
            return;
        }
        const double r = sqrt(d);
        const double inv = 1.0 / r, invd = 1.0 / d;
        // a(i,j) -= a(i,kk) a(j,kk) / d for kk < j <= i (right-looking, a warp per column)
        for (int j = kk + 1 + wid; j < p; j += nw) {
            double* cj = colp(j);
            const double w = ck[j] * invd;
#pragma unroll 4
            for (int i = j + lane; i < p; i += 32) cj[i] = fma(-ck[i], w, cj[i]);
        }
        __syncthreads();
        for (int i = kk + 1 + tid; i < p; i += T) ck[i] *= inv;
        if (tid == 0) ck[kk] = r;
        // column kk is final; the next step reads only columns > kk
    }
    __syncthreads();
    for (int j = wid; j < p; j += nw) {
        const double* cj = colp(j);
        for (int i = lane; i < p; i += 32) {
            const double v = i >= j ? cj[i] : 0.0;
            Lf[static_cast<int64_t>(j) * p + i] = v;
        }
    }
}

// X (p x n, ld p) <- L^-1 X for lower-triangular L (p x p, ld p): forward
// substitution per column, a warp per kRhs columns held in shared memory, L
// staged packed in shared memory when it fits.
constexpr int kRhs = 4;

template <bool kPacked>
__global__ void __launch_bounds__(256)
trsv_lower_many_kernel(const double* __restrict__ L, int p, int64_t n, double* __restrict__ X) {
    extern __shared__ double sm[];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, W = blockDim.x >> 5;
    double* xs = sm;                                         // W * kRhs * p
    double* Lp = xs + static_cast<size_t>(W) * kRhs * p;     // p(p+1)/2 when packed
    auto cstart = [&](int j) { return j * p - j * (j - 1) / 2; };
    if constexpr (kPacked) {
        for (int j = wid; j < p; j += W) {
            const int c0j = cstart(j);
            for (int i = j + lane; i < p; i += 32) Lp[c0j + i - j] = L[static_cast<int64_t>(j) * p + i];
        }
        __syncthreads();
    }
    auto Lc = [&](int j) -> const double* {
        if constexpr (kPacked) return Lp + cstart(j) - j;
        else return L + static_cast<int64_t>(j) * p;
    };
    const int64_t c0 = (static_cast<int64_t>(blockIdx.x) * W + wid) * kRhs;
    if (c0 >= n) return;
    const int nc = static_cast<int>(min(static_cast<int64_t>(kRhs), n - c0));
    double* x = xs + static_cast<size_t>(wid) * kRhs * p;
    for (int c = 0; c < kRhs; ++c)
        for (int i = lane; i < p; i += 32) x[c * p + i] = c < nc ? X[(c0 + c) * p + i] : 0.0;
    __syncwarp();
    for (int j = 0; j < p; ++j) {
        const double* lj = Lc(j);
        const double dj = lj[j];
        double y[kRhs];
#pragma unroll
        for (int c = 0; c < kRhs; ++c) y[c] = x[c * p + j] / dj;
        __syncwarp();
        if (lane < kRhs) x[lane * p + j] = y[lane == 0 ? 0 : lane == 1 ? 1 : lane == 2 ? 2 : 3];
        for (int i = j + 1 + lane; i < p; i += 32) {
            const double l = lj[i];
#pragma unroll
            for (int c = 0; c < kRhs; ++c) x[c * p + i] = fma(-l, y[c], x[c * p + i]);
        }
        __syncwarp();
    }
    for (int c = 0; c < nc; ++c)
        for (int i = lane; i < p; i += 32) X[(c0 + c) * p + i] = x[c * p + i];
}

// Frobenius-norm-squared of the columns: trace(G) -> *out (one CTA, fixed
// order); *zero_col = 1 if a column is exactly zero (G_ii == 0).
__global__ void trace_kernel(const double* __restrict__ G, int p, double* __restrict__ out, int* __restrict__ zero_col) {
    __shared__ double part[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < p; i += blockDim.x) {
        const double g = G[static_cast<int64_t>(i) * p + i];
        if (g == 0.0) *zero_col = 1;
        s += g;
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.0;
        t = warp_sum(t);
        if (threadIdx.x == 0) *out = t;
    }
}

}  // namespace

size_t cholesky_smem_bytes(int p) { return sizeof(double) * static_cast<size_t>(p) * (p + 1) / 2; }

cudaError_t cholesky_lower(const double* G, int p, const double* trace, double shift_factor, double* L, int* status,
                           cudaStream_t stream) {
    const size_t cap = 220 * 1024;
    int s0 = 0;
    while (s0 < p && sizeof(double) * static_cast<size_t>(p - s0) * (p - s0 + 1) / 2 > cap) ++s0;
    const size_t smem = std::max<size_t>(sizeof(double) * static_cast<size_t>(p - s0) * (p - s0 + 1) / 2, 1024);
    cudaError_t e = cudaFuncSetAttribute(cholesky_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    cholesky_kernel<<<1, kCholThreads, smem, stream>>>(G, p, trace, shift_factor, L, status, s0);
    return cudaGetLastError();
}

cudaError_t trsv_lower_many(const double* L, int p, int64_t n, double* X, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    const size_t cap = 220 * 1024;
    const size_t lbytes = sizeof(double) * static_cast<size_t>(p) * (p + 1) / 2;
    auto xbytes = [&](int W) { return sizeof(double) * static_cast<size_t>(W) * kRhs * p; };
    int W = 8;
    bool packed = true;
    while (W > 1 && xbytes(W) + lbytes > cap) W >>= 1;
    if (W < 4 || xbytes(W) + lbytes > cap) {  // staging L for one or two warps does not pay: read it from L2
        packed = false;
        W = 8;
        while (W > 1 && xbytes(W) > cap) W >>= 1;
    }
    const size_t smem = xbytes(W) + (packed ? lbytes : 0);
    const int64_t per = static_cast<int64_t>(W) * kRhs;
    const unsigned grid = static_cast<unsigned>((n + per - 1) / per);
    void (*fn)(const double*, int, int64_t, double*) = packed ? trsv_lower_many_kernel<true> : trsv_lower_many_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    fn<<<grid, 32 * W, smem, stream>>>(L, p, n, X);
    return cudaGetLastError();
}

cudaError_t gram_trace(const double* G, int p, double* out, int* zero_col, cudaStream_t stream) {
    trace_kernel<<<1, 256, 0, stream>>>(G, p, out, zero_col);
    return cudaGetLastError();
}

}  // namespace idk

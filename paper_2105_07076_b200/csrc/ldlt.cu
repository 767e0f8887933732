// ldlt.cu -- symmetric-indefinite solve for optim_rid's Z (id.cpp:65-72).
//
// Reference: solve_symmetric_indefinite (solve.cpp:262-274): symmetrise the
// k x k Gram matrix R_k^T R_k, Bunch-Kaufman LDL^T with 1x1 / 2x2 pivots
// (alpha = (1+sqrt(17))/8, ldlt_bunch_kaufman solve.cpp:106-193), then the
// block solve replaying the interchanges (ldlt_solve solve.cpp:200-258) for
// the n right-hand sides C^T A.
//
// The factorisation is O(k^3) on a k <= 256 matrix: one CTA, the matrix in
// shared memory when it fits (k <= 160) or in global memory (L2) otherwise,
// pivot search by block reduction, the trailing update spread over the CTA.
// The solve is O(k^2 n): each warp owns kLC right-hand sides in shared memory
// and walks the pivot blocks forward, through D, and backward.
#include <climits>

#include "common.cuh"

namespace idk {

namespace {

constexpr int kLdltThreads = 512;
constexpr int kLC = 4;  // right-hand sides per warp in the solve

struct Blk {
    int start, size, swap;
};

// One CTA.  S (k x k, column-major, ld k) -> symmetrised, factored (lower
// triangle: L below the pivot blocks, D on them) into F.  Every access of the
// reference's algorithm is to the lower triangle, so in shared memory the
// matrix is stored packed by columns (k(k+1)/2 doubles: k <= 234 fits); for
// larger k the first steps work on F in L2 until the trailing triangle fits.  blocks/nblk out; *status = index of a
// singular pivot block (left untouched on success).
//
// One __syncthreads per 1x1 step: the warp that updates the next pivot column
// also reduces its column max (first index among equals, solve.cpp:115-125),
// every thread takes the pivot decision redundantly, and the scaling of the
// finished column needs no barrier (no later step reads it).
__device__ __forceinline__ void warp_argmax_first(double& v, int& idx) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (ov > v || (ov == v && oi < idx)) {
            v = ov;
            idx = oi;
        }
    }
}

// Storage: the working lower triangle starts in F (L2); once the trailing
// triangle from the current step on fits in shared memory (`switch_at`, 0 when
// the whole matrix fits) it is moved there, packed by columns, and the
// remaining steps run on chip.  Every step touches only columns >= its own.
__global__ void __launch_bounds__(kLdltThreads)
ldlt_bk_kernel(const double* __restrict__ S, int k, double* __restrict__ F, Blk* __restrict__ blocks,
               int* __restrict__ nblk, int* __restrict__ status, int switch_at) {
    extern __shared__ double sm[];
    __shared__ double sv[32];
    __shared__ double s_cm[2];  // max |a(i, kk)|, i > kk, of the next pivot column (by step parity)
    __shared__ int s_ci[2];
    const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = T >> 5;
    if (tid == 0) *nblk = 0;  // a failed factorisation leaves the solve a no-op
    int s0 = INT_MAX;  // first column held in shared memory (after the switch)
    // column j from row 0 (entries i >= j valid)
    auto colp = [&](int j) -> double* {
        if (j >= s0) {
            const int jj = j - s0, nn = k - s0;
            return sm + (jj * nn - jj * (jj - 1) / 2 - jj - s0);
        }
        return F + static_cast<int64_t>(j) * k;
    };
    auto move_on_chip = [&](int from) {  // columns >= from: F -> shared memory
        const int nn = k - from;
        for (int j = from + wid; j < k; j += nw) {
            const int jj = j - from;
            double* dst = sm + (jj * nn - jj * (jj - 1) / 2 - jj - from);
            const double* src = F + static_cast<int64_t>(j) * k;
            for (int i = j + lane; i < k; i += 32) dst[i] = src[i];
        }
        __syncthreads();
        s0 = from;
    };
    // (i, j) with i >= j
    auto at = [&](int i, int j) -> double& { return colp(j)[i]; };
    // symmetrise (solve.cpp:268-270), lower triangle only
    for (int j = wid; j < k; j += nw)
        for (int i = j + lane; i < k; i += 32)
            at(i, j) = 0.5 * (S[static_cast<int64_t>(j) * k + i] + S[static_cast<int64_t>(i) * k + j]);
    __syncthreads();
    if (wid == 0) {
        double v = -1.0;
        int idx = INT_MAX;
        for (int i = 1 + lane; i < k; i += 32) {
            const double x = fabs(at(i, 0));
            if (x > v) {
                v = x;
                idx = i;
            }
        }
        warp_argmax_first(v, idx);
        if (lane == 0) {
            s_cm[0] = v;
            s_ci[0] = idx;
        }
    }
    __syncthreads();
    const double alpha = (1.0 + sqrt(17.0)) / 8.0;
    int kk = 0, nb = 0, par = 0;
    while (kk < k) {
        if (s0 == INT_MAX && kk >= switch_at) move_on_chip(kk);
        double colmax = s_cm[par];
        int imax = s_ci[par];
        if (colmax < 0.0) {
            colmax = 0.0;
            imax = kk;
        }
        const double absakk = fabs(at(kk, kk));
        if (fmax(absakk, colmax) == 0.0) {
            if (tid == 0) *status = kk;
            return;
        }
        int kstep = 1, kp = kk;
        if (absakk < alpha * colmax) {
            // row max of row imax (solve.cpp:133-136)
            double rv = 0.0;
            for (int j = kk + tid; j < imax; j += T) rv = fmax(rv, fabs(at(imax, j)));
            for (int i = imax + 1 + tid; i < k; i += T) rv = fmax(rv, fabs(at(i, imax)));
            rv = warp_max(rv);
            if (lane == 0) sv[wid] = rv;
            __syncthreads();
            const double rowmax = warp_max(lane < nw ? sv[lane] : 0.0);
            if (absakk >= alpha * colmax * (colmax / rowmax)) {
                kp = kk;
            } else if (fabs(at(imax, imax)) >= alpha * rowmax) {
                kp = imax;
            } else {
                kp = imax;
                kstep = 2;
            }
        }
        const int kq = kk + kstep - 1;
        if (kp != kq) {  // swap_symmetric_lower(a, kq, kp) (solve.cpp:97-104)
            for (int i = kp + 1 + tid; i < k; i += T) {
                const double t = at(i, kq);
                at(i, kq) = at(i, kp);
                at(i, kp) = t;
            }
            for (int j = kq + 1 + tid; j < kp; j += T) {
                const double t = at(j, kq);
                at(j, kq) = at(kp, j);
                at(kp, j) = t;
            }
            if (tid == 0) {
                double t = at(kq, kq);
                at(kq, kq) = at(kp, kp);
                at(kp, kp) = t;
                if (kstep == 2) {
                    t = at(kq, kk);
                    at(kq, kk) = at(kp, kk);
                    at(kp, kk) = t;
                }
            }
            __syncthreads();
        }
        const int nxt = kk + kstep;  // next pivot column: updated by warp 0, which also reduces its max
        if (kstep == 1) {
            const double d = at(kk, kk);
            if (d == 0.0) {
                if (tid == 0) *status = kk;
                return;
            }
            const double inv = 1.0 / d;
            // a(i,j) -= a(i,kk) * (a(j,kk) * inv), kk < j <= i (solve.cpp:158-162): a warp per column
            const double* ck = colp(kk);
            for (int j = nxt + wid; j < k; j += nw) {
                const double w = ck[j] * inv;
                double* cj = colp(j);
                double v = -1.0;
                int idx = INT_MAX;
#pragma unroll 4
                for (int i = j + lane; i < k; i += 32) {
                    const double y = cj[i] - ck[i] * w;
                    cj[i] = y;
                    if (j == nxt && i > j && fabs(y) > v) {
                        v = fabs(y);
                        idx = i;
                    }
                }
                if (j == nxt) {
                    warp_argmax_first(v, idx);
                    if (lane == 0) {
                        s_cm[par ^ 1] = v;
                        s_ci[par ^ 1] = idx;
                    }
                }
            }
            __syncthreads();
            double* ckw = colp(kk);
            for (int i = kk + 1 + tid; i < k; i += T) ckw[i] *= inv;  // column kk is final; no reader
        } else {
            const double d21 = at(kk + 1, kk);
            const double d11 = at(kk + 1, kk + 1) / d21;
            const double d22 = at(kk, kk) / d21;
            const double det = d11 * d22 - 1.0;
            if (d21 == 0.0 || det == 0.0) {
                if (tid == 0) *status = kk;
                return;
            }
            const double t = 1.0 / det / d21;
            // w = t (d11 a(j,k) - a(j,k+1)), w1 = t (d22 a(j,k+1) - a(j,k)) (solve.cpp:177-184)
            const double* ck = colp(kk);
            const double* ck1 = colp(kk + 1);
            for (int j = nxt + wid; j < k; j += nw) {
                const double wk = t * (d11 * ck[j] - ck1[j]);
                const double wk1 = t * (d22 * ck1[j] - ck[j]);
                double* cj = colp(j);
                double v = -1.0;
                int idx = INT_MAX;
#pragma unroll 4
                for (int i = j + lane; i < k; i += 32) {
                    const double y = cj[i] - (ck[i] * wk + ck1[i] * wk1);
                    cj[i] = y;
                    if (j == nxt && i > j && fabs(y) > v) {
                        v = fabs(y);
                        idx = i;
                    }
                }
                if (j == nxt) {
                    warp_argmax_first(v, idx);
                    if (lane == 0) {
                        s_cm[par ^ 1] = v;
                        s_ci[par ^ 1] = idx;
                    }
                }
            }
            __syncthreads();
            for (int j = nxt + tid; j < k; j += T) {  // columns kk, kk+1 are final; no reader
                const double wk = t * (d11 * at(j, kk) - at(j, kk + 1));
                const double wk1 = t * (d22 * at(j, kk + 1) - at(j, kk));
                at(j, kk) = wk;
                at(j, kk + 1) = wk1;
            }
        }
        if (tid == 0) {
            blocks[nb].start = kk;
            blocks[nb].size = kstep;
            blocks[nb].swap = kp;
        }
        ++nb;
        kk = nxt;
        par ^= 1;
    }
    __syncthreads();
    if (s0 != INT_MAX)
        for (int j = s0 + wid; j < k; j += nw)
            for (int i = j + lane; i < k; i += 32) F[static_cast<int64_t>(j) * k + i] = at(i, j);
    if (tid == 0) *nblk = nb;
}

// ldlt_solve (solve.cpp:200-258) for n right-hand sides (k x n, ld k), in
// place.  Warp w owns kLC columns held in shared memory and updates them
// together (one L load feeds kLC FMAs); the CTA first stages L's lower
// triangle packed in shared memory when it fits (kPacked), else L is read from
// L2.
template <bool kPacked>
__global__ void __launch_bounds__(256)
ldlt_solve_kernel(const double* __restrict__ F, const Blk* __restrict__ blocks_g, const int* __restrict__ nblk_p,
                  int k, int64_t n, double* __restrict__ B) {
    extern __shared__ double sm[];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, W = blockDim.x >> 5;
    const int nb = *nblk_p;
    double* xs = sm;                                                     // W * kLC * k
    double* Lp = xs + static_cast<size_t>(W) * kLC * k;                  // k(k+1)/2 when packed
    Blk* blk = reinterpret_cast<Blk*>(Lp + (kPacked ? static_cast<size_t>(k) * (k + 1) / 2 : 0));
    auto cstart = [&](int j) { return j * k - j * (j - 1) / 2; };
    if constexpr (kPacked) {
        for (int j = wid; j < k; j += W) {
            const int c0j = cstart(j);
            for (int i = j + lane; i < k; i += 32) Lp[c0j + i - j] = F[static_cast<int64_t>(j) * k + i];
        }
    }
    for (int b = tid; b < nb; b += blockDim.x) blk[b] = blocks_g[b];
    __syncthreads();
    // column j of L from row i on: Lc(j)[i]
    auto Lc = [&](int j) -> const double* {
        if constexpr (kPacked) return Lp + cstart(j) - j;
        else return F + static_cast<int64_t>(j) * k;
    };
    const int64_t c0 = (static_cast<int64_t>(blockIdx.x) * W + wid) * kLC;
    if (c0 >= n) return;
    const int nc = static_cast<int>(min(static_cast<int64_t>(kLC), n - c0));
    double* x = xs + static_cast<size_t>(wid) * kLC * k;  // x[c*k + i]
    for (int c = 0; c < kLC; ++c)
        for (int i = lane; i < k; i += 32) x[c * k + i] = c < nc ? B[(c0 + c) * k + i] : 0.0;
    __syncwarp();
    // forward: interchange, then eliminate below the block
    for (int b = 0; b < nb; ++b) {
        const Blk bl = blk[b];
        const int kk = bl.start, r = kk + bl.size - 1;
        if (bl.swap != r && lane < kLC) {
            const double t = x[lane * k + r];
            x[lane * k + r] = x[lane * k + bl.swap];
            x[lane * k + bl.swap] = t;
        }
        __syncwarp();
        double b0[kLC], b1[kLC];
#pragma unroll
        for (int c = 0; c < kLC; ++c) {
            b0[c] = x[c * k + kk];
            b1[c] = bl.size == 2 ? x[c * k + kk + 1] : 0.0;
        }
        const double* l0 = Lc(kk);
        if (bl.size == 1) {
            for (int i = kk + 1 + lane; i < k; i += 32) {
                const double l = l0[i];
#pragma unroll
                for (int c = 0; c < kLC; ++c) x[c * k + i] -= l * b0[c];
            }
        } else {
            const double* l1 = Lc(kk + 1);
            for (int i = kk + 2 + lane; i < k; i += 32) {
                const double la = l0[i], lb = l1[i];
#pragma unroll
                for (int c = 0; c < kLC; ++c) x[c * k + i] -= la * b0[c] + lb * b1[c];
            }
        }
        __syncwarp();
    }
    // block diagonal
    if (lane < kLC) {
        double* xc = x + lane * k;
        for (int b = 0; b < nb; ++b) {
            const Blk bl = blk[b];
            const int kk = bl.start;
            const double* l0 = Lc(kk);
            if (bl.size == 1) {
                xc[kk] /= l0[kk];
            } else {
                const double* l1 = Lc(kk + 1);
                const double akm1k = l0[kk + 1];
                const double akm1 = l0[kk] / akm1k;
                const double ak = l1[kk + 1] / akm1k;
                const double denom = akm1 * ak - 1.0;
                const double bkm1 = xc[kk] / akm1k;
                const double bk = xc[kk + 1] / akm1k;
                xc[kk] = (ak * bkm1 - bk) / denom;
                xc[kk + 1] = (akm1 * bk - bkm1) / denom;
            }
        }
    }
    __syncwarp();
    // backward: x_c -= sum_{i >= below} L(i, c) x_i, then undo the interchange
    for (int b = nb - 1; b >= 0; --b) {
        const Blk bl = blk[b];
        const int kk = bl.start, below = kk + bl.size;
        for (int cc = kk; cc < below; ++cc) {
            const double* lc = Lc(cc);
            double acc[kLC];
#pragma unroll
            for (int c = 0; c < kLC; ++c) acc[c] = 0.0;
            for (int i = below + lane; i < k; i += 32) {
                const double l = lc[i];
#pragma unroll
                for (int c = 0; c < kLC; ++c) acc[c] = fma(l, x[c * k + i], acc[c]);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int c = 0; c < kLC; ++c) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
            if (lane < kLC) x[lane * k + cc] -= acc[lane == 0 ? 0 : lane == 1 ? 1 : lane == 2 ? 2 : 3];
            __syncwarp();
        }
        const int r = kk + bl.size - 1;
        if (bl.swap != r && lane < kLC) {
            const double t = x[lane * k + r];
            x[lane * k + r] = x[lane * k + bl.swap];
            x[lane * k + bl.swap] = t;
        }
        __syncwarp();
    }
    for (int c = 0; c < nc; ++c)
        for (int i = lane; i < k; i += 32) B[(c0 + c) * k + i] = x[c * k + i];
}

__global__ void map_cols_kernel(const long long* __restrict__ sampled, const long long* __restrict__ piv, int k,
                                long long* __restrict__ cols) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) cols[i] = sampled[piv[i]];
}

}  // namespace

size_t ldlt_scratch_bytes(int k) { return sizeof(Blk) * static_cast<size_t>(k) + 2 * sizeof(int); }

// first step whose trailing triangle fits the shared-memory budget
static int onchip_switch(int n, size_t cap) {
    int s0 = 0;
    while (s0 < n && sizeof(double) * static_cast<size_t>(n - s0) * (n - s0 + 1) / 2 > cap) ++s0;
    return s0;
}

cudaError_t ldlt_factor(const double* S, int k, double* F, void* scratch, int* status, cudaStream_t stream) {
    Blk* blocks = static_cast<Blk*>(scratch);
    int* nblk = reinterpret_cast<int*>(blocks + k);
    const size_t cap = 220 * 1024;
    const int s0 = onchip_switch(k, cap);
    const size_t smem = sizeof(double) * static_cast<size_t>(k - s0) * (k - s0 + 1) / 2;
    cudaError_t e = cudaFuncSetAttribute(ldlt_bk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(std::max<size_t>(smem, 1024)));
    if (e != cudaSuccess) return e;
    ldlt_bk_kernel<<<1, kLdltThreads, std::max<size_t>(smem, 1024), stream>>>(S, k, F, blocks, nblk, status, s0);
    return cudaGetLastError();
}

cudaError_t ldlt_solve(const double* F, const void* scratch, int k, int64_t n, double* B, cudaStream_t stream) {
    const Blk* blocks = static_cast<const Blk*>(scratch);
    const int* nblk = reinterpret_cast<const int*>(blocks + k);
    const size_t cap = 220 * 1024;
    const size_t lbytes = sizeof(double) * static_cast<size_t>(k) * (k + 1) / 2;
    const size_t bbytes = sizeof(Blk) * static_cast<size_t>(k);
    auto xbytes = [&](int W) { return sizeof(double) * static_cast<size_t>(W) * kLC * k; };
    int W = 8;
    bool packed = true;
    while (W > 1 && xbytes(W) + lbytes + bbytes > cap) W >>= 1;
    if (xbytes(W) + lbytes + bbytes > cap) {  // L does not fit: read it from L2
        packed = false;
        W = 8;
        while (W > 1 && xbytes(W) + bbytes > cap) W >>= 1;
    }
    const size_t smem = xbytes(W) + (packed ? lbytes : 0) + bbytes;
    const int64_t per_cta = static_cast<int64_t>(W) * kLC;
    const unsigned grid = static_cast<unsigned>((n + per_cta - 1) / per_cta);
    void (*fn)(const double*, const Blk*, const int*, int, int64_t, double*) =
        packed ? ldlt_solve_kernel<true> : ldlt_solve_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    fn<<<grid, 32 * W, smem, stream>>>(F, blocks, nblk, k, n, B);
    return cudaGetLastError();
}

cudaError_t map_cols(const long long* sampled, const long long* piv, int k, long long* cols, cudaStream_t stream) {
    map_cols_kernel<<<1, 256, 0, stream>>>(sampled, piv, k, cols);
    return cudaGetLastError();
}

}  // namespace idk

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

constexpr int kLdltThreads = 1024;
constexpr int kLC = 4;  // right-hand sides per warp in the solve

struct Blk {
    int start, size, swap;
};

__device__ __forceinline__ double block_max_idx(double v, int idx, double* sv, int* si, int& out_idx) {
    // max |value| with the smallest index among equals (first strict max, like
    // the reference's `if (v > colmax)` scan)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (ov > v || (ov == v && oi < idx)) {
            v = ov;
            idx = oi;
        }
    }
    __syncthreads();
    if (lane == 0) {
        sv[wid] = v;
        si[wid] = idx;
    }
    __syncthreads();
    v = lane < nw ? sv[lane] : -1.0;
    idx = lane < nw ? si[lane] : INT_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (ov > v || (ov == v && oi < idx)) {
            v = ov;
            idx = oi;
        }
    }
    out_idx = idx;
    return v;
}

// One CTA.  S (k x k, column-major, ld k) -> symmetrised, factored in place
// (lower triangle: L below the pivot blocks, D on them).  blocks/nblk out;
// *status = index of a singular pivot block (left untouched on success).
__global__ void __launch_bounds__(kLdltThreads)
ldlt_bk_kernel(const double* __restrict__ S, int k, double* __restrict__ F, Blk* __restrict__ blocks,
               int* __restrict__ nblk, int* __restrict__ status, bool in_smem) {
    extern __shared__ double sm[];
    __shared__ double sv[32];
    __shared__ int si[32];
    __shared__ int s_dec[3];  // kstep, kp, stop
    const int tid = threadIdx.x, T = blockDim.x;
    double* a = in_smem ? sm : F;
    if (tid == 0) *nblk = 0;  // a failed factorisation leaves the solve a no-op
    auto at = [&](int i, int j) -> double& { return a[static_cast<int64_t>(j) * k + i]; };

    // symmetrise (solve.cpp:268-270)
    for (int e = tid; e < k * k; e += T) {
        const int j = e / k, i = e - j * k;
        a[e] = 0.5 * (S[e] + S[static_cast<int64_t>(i) * k + j]);
    }
    __syncthreads();
    const double alpha = (1.0 + sqrt(17.0)) / 8.0;
    int kk = 0, nb = 0;
    while (kk < k) {
        // column max below the diagonal (solve.cpp:115-125)
        double v = -1.0;
        int idx = INT_MAX;
        for (int i = kk + 1 + tid; i < k; i += T) {
            const double x = fabs(at(i, kk));
            if (x > v) {
                v = x;
                idx = i;
            }
        }
        int imax;
        double colmax = block_max_idx(v, idx, sv, si, imax);
        if (colmax < 0.0) {
            colmax = 0.0;
            imax = kk;
        }
        if (tid == 0) {
            const double absakk = fabs(at(kk, kk));
            int kstep = 1, kp = kk, stop = 0;
            if (fmax(absakk, colmax) == 0.0) {
                stop = 1;
            }
            s_dec[0] = kstep;
            s_dec[1] = kp;
            s_dec[2] = stop;
        }
        __syncthreads();
        if (s_dec[2]) {
            if (tid == 0) *status = kk;
            return;
        }
        const double absakk = fabs(at(kk, kk));
        if (absakk < alpha * colmax) {
            // row max of row imax (solve.cpp:133-136)
            double rv = 0.0;
            for (int j = kk + tid; j < imax; j += T) rv = fmax(rv, fabs(at(imax, j)));
            for (int i = imax + 1 + tid; i < k; i += T) rv = fmax(rv, fabs(at(i, imax)));
            rv = warp_max(rv);
            __syncthreads();
            if ((tid & 31) == 0) sv[tid >> 5] = rv;
            __syncthreads();
            if (tid < 32) {
                double t = tid < T / 32 ? sv[tid] : 0.0;
                t = warp_max(t);
                if (tid == 0) {
                    const double rowmax = t;
                    int kstep = 1, kp;
                    if (absakk >= alpha * colmax * (colmax / rowmax)) kp = kk;
                    else if (fabs(at(imax, imax)) >= alpha * rowmax) kp = imax;
                    else {
                        kp = imax;
                        kstep = 2;
                    }
                    s_dec[0] = kstep;
                    s_dec[1] = kp;
                }
            }
            __syncthreads();
        }
        const int kstep = s_dec[0], kp = s_dec[1];
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
        if (kstep == 1) {
            const double d = at(kk, kk);
            if (d == 0.0) {
                if (tid == 0) *status = kk;
                return;
            }
            const double inv = 1.0 / d;
            // a(i,j) -= a(i,kk) * (a(j,kk) * inv) for kk < j <= i (solve.cpp:158-162)
            const int r = k - kk - 1;
            for (int e = tid; e < r * r; e += T) {
                const int jj = e / r, ii = e - jj * r;
                if (ii >= jj) {
                    const int j = kk + 1 + jj, i = kk + 1 + ii;
                    at(i, j) -= at(i, kk) * (at(j, kk) * inv);
                }
            }
            __syncthreads();
            for (int i = kk + 1 + tid; i < k; i += T) at(i, kk) *= inv;
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
            const int r = k - kk - 2;
            // w = t * (d11 a(j,k) - a(j,k+1)), w1 = t * (d22 a(j,k+1) - a(j,k)) (solve.cpp:177-184)
            for (int e = tid; e < r * r; e += T) {
                const int jj = e / r, ii = e - jj * r;
                if (ii >= jj) {
                    const int j = kk + 2 + jj, i = kk + 2 + ii;
                    const double wk = t * (d11 * at(j, kk) - at(j, kk + 1));
                    const double wk1 = t * (d22 * at(j, kk + 1) - at(j, kk));
                    at(i, j) -= at(i, kk) * wk + at(i, kk + 1) * wk1;
                }
            }
            __syncthreads();
            for (int j = kk + 2 + tid; j < k; j += T) {
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
        kk += kstep;
        __syncthreads();
    }
    if (in_smem)
        for (int e = tid; e < k * k; e += T) F[e] = a[e];
    if (tid == 0) *nblk = nb;
}

// ldlt_solve (solve.cpp:200-258) for n right-hand sides (k x n, ld k), in
// place.  Warp w owns columns [c0, c0 + kLC) held in shared memory.
__global__ void __launch_bounds__(128)
ldlt_solve_kernel(const double* __restrict__ F, const Blk* __restrict__ blocks, const int* __restrict__ nblk_p,
                  int k, int64_t n, double* __restrict__ B) {
    extern __shared__ double sm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t c0 = (static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + wid) * kLC;
    if (c0 >= n) return;
    const int nc = static_cast<int>(min(static_cast<int64_t>(kLC), n - c0));
    double* x = sm + static_cast<size_t>(wid) * kLC * k;  // x[c*k + i]
    for (int c = 0; c < nc; ++c)
        for (int i = lane; i < k; i += 32) x[c * k + i] = B[(c0 + c) * k + i];
    __syncwarp();
    const int nb = *nblk_p;
    auto L = [&](int i, int j) { return F[static_cast<int64_t>(j) * k + i]; };
    // forward: interchange, then eliminate below the block
    for (int b = 0; b < nb; ++b) {
        const Blk blk = blocks[b];
        const int kk = blk.start, r = kk + blk.size - 1;
        if (blk.swap != r && lane < nc) {
            const double t = x[lane * k + r];
            x[lane * k + r] = x[lane * k + blk.swap];
            x[lane * k + blk.swap] = t;
        }
        __syncwarp();
        for (int c = 0; c < nc; ++c) {
            const double bk = x[c * k + kk];
            const double bk1 = blk.size == 2 ? x[c * k + kk + 1] : 0.0;
            for (int i = kk + blk.size + lane; i < k; i += 32) {
                double v = x[c * k + i] - L(i, kk) * bk;
                if (blk.size == 2) v -= L(i, kk + 1) * bk1;
                x[c * k + i] = v;
            }
        }
        __syncwarp();
    }
    // block diagonal
    for (int b = 0; b < nb; ++b) {
        const Blk blk = blocks[b];
        const int kk = blk.start;
        if (lane < nc) {
            double* xc = x + lane * k;
            if (blk.size == 1) {
                xc[kk] /= L(kk, kk);
            } else {
                const double akm1k = L(kk + 1, kk);
                const double akm1 = L(kk, kk) / akm1k;
                const double ak = L(kk + 1, kk + 1) / akm1k;
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
        const Blk blk = blocks[b];
        const int kk = blk.start, below = kk + blk.size;
        for (int c = 0; c < nc; ++c) {
            for (int cc = kk; cc < below; ++cc) {
                double acc = 0.0;
                for (int i = below + lane; i < k; i += 32) acc += L(i, cc) * x[c * k + i];
                acc = warp_sum(acc);
                if (lane == 0) x[c * k + cc] -= acc;
            }
        }
        __syncwarp();
        const int r = kk + blk.size - 1;
        if (blk.swap != r && lane < nc) {
            const double t = x[lane * k + r];
            x[lane * k + r] = x[lane * k + blk.swap];
            x[lane * k + blk.swap] = t;
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

cudaError_t ldlt_factor(const double* S, int k, double* F, void* scratch, int* status, cudaStream_t stream) {
    Blk* blocks = static_cast<Blk*>(scratch);
    int* nblk = reinterpret_cast<int*>(blocks + k);
    const size_t smem = sizeof(double) * static_cast<size_t>(k) * k;
    const bool in_smem = smem <= 200 * 1024;
    if (in_smem) {
        cudaError_t e = cudaFuncSetAttribute(ldlt_bk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    ldlt_bk_kernel<<<1, kLdltThreads, in_smem ? smem : 0, stream>>>(S, k, F, blocks, nblk, status, in_smem);
    return cudaGetLastError();
}

cudaError_t ldlt_solve(const double* F, const void* scratch, int k, int64_t n, double* B, cudaStream_t stream) {
    const Blk* blocks = static_cast<const Blk*>(scratch);
    const int* nblk = reinterpret_cast<const int*>(blocks + k);
    const int64_t warps = (n + kLC - 1) / kLC;
    const size_t smem = sizeof(double) * 4 * kLC * static_cast<size_t>(k);
    cudaError_t e = cudaFuncSetAttribute(ldlt_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    ldlt_solve_kernel<<<static_cast<unsigned>((warps + 3) / 4), 128, smem, stream>>>(F, blocks, nblk, k, n, B);
    return cudaGetLastError();
}

cudaError_t map_cols(const long long* sampled, const long long* piv, int k, long long* cols, cudaStream_t stream) {
    map_cols_kernel<<<1, 256, 0, stream>>>(sampled, piv, k, cols);
    return cudaGetLastError();
}

}  // namespace idk

// batched.cu -- many small IDs, one CTA per matrix, everything fused.
//
// BASELINE cfg3: 4096 independent 64 x 256 matrices, k = 16.  The whole
// matrix (128 KiB) lives in shared memory, so HBM sees exactly one read of A
// and one write of Z and C per matrix.  Inside the CTA the reference's own
// algorithm runs unchanged, one thread per column, with the reference's
// sequential summation order and unfused IEEE multiply/add:
//   norms                     qr.cpp:56-62
//   pivot + physical swap     qr.cpp:66-86
//   make_householder          qr.cpp:16-28   (thread 0, sequential tail sum)
//   apply_householder         qr.cpp:31-38   (thread per trailing column)
//   downdate / recompute      qr.cpp:96-106
//   solve_triangular (upper)  solve.cpp:23-53 (thread per right-hand side)
//   Z scatter by perm, C = select_columns(A, cols)   matrix.cpp:121-130
// so the output is bit-identical to the reference composition
// qr_column_pivoted -> solve_triangular -> select_columns on the same matrix.
// The shared-memory stride is odd (m | 1), so thread-per-column accesses are
// bank-conflict free.
#include <climits>

#include "common.cuh"

namespace idk {

namespace {

constexpr int kBatchThreads = 256;
constexpr double kTie = 1.0 - 1e-14;

__device__ __forceinline__ double bmax(double v, double* scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    double t = lane < nw ? scratch[lane] : 0.0;
    return warp_max(t);
}

__device__ __forceinline__ int bmin_i(int v, int* scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    int t = lane < nw ? scratch[lane] : INT_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t = min(t, __shfl_xor_sync(0xffffffffu, t, o));
    return t;
}

__global__ void __launch_bounds__(kBatchThreads)
batched_id_kernel(const double* __restrict__ A, int64_t lda, int64_t stride, int m, int n, int k,
                  long long* __restrict__ cols_out, double* __restrict__ Z, double* __restrict__ C,
                  int* __restrict__ status) {
    extern __shared__ __align__(16) double sm[];
    const int ld = m | 1;
    double* S = sm;                                  // n columns, stride ld
    double* live = S + static_cast<size_t>(n) * ld;  // n
    double* anchor = live + n;                       // n
    int* perm = reinterpret_cast<int*>(anchor + n);  // n
    int* inv = perm + n;                             // n
    __shared__ double red_d[32];
    __shared__ int red_i[32];
    __shared__ double sc[3];

    const int tid = threadIdx.x;
    const int64_t b = blockIdx.x;
    const double* Ab = A + b * stride;

    for (int e = tid; e < m * n; e += blockDim.x) {
        const int j = e / m, i = e - j * m;
        S[j * ld + i] = __ldg(Ab + static_cast<int64_t>(j) * lda + i);
    }
    __syncthreads();
    for (int j = tid; j < n; j += blockDim.x) {
        const double* col = S + j * ld;
        double s = 0.0;
        for (int i = 0; i < m; ++i) s = add_rn(s, mul_rn(col[i], col[i]));
        live[j] = anchor[j] = s;
        perm[j] = j;
    }
    __syncthreads();

    for (int step = 0; step < k; ++step) {
        double v = 0.0;
        for (int l = step + tid; l < n; l += blockDim.x) v = fmax(v, live[l]);
        const double vmax = bmax(v, red_d);
        int pivot = step;
        if (vmax > 0.0) {
            const double thr = kTie * sqrt(vmax);
            int best = INT_MAX;
            for (int l = step + tid; l < n; l += blockDim.x)
                if (sqrt(live[l]) >= thr) best = min(best, l);
            pivot = bmin_i(best, red_i);
        }
        if (pivot != step) {
            double* cs = S + step * ld;
            double* cp = S + pivot * ld;
            for (int i = tid; i < m; i += blockDim.x) {
                const double t = cs[i];
                cs[i] = cp[i];
                cp[i] = t;
            }
            if (tid == 0) {
                int ti = perm[step]; perm[step] = perm[pivot]; perm[pivot] = ti;
                double t = live[step]; live[step] = live[pivot]; live[pivot] = t;
                t = anchor[step]; anchor[step] = anchor[pivot]; anchor[pivot] = t;
            }
        }
        __syncthreads();
        double* x = S + step * ld + step;
        const int len = m - step;
        if (tid == 0) {
            double tau = 0.0;
            if (len > 1) {
                double tail = 0.0;
                for (int i = 1; i < len; ++i) tail = add_rn(tail, mul_rn(x[i], x[i]));
                if (tail != 0.0) {
                    const double alpha = x[0];
                    const double beta = -copysign(sqrt(add_rn(mul_rn(alpha, alpha), tail)), alpha);
                    tau = (beta - alpha) / beta;
                    sc[1] = 1.0 / (alpha - beta);
                    sc[2] = beta;
                }
            }
            sc[0] = tau;
        }
        __syncthreads();
        const double tau = sc[0];
        if (tau != 0.0) {
            const double scale = sc[1];
            for (int i = 1 + tid; i < len; i += blockDim.x) x[i] = mul_rn(x[i], scale);
        }
        __syncthreads();
        if (tid == 0 && tau != 0.0) x[0] = sc[2];
        for (int l = step + 1 + tid; l < n; l += blockDim.x) {
            double* y = S + l * ld + step;
            if (tau != 0.0) {
                double w = y[0];
                for (int i = 1; i < len; ++i) w = add_rn(w, mul_rn(x[i], y[i]));
                w = mul_rn(w, tau);
                y[0] = sub_rn(y[0], w);
                for (int i = 1; i < len; ++i) y[i] = sub_rn(y[i], mul_rn(w, x[i]));
            }
            const double head = y[0];
            double lv = sub_rn(live[l], mul_rn(head, head));
            if (lv < 0.0) lv = 0.0;
            if (lv <= mul_rn(1e-6, anchor[l])) {
                double f = 0.0;
                for (int i = 1; i < len; ++i) f = add_rn(f, mul_rn(y[i], y[i]));
                lv = f;
                anchor[l] = f;
            }
            live[l] = lv;
        }
        __syncthreads();
    }

    // Singular floor (solve.cpp:27-30) on R11's diagonal.
    if (tid == 0) {
        int bad = -1;
        for (int i = 0; i < k; ++i)
            if (fabs(S[i * ld + i]) <= 1e-300) {
                bad = i;
                break;
            }
        status[b] = bad;
    }
    // T = R11^-1 R12, in place over rows 0..k-1 of the non-pivot columns.
    for (int j = k + tid; j < n; j += blockDim.x) {
        double* xj = S + j * ld;
        for (int i = k - 1; i >= 0; --i) {
            double acc = xj[i];
            for (int l = i + 1; l < k; ++l) acc = sub_rn(acc, mul_rn(S[l * ld + i], xj[l]));
            xj[i] = acc / S[i * ld + i];
        }
    }
    for (int j = tid; j < n; j += blockDim.x) inv[perm[j]] = j;
    __syncthreads();

    long long* cb = cols_out + b * k;
    for (int j = tid; j < k; j += blockDim.x) cb[j] = perm[j];
    double* Zb = Z + b * static_cast<int64_t>(k) * n;
    for (int e = tid; e < k * n; e += blockDim.x) {
        const int c = e / k, i = e - c * k;
        const int p = inv[c];
        Zb[e] = p < k ? (i == p ? 1.0 : 0.0) : S[p * ld + i];
    }
    if (C) {
        double* Cb = C + b * static_cast<int64_t>(m) * k;
        for (int e = tid; e < m * k; e += blockDim.x) {
            const int j = e / m, i = e - j * m;
            Cb[e] = __ldg(Ab + static_cast<int64_t>(perm[j]) * lda + i);
        }
    }
}

}  // namespace

size_t batched_id_smem_bytes(int m, int n) {
    return sizeof(double) * (static_cast<size_t>(n) * (m | 1) + 2 * static_cast<size_t>(n)) + 2 * sizeof(int) * n;
}

cudaError_t batched_id(const double* A, int64_t lda, int64_t stride, int64_t batch, int m, int n, int k,
                       long long* cols, double* Z, double* C, int* status, cudaStream_t stream) {
    if (batch <= 0) return cudaSuccess;
    const size_t smem = batched_id_smem_bytes(m, n);
    cudaError_t e = cudaFuncSetAttribute(batched_id_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    batched_id_kernel<<<static_cast<unsigned>(batch), kBatchThreads, smem, stream>>>(A, lda, stride, m, n, k, cols,
                                                                                      Z, C, status);
    return cudaGetLastError();
}

}  // namespace idk

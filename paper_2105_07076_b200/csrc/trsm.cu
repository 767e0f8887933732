// trsm.cu -- coefficient solve Z = [I | R11^-1 R12] P^T and the column gather.
//
// Reference: the north-star Z replaces optim_id's normal-equation solve
// (id.cpp:37-41) by the interpolation form built from the reference's own
// solve_triangular (solve.cpp:23-53, upper, back substitution) on
// R11 = leading_block(R, k) (id.cpp:20-25) and R12 = R[:, k:].  The scatter
// by perm needs no permutation pass: column c of Z depends only on column c
// of the factored matrix W, so each CTA solves a block of *physical* columns
// and writes e_pos(c) for the k pivot columns.
//
// The singular-diagonal floor |r_ii| <= 1e-300 (solve.cpp:19,27-30) is
// checked while R11 is gathered; the host maps it to SingularMatrixError
// (sketch) or NotPositiveDefiniteError (deterministic, solve.cpp:66-68).
#include <climits>

#include "common.cuh"

namespace idk {

namespace {

constexpr int kTrsmNB = 32;      // right-hand sides per CTA
constexpr int kTrsmThreads = 256;

__global__ void gather_r11_kernel(const double* __restrict__ W, int64_t ldw, const long long* __restrict__ pivots,
                                  int k, double* __restrict__ R11, int* __restrict__ status) {
    const int64_t total = static_cast<int64_t>(k) * k;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(e / k), i = static_cast<int>(e % k);
        const double v = (i <= j) ? W[pivots[j] * ldw + i] : 0.0;
        R11[e] = v;
        if (i == j && fabs(v) <= 1e-300) atomicMin(status, j);
    }
}

// X (k x nb tile of W's top k rows) <- R11^-1 X, blocked back substitution:
// 32-row diagonal blocks are solved warp-synchronously (lane = row, one warp
// per right-hand side), the rows above are updated by all threads.
__global__ void __launch_bounds__(kTrsmThreads)
id_trsm_kernel(const double* __restrict__ W, int64_t ldw, const double* __restrict__ R11, int k, int64_t n,
               const long long* __restrict__ pos, double* __restrict__ Z, int NB) {
    extern __shared__ double X[];
    const int ldx = k | 1;  // odd stride: lane-per-column accesses are bank-conflict free
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * NB;
    const int nb = static_cast<int>(min(static_cast<long long>(NB), static_cast<long long>(n - c0)));

    for (int e = tid; e < nb * k; e += blockDim.x) {
        const int c = e / k, i = e - c * k;
        X[c * ldx + i] = W[(c0 + c) * ldw + i];
    }
    __syncthreads();

    for (int hi = k; hi > 0;) {
        const int lo = hi > 32 ? hi - 32 : 0;
        const int bs = hi - lo;
        for (int c = warp; c < nb; c += nwarps) {
            double x = lane < bs ? X[c * ldx + lo + lane] : 0.0;
            for (int i = bs - 1; i >= 0; --i) {
                double xi = __shfl_sync(0xffffffffu, x, i);
                xi = xi / R11[static_cast<int64_t>(lo + i) * k + lo + i];
                if (lane == i) x = xi;
                if (lane < i) x = sub_rn(x, mul_rn(R11[static_cast<int64_t>(lo + i) * k + lo + lane], xi));
            }
            if (lane < bs) X[c * ldx + lo + lane] = x;
        }
        __syncthreads();
        for (int e = tid; e < lo * nb; e += blockDim.x) {
            const int c = e / lo, r = e - c * lo;
            const double* xc = X + c * ldx;
            double acc = 0.0;
            for (int l = lo; l < hi; ++l) acc += R11[static_cast<int64_t>(l) * k + r] * xc[l];
            X[c * ldx + r] = xc[r] - acc;
        }
        __syncthreads();
        hi = lo;
    }

    for (int e = tid; e < nb * k; e += blockDim.x) {
        const int c = e / k, i = e - c * k;
        const int64_t col = c0 + c;
        const long long p = pos[col];
        Z[col * k + i] = p < k ? (i == p ? 1.0 : 0.0) : X[c * ldx + i];
    }
}

// C[:, j] = A[:, cols[j]]  (matrix.cpp:121-130), or for the id_auto dual
// C[:, j] = A[cols[j], :]^T (a row of the tall A is a column of A^T).
__global__ void gather_columns_kernel(const double* __restrict__ A, int64_t lda, int64_t rows,
                                      const long long* __restrict__ cols, int k, bool rows_of_a,
                                      double* __restrict__ C) {
    const int64_t total = rows * k;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = e / rows, i = e - j * rows;
        C[e] = rows_of_a ? A[cols[j] + i * lda] : A[cols[j] * lda + i];
    }
}

__global__ void copy_pivots_kernel(const long long* __restrict__ src, int k, long long* __restrict__ dst) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) dst[i] = src[i];
}

}  // namespace

// Right-hand sides per CTA: 32 while the k x 32 tile fits in ~160 KB.
int id_trsm_nb(int k) {
    const int cap = static_cast<int>((160 * 1024 / sizeof(double)) / (k | 1));
    return cap >= kTrsmNB ? kTrsmNB : (cap < 1 ? 1 : cap);
}

size_t id_trsm_smem_bytes(int k) { return sizeof(double) * static_cast<size_t>(id_trsm_nb(k)) * (k | 1); }

// Z[:, j] for the columns j in [c_begin, c_begin + n) of W (Z has ld k and
// starts at column c_begin); R11 is gathered from the pivot columns of W.
cudaError_t id_solve_z(const double* W, int64_t ldw, int k, int64_t c_begin, int64_t n, const long long* pivots,
                       const long long* pos, double* R11, int* status, double* Z, cudaStream_t stream) {
    const int64_t kk = static_cast<int64_t>(k) * k;
    gather_r11_kernel<<<static_cast<int>(std::min<int64_t>((kk + 255) / 256, 1024)), 256, 0, stream>>>(
        W, ldw, pivots, k, R11, status);
    W += c_begin * ldw;
    pos += c_begin;
    if (n <= 0) return cudaGetLastError();
    const size_t smem = id_trsm_smem_bytes(k);
    cudaError_t e = cudaFuncSetAttribute(id_trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const int nb = id_trsm_nb(k);
    const int64_t blocks = (n + nb - 1) / nb;
    id_trsm_kernel<<<static_cast<unsigned>(blocks), kTrsmThreads, smem, stream>>>(W, ldw, R11, k, n, pos, Z, nb);
    return cudaGetLastError();
}

cudaError_t gather_columns(const double* A, int64_t lda, int64_t rows, const long long* cols, int k,
                           bool rows_of_a, double* C, cudaStream_t stream) {
    const int64_t total = rows * k;
    if (total <= 0) return cudaSuccess;
    gather_columns_kernel<<<static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 8)), 256, 0, stream>>>(
        A, lda, rows, cols, k, rows_of_a, C);
    return cudaGetLastError();
}

cudaError_t copy_pivots(const long long* src, int k, long long* dst, cudaStream_t stream) {
    copy_pivots_kernel<<<1, 256, 0, stream>>>(src, k, dst);
    return cudaGetLastError();
}

}  // namespace idk

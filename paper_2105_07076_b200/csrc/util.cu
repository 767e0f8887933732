// util.cu -- layout helpers for the id_auto dual (id.cpp:85: transpose(a)) and
// the reference-order product used for IdResult::approx.
#include <algorithm>

#include "common.cuh"

namespace idk {

namespace {
// B (cols x rows) = A (rows x cols)^T through a 32 x 33 shared tile.
__global__ void transpose_kernel(const double* __restrict__ A, int64_t lda, int64_t rows, int64_t cols,
                                 double* __restrict__ B, int64_t ldb) {
    __shared__ double tile[32][33];
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * 32, j0 = static_cast<int64_t>(blockIdx.y) * 32;
    for (int jj = threadIdx.y; jj < 32; jj += blockDim.y) {
        const int64_t i = i0 + threadIdx.x, j = j0 + jj;
        if (i < rows && j < cols) tile[jj][threadIdx.x] = A[j * lda + i];
    }
    __syncthreads();
    for (int ii = threadIdx.y; ii < 32; ii += blockDim.y) {
        const int64_t j = j0 + threadIdx.x, i = i0 + ii;
        if (i < rows && j < cols) B[i * ldb + j] = tile[threadIdx.x][ii];
    }
}

// C (M x N) = A (M x K) * B (K x N) with matrix.cpp:28-48's arithmetic: every
// output starts at +0.0 and accumulates a(i,l)*b(l,j) for l = 0..K-1 in order,
// skipping b(l,j) == 0, with unfused IEEE multiply and add (the reference is
// built without FMA).  Bit-identical to the reference's matmul; one thread per
// output, rows across lanes (coalesced A, broadcast B).
// b_trans: B(l, j) = B[j + l * ldb] (the sketch of the id_auto dual reads the
// stored tall A transposed, like matmul(Omega, transpose(A))).
__global__ void matmul_ref_order_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ B,
                                        int64_t ldb, bool b_trans, int64_t M, int64_t N, int K,
                                        double* __restrict__ C, int64_t ldc) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= M) return;
    const double* ai = A + i;
    for (int64_t j = blockIdx.y; j < N; j += gridDim.y) {  // N may exceed the 65535 grid rows
        const double* bj = b_trans ? B + j : B + j * ldb;
        const int64_t bstep = b_trans ? ldb : 1;
        double acc = 0.0;
        for (int l = 0; l < K; ++l) {
            const double b = __ldg(bj + l * bstep);
            if (b == 0.0) continue;
            acc = __dadd_rn(acc, __dmul_rn(ai[static_cast<int64_t>(l) * lda], b));
        }
        C[j * ldc + i] = acc;
    }
}
}  // namespace

cudaError_t matmul_ref_order(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t M, int64_t N, int K,
                             double* C, int64_t ldc, cudaStream_t stream, bool b_trans) {
    if (M <= 0 || N <= 0) return cudaSuccess;
    dim3 grid(static_cast<unsigned>((M + 127) / 128), static_cast<unsigned>(std::min<int64_t>(N, 65535)));
    matmul_ref_order_kernel<<<grid, 128, 0, stream>>>(A, lda, B, ldb, b_trans, M, N, K, C, ldc);
    return cudaGetLastError();
}

cudaError_t transpose_copy(const double* A, int64_t lda, int64_t rows, int64_t cols, double* B, int64_t ldb,
                           cudaStream_t stream) {
    if (rows <= 0 || cols <= 0) return cudaSuccess;
    dim3 grid(static_cast<unsigned>((rows + 31) / 32), static_cast<unsigned>((cols + 31) / 32));
    transpose_kernel<<<grid, dim3(32, 8), 0, stream>>>(A, lda, rows, cols, B, ldb);
    return cudaGetLastError();
}

}  // namespace idk

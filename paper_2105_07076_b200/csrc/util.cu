// util.cu -- layout helpers for the id_auto dual (id.cpp:85: transpose(a)).
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
}  // namespace

cudaError_t transpose_copy(const double* A, int64_t lda, int64_t rows, int64_t cols, double* B, int64_t ldb,
                           cudaStream_t stream) {
    if (rows <= 0 || cols <= 0) return cudaSuccess;
    dim3 grid(static_cast<unsigned>((rows + 31) / 32), static_cast<unsigned>((cols + 31) / 32));
    transpose_kernel<<<grid, dim3(32, 8), 0, stream>>>(A, lda, rows, cols, B, ldb);
    return cudaGetLastError();
}

}  // namespace idk

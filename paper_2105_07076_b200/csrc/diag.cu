// diag.cu -- the Z statistics of idkit::diagnostics (id.cpp:97-122):
// max |Z| and the identity-block deviation max |Z[i, cols[j]] - delta_ij|.
#include "common.cuh"

namespace idk {

namespace {
__global__ void z_stats_kernel(const double* __restrict__ Z, int k, int64_t zc, const long long* __restrict__ cols,
                               double* __restrict__ out2) {
    __shared__ double s0[32], s1[32];
    double mz = 0.0, dev = 0.0;
    const int64_t total = static_cast<int64_t>(k) * zc;
    for (int64_t e = threadIdx.x; e < total; e += blockDim.x) mz = fmax(mz, fabs(Z[e]));
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
        const int j = e / k, i = e - j * k;
        dev = fmax(dev, fabs(Z[cols[j] * k + i] - (i == j ? 1.0 : 0.0)));
    }
    mz = warp_max(mz);
    dev = warp_max(dev);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        s0[wid] = mz;
        s1[wid] = dev;
    }
    __syncthreads();
    if (wid == 0) {
        mz = lane < static_cast<int>(blockDim.x >> 5) ? s0[lane] : 0.0;
        dev = lane < static_cast<int>(blockDim.x >> 5) ? s1[lane] : 0.0;
        mz = warp_max(mz);
        dev = warp_max(dev);
        if (lane == 0) {
            out2[0] = mz;
            out2[1] = dev;
        }
    }
}
}  // namespace

cudaError_t z_stats(const double* Z, int k, int64_t zc, const long long* cols, double* out2, cudaStream_t stream) {
    z_stats_kernel<<<1, 1024, 0, stream>>>(Z, k, zc, cols, out2);
    return cudaGetLastError();
}

}  // namespace idk

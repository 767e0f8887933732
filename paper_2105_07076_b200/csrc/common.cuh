// common.cuh -- shared device helpers for the idkit-b200 kernels (sm_100a only).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#ifndef __CUDACC__
#error "compile with nvcc"
#endif

namespace idk {

constexpr int kWarp = 32;

// IEEE ops that must not be contracted into FMA: the reference is built
// without FMA (proj/CMakeLists.txt:3-10), and the norm downdate / reflector
// scalars are replayed bit-for-bit (qr.cpp:19-24, :98-100).
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ long long warp_min_ll(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}

// Deterministic block reduction: fixed per-warp xor tree, then warp 0 reduces
// the per-warp partials in a fixed tree.  `scratch` needs blockDim/32 doubles.
// All threads receive the result.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    double t = lane < nw ? scratch[lane] : 0.0;
    t = warp_sum(t);
    return t;
}

// L2-coherent accesses for data shared between CTAs of one launch.
__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ void st_cg(double* p, double v) { __stcg(p, v); }

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Grid-wide barrier for cooperatively launched (co-resident) grids.  The
// counter is monotonic: the e-th barrier waits until it reaches e*gridDim.
// The host zeroes the counter before each launch.
__device__ __forceinline__ void grid_barrier(unsigned* counter, unsigned& epoch) {
    __syncthreads();
    epoch += 1;
    if (threadIdx.x == 0) {
        const unsigned target = epoch * gridDim.x;
        __threadfence();
        atomicAdd(counter, 1u);
        while (ld_acquire_u32(counter) < target) {
        }
        __threadfence();
    }
    __syncthreads();
}

}  // namespace idk

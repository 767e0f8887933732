// Do DMMA (mma.sync m8n8k4 f64) and DFMA share the FP64 hardware on B200?
// Warps of one kernel run either a DMMA loop or a DFMA loop; if the two pipes
// are separate, the mixed kernel's total FP64 rate exceeds either alone.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_fp64_mix tools/probe_fp64_mix.cu
#include <cstdio>

#include <cuda_runtime.h>

__device__ __forceinline__ void dmma8(double (&c)[8][2], double a, double b) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[t][0]), "+d"(c[t][1])
                     : "d"(a), "d"(b));
}

// mode 0: all warps DMMA; 1: all DFMA; 2: warps alternate (even DMMA, odd DFMA);
// 3: every warp interleaves one DMMA group and one DFMA group per iteration
__global__ void mix(double* out, int iters, int mode, int dfma_per_iter) {
    const int warp = threadIdx.x >> 5;
    const double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[8][2];
    double f[16];
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = 0.0;
#pragma unroll
    for (int t = 0; t < 16; ++t) f[t] = t;
    const bool do_mma = mode == 0 || mode == 3 || (mode == 2 && (warp & 1) == 0);
    const bool do_fma = mode == 1 || mode == 3 || (mode == 2 && (warp & 1) == 1);
    for (int it = 0; it < iters; ++it) {
        if (do_mma) dmma8(c, a, b);
        if (do_fma) {
            for (int r = 0; r < dfma_per_iter; ++r) {
#pragma unroll
                for (int t = 0; t < 16; ++t) f[t] = fma(a, f[t], b);
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
#pragma unroll
    for (int t = 0; t < 16; ++t) s += f[t];
    if (s == 12345.0) out[0] = s;
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000, grid = p.multiProcessorCount * 2, threads = 256;
    const char* names[4] = {"DMMA only", "DFMA only", "warps alternate", "interleaved"};
    for (int dpi = 1; dpi <= 2; ++dpi) {
        for (int mode = 0; mode < 4; ++mode) {
            mix<<<grid, threads>>>(out, 100, mode, dpi);
            cudaEventRecord(e0);
            mix<<<grid, threads>>>(out, iters, mode, dpi);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double warps = static_cast<double>(grid) * (threads / 32);
            const double mma_w = mode == 0 || mode == 3 ? warps : (mode == 2 ? warps / 2 : 0);
            const double fma_w = mode == 1 || mode == 3 ? warps : (mode == 2 ? warps / 2 : 0);
            const double fl_mma = mma_w * iters * 8 * 2.0 * 256;      // 8 DMMA of 8x8x4 per iteration
            const double fl_fma = fma_w * 32 * iters * dpi * 16 * 2.0;  // dpi x 16 DFMA per thread
            printf("%-16s dfma/iter %d: DMMA %.2f + DFMA %.2f = %.2f TFLOP/s (%.3f ms)\n", names[mode], dpi,
                   fl_mma / ms / 1e9, fl_fma / ms / 1e9, (fl_mma + fl_fma) / ms / 1e9, ms);
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

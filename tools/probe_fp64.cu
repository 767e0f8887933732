// Microbenchmark: FP64 DMMA (mma.sync m8n8k4 f64) vs DFMA throughput on one B200.
// Used once to fix the FP64 roofline denominator (MEASURED_PEAKS.json has none).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[8][2];
    #pragma unroll
    for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
    for (int it = 0; it < iters; ++it) {
        #pragma unroll
        for (int t = 0; t < 8; ++t) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
        }
    }
    double s = 0;
    #pragma unroll
    for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
    if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[16];
    #pragma unroll
    for (int t = 0; t < 16; ++t) c[t] = t;
    for (int it = 0; it < iters; ++it) {
        #pragma unroll
        for (int t = 0; t < 16; ++t) c[t] = fma(a, c[t], b);
    }
    double s = 0;
    #pragma unroll
    for (int t = 0; t < 16; ++t) s += c[t];
    if (s == 12345.0) out[0] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    printf("device %s SMs %d smemOptin %zu L2 %d clock %d kHz\n", p.name, p.multiProcessorCount,
           p.sharedMemPerBlockOptin, p.l2CacheSize, p.clockRate);
    double* out; cudaMalloc(&out, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int iters = 20000;
    for (int bpsm = 1; bpsm <= 4; bpsm *= 2) for (int threads = 128; threads <= 512; threads *= 2) {
        int grid = p.multiProcessorCount * bpsm;
        dmma_loop<<<grid, threads>>>(out, 100);
        cudaEventRecord(e0);
        dmma_loop<<<grid, threads>>>(out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 256 * 8 * (double)iters * (threads / 32) * grid;
        printf("DMMA grid %d thr %d: %.2f TFLOP/s\n", grid, threads, flops / ms / 1e9);
        dfma_loop<<<grid, threads>>>(out, 100);
        cudaEventRecord(e0);
        dfma_loop<<<grid, threads>>>(out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        flops = 2.0 * 16 * (double)iters * threads * grid;
        printf("DFMA grid %d thr %d: %.2f TFLOP/s\n", grid, threads, flops / ms / 1e9);
    }
    size_t n = (size_t)1 << 27;  // 2 GiB per buffer as double2 x 2^27 = 2 GiB
    double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
    cudaMemset(a, 0, n * 16);
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        copy_kernel<<<p.multiProcessorCount * 8, 512>>>(a, b, n);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("copy: %.1f GB/s\n", 2.0 * n * 16 / ms / 1e6);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

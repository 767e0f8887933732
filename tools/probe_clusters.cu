// How many thread-block clusters of size C can be co-resident on this B200
// (cudaOccupancyMaxActiveClusters) for a CPQR-like CTA (512 threads, ~200 KB
// shared memory, one CTA per SM), and which SMs each cluster lands on.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__global__ void probe(unsigned* out, unsigned long long spin) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    unsigned cid;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
    if (threadIdx.x == 0) out[blockIdx.x] = smid;
    const unsigned long long t0 = clock64();
    while (clock64() - t0 < spin) {}
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    printf("%s: %d SMs\n", p.name, p.multiProcessorCount);
    cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    unsigned* d;
    cudaMalloc(&d, 4096 * sizeof(unsigned));
    for (int smem : {0, 200 * 1024}) {
        for (int c : {1, 2, 4, 6, 8, 9, 10, 12, 14, 16}) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(c * 64);
            cfg.blockDim = dim3(512);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = c;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int n = -1;
            cudaError_t e = cudaOccupancyMaxActiveClusters(&n, probe, &cfg);
            printf("smem %6d cluster %2d: max active clusters %3d (%3d SMs) %s\n", smem, c, n, n * c,
                   e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    }
    // SM layout: launch 1 CTA per SM with cluster 1 and read smid -> nothing about GPCs.
    // Launch max clusters of 16 at 200 KB and print their SM sets.
    for (int c : {8, 9, 16}) {
        cudaLaunchConfig_t cfg = {};
        int n = 0;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = c;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = 200 * 1024;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(c);
        cudaOccupancyMaxActiveClusters(&n, probe, &cfg);
        cfg.gridDim = dim3(c * n);
        cudaLaunchKernelEx(&cfg, probe, d, 2000000ull);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<unsigned> h(c * n);
        cudaMemcpy(h.data(), d, sizeof(unsigned) * c * n, cudaMemcpyDeviceToHost);
        printf("cluster %d x %d: %s\n", c, n, cudaGetErrorString(e));
        for (int i = 0; i < n; ++i) {
            printf("  cluster %2d SMs:", i);
            for (int j = 0; j < c; ++j) printf(" %3u", h[i * c + j]);
            printf("\n");
        }
    }
    return 0;
}

// Microbenchmarks of the CPQR exchange primitives on one B200:
//   grid barrier (148 CTAs), cluster barrier (16 CTAs), L2 / DSMEM dependent
//   load latency, and a full "publish + barrier + read G records + read a
//   column" exchange.  Times from %globaltimer, averaged over many rounds.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ long long gtime() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void grid_barrier_kernel(unsigned* ctr, int rounds, long long* out, int variant) {
    long long t0 = gtime();
    for (int r = 1; r <= rounds; ++r) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(ctr, 1u);
            const unsigned target = r * gridDim.x;
            if (variant == 0) {
                while (ld_acq(ctr) < target) {
                }
            } else {
                while (ld_acq(ctr) < target) __nanosleep(32);
            }
            __threadfence();
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (gtime() - t0) / rounds;
}

__global__ void l2_chase_kernel(const unsigned* next, int hops, long long* out) {
    unsigned p = 0;
    long long t0 = gtime();
    for (int i = 0; i < hops; ++i) p = __ldcg(next + p);
    long long t1 = gtime();
    if (p == 0xffffffff) out[1] = p;
    out[0] = (t1 - t0) / hops;
}

__global__ void __cluster_dims__(16, 1, 1) cluster_kernel(int rounds, long long* out) {
    __shared__ unsigned buf[64];
    cg::cluster_group cl = cg::this_cluster();
    buf[threadIdx.x & 63] = (cl.block_rank() + 1) & 15;
    cl.sync();
    long long t0 = gtime();
    for (int r = 0; r < rounds; ++r) cl.sync();
    long long t1 = gtime();
    // dependent DSMEM chase across the cluster
    unsigned p = 0;
    long long t2 = gtime();
    for (int r = 0; r < rounds; ++r) {
        const unsigned* rb = cl.map_shared_rank(buf, p);
        p = rb[0];
    }
    long long t3 = gtime();
    cl.sync();
    if (cl.block_rank() == 0 && threadIdx.x == 0) {
        out[0] = (t1 - t0) / rounds;
        out[1] = (t3 - t2) / rounds + (p == 99 ? 1 : 0);
    }
}

// One exchange round as the grid-mode CPQR does it.
__global__ void exchange_kernel(unsigned* ctr, double* recs, double* cols, int rounds, int m, long long* out) {
    __shared__ double xv[1024];
    __shared__ long long win;
    const int G = gridDim.x;
    long long t0 = gtime();
    for (int r = 1; r <= rounds; ++r) {
        const int par = r & 1;
        // publish: record (6 doubles) + a column of m doubles
        double* myrec = recs + (static_cast<size_t>(par) * G + blockIdx.x) * 6;
        double* mycol = cols + (static_cast<size_t>(par) * G + blockIdx.x) * m;
        for (int i = threadIdx.x; i < m; i += blockDim.x) __stcg(mycol + i, i + r);
        if (threadIdx.x < 6) __stcg(myrec + threadIdx.x, static_cast<double>(blockIdx.x * 7 % G + r));
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(ctr, 1u);
            while (ld_acq(ctr) < static_cast<unsigned>(r * G)) {
            }
            __threadfence();
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            double best = -1.0;
            int bi = 0;
            for (int g = threadIdx.x; g < G; g += 32) {
                const double v = __ldcg(recs + (static_cast<size_t>(par) * G + g) * 6);
                if (v > best) {
                    best = v;
                    bi = g;
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) {
                    best = ob;
                    bi = oi;
                }
            }
            if (threadIdx.x == 0) win = bi;
        }
        __syncthreads();
        const double* src = cols + (static_cast<size_t>(par) * G + win) * m;
        for (int i = threadIdx.x; i < m; i += blockDim.x) xv[i] = __ldcg(src + i);
        __syncthreads();
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (gtime() - t0) / rounds;
    if (xv[3] == -1.0) out[1] = 1;
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const int G = p.multiProcessorCount;
    unsigned* ctr;
    long long* out;
    cudaMalloc(&ctr, 4);
    cudaMalloc(&out, 64);
    long long h[2];
    for (int variant = 0; variant < 2; ++variant)
        for (int threads : {32, 256}) {
            cudaMemset(ctr, 0, 4);
            int rounds = 2000;
            void* args[] = {&ctr, &rounds, &out, &variant};
            cudaLaunchCooperativeKernel((void*)grid_barrier_kernel, G, threads, args, 0, 0);
            cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
            printf("grid barrier %d CTAs x %d thr (%s): %lld ns/round\n", G, threads, variant ? "nanosleep" : "spin", h[0]);
        }
    // L2 pointer chase (16 MB array, random-ish stride, L2 resident after warm)
    const int N = 1 << 20;
    unsigned* hn = new unsigned[N];
    for (int i = 0; i < N; ++i) hn[i] = (static_cast<unsigned long long>(i) * 7919 + 104729) % N;
    unsigned* dn;
    cudaMalloc(&dn, N * 4);
    cudaMemcpy(dn, hn, N * 4, cudaMemcpyHostToDevice);
    l2_chase_kernel<<<1, 1>>>(dn, 20000, out);
    l2_chase_kernel<<<1, 1>>>(dn, 20000, out);
    cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
    printf("L2 dependent load (ld.cg): %lld ns\n", h[0]);
    cluster_kernel<<<16, 128>>>(2000, out);
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("cluster.sync (16 CTAs): %lld ns/round; DSMEM dependent load: %lld ns\n", h[0], h[1]);
    double *recs, *cols;
    cudaMalloc(&recs, 2 * G * 6 * 8);
    cudaMalloc(&cols, 2 * G * 1024 * 8);
    for (int m : {110, 500}) {
        for (int threads : {128, 512}) {
            cudaMemset(ctr, 0, 4);
            int rounds = 1000;
            void* args[] = {&ctr, &recs, &cols, &rounds, &m, &out};
            cudaLaunchCooperativeKernel((void*)exchange_kernel, G, threads, args, 0, 0);
            cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
            printf("grid exchange (publish+barrier+records+column m=%d, %d thr): %lld ns/round\n", m, threads, h[0]);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}

// Microbenchmark of cluster (DSMEM) exchange patterns for the resident CPQR:
// one 16-CTA cluster, 512 threads per CTA, per round every CTA publishes a
// 6-double header + `rows` doubles and learns every other CTA's header and one
// winner's rows.  Variants:
//   0 cluster.sync only
//   1 bulk push header+rows to all peers (2 cp.async.bulk per peer) + mbarrier wait
//   2 bulk push one contiguous copy per peer + mbarrier wait
//   3 st.shared::cluster header to all peers + cluster.sync + ld.shared::cluster winner rows
//   4 st.shared::cluster header+rows to all peers + cluster.sync
//   5 bulk push header only + mbarrier wait + ld.shared::cluster winner rows
//   6 warp 0: st.shared::cluster header + remote mbarrier arrive (release.cluster); all wait (acquire.cluster)
//   7 variant 6 + ld.shared::cluster winner rows + __syncthreads
//   8 warp 0: bulk push hdr+rows 1/peer (mbarrier tx), all wait (the kernel's push mode)
//   9 15 warps issue one bulk push each
//  10 warp 0: st.async 16-B remote stores of hdr+rows to every peer (mbarrier tx)
//  11 warps 0..14: warp w st.async's hdr+rows to peer w (mbarrier tx)
//  12 warp 0: hdr+rows stored to a global slot, then ONE cp.async.bulk
//     global -> shared::cluster .multicast::cluster to all 16 CTAs (mbarrier tx)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_dsmem tools/probe_dsmem.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ long long gtime() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ unsigned mapa_u32(unsigned a, int rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void bulk_push(unsigned dst, unsigned src, unsigned bytes, unsigned mbar) {
    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "r"(src), "r"(bytes), "r"(mbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned a, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned a, unsigned b) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(unsigned a_cluster) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a_cluster) : "memory");
}
__device__ __forceinline__ void st_cluster_v2(unsigned a, double x, double y) {
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ void st_async_v2(unsigned a, double x, double y, unsigned mbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(a), "d"(x),
                 "d"(y), "r"(mbar)
                 : "memory");
}
__device__ __forceinline__ void bulk_mcast(unsigned dst, const void* src, unsigned bytes, unsigned mbar,
                                           unsigned short mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(mbar), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void mbar_wait_cl(unsigned a, unsigned par) {
    asm volatile(
        "{\n\t.reg .pred p;\nWC_%=:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t@!p bra WC_%=;\n}" ::"r"(a),
        "r"(par)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned a, unsigned par) {
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(a),
        "r"(par)
        : "memory");
}

constexpr int G = 16;
constexpr int HDR = 6;

__global__ void __cluster_dims__(G, 1, 1) probe(int variant, int rows, int rounds, long long* out, double* gslots) {
    extern __shared__ __align__(16) double sm[];
    __shared__ unsigned long long mbar[2];
    __shared__ unsigned long long mbar2[2];
    __shared__ __align__(16) double hdrs[2][G][HDR];
    __shared__ double xb[1024];
    cg::cluster_group cl = cg::this_cluster();
    const int me = cl.block_rank(), tid = threadIdx.x, T = blockDim.x;
    const int slot = HDR + rows;  // rows even
    for (int i = tid; i < 2 * G * slot; i += T) sm[i] = 0.0;
    if (tid == 0) {
        mbar_init(smem_u32(&mbar[0]), 1);
        mbar_init(smem_u32(&mbar[1]), 1);
        mbar_init(smem_u32(&mbar2[0]), G);
        mbar_init(smem_u32(&mbar2[1]), G);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cl.sync();
    unsigned phase = 0;
    double acc = 0.0;
    long long t0 = gtime();
    for (int r = 0; r < rounds; ++r) {
        const int p = r & 1;
        double* own = sm + (p * G + me) * slot;
        if (tid < rows + HDR) own[tid] = r + me + tid;
        __syncthreads();
        if (variant == 0) {
            cl.sync();
        } else if (variant == 1 || variant == 2 || variant == 5) {
            const unsigned mb = smem_u32(&mbar[p]);
            const unsigned per = variant == 5 ? HDR * 8 : (HDR + rows) * 8;
            if (tid == 0) mbar_expect_tx(mb, (G - 1) * per);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (variant == 1) {
                if (tid < 2 * (G - 1)) {
                    const int gi = tid >> 1, g = gi < me ? gi : gi + 1;
                    const double* src = (tid & 1) ? own + HDR : own;
                    const unsigned sa = smem_u32(src);
                    bulk_push(mapa_u32(sa, g), sa, (tid & 1) ? rows * 8 : HDR * 8, mapa_u32(mb, g));
                }
            } else {
                if (tid < G - 1) {
                    const int g = tid < me ? tid : tid + 1;
                    const unsigned sa = smem_u32(own);
                    bulk_push(mapa_u32(sa, g), sa, per, mapa_u32(mb, g));
                }
            }
            mbar_wait(mb, (phase >> p) & 1u);
            phase ^= 1u << p;
            if (variant == 5) {
                const int w = r % G;
                const double* src = cl.map_shared_rank(sm + (p * G + w) * slot, w);
                if (tid < rows) xb[tid] = src[HDR + tid];
                __syncthreads();
            }
        } else if (variant == 6 || variant == 7) {
            const unsigned mb = smem_u32(&mbar2[p]);
            if (threadIdx.x < 32) {
                const int lane = threadIdx.x;
                if (lane < G - 1) {
                    const int g = lane < me ? lane : lane + 1;
                    const unsigned ha = mapa_u32(smem_u32(&hdrs[p][me][0]), g);
                    st_cluster_v2(ha, own[0], own[1]);
                    st_cluster_v2(ha + 16, own[2], own[3]);
                    st_cluster_v2(ha + 32, own[4], own[5]);
                    mbar_arrive_remote(mapa_u32(mb, g));
                } else if (lane == 31) {
                    for (int j = 0; j < HDR; ++j) hdrs[p][me][j] = own[j];
                    mbar_arrive_remote(mapa_u32(mb, me));
                }
            }
            mbar_wait_cl(mb, (phase >> p) & 1u);
            phase ^= 1u << p;
            if (variant == 7) {
                const int w = r % G;
                const double* src = cl.map_shared_rank(sm + (p * G + w) * slot, w);
                if (tid < rows) xb[tid] = src[HDR + tid];
                __syncthreads();
            }
        } else if (variant == 9) {
            const unsigned mb = smem_u32(&mbar[p]);
            const unsigned per = (HDR + rows) * 8;
            const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
            if (tid == 0) mbar_expect_tx(mb, (G - 1) * per);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (ln == 0 && w < G - 1) {
                const int g = w < me ? w : w + 1;
                const unsigned sa = smem_u32(own);
                bulk_push(mapa_u32(sa, g), sa, per, mapa_u32(mb, g));
            }
            mbar_wait(mb, (phase >> p) & 1u);
            phase ^= 1u << p;
        } else if (variant == 8) {
            const unsigned mb = smem_u32(&mbar[p]);
            const unsigned per = (HDR + rows) * 8;
            if (threadIdx.x < 32) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (threadIdx.x == 0) mbar_expect_tx(mb, (G - 1) * per);
                if (threadIdx.x < G - 1) {
                    const int g = threadIdx.x < me ? threadIdx.x : threadIdx.x + 1;
                    const unsigned sa = smem_u32(own);
                    bulk_push(mapa_u32(sa, g), sa, per, mapa_u32(mb, g));
                }
            }
            mbar_wait(mb, (phase >> p) & 1u);
            phase ^= 1u << p;
        } else if (variant == 10 || variant == 11) {
            const unsigned mb = smem_u32(&mbar[p]);
            const int per = HDR + rows, nch = per / 2;
            if (tid == 0) mbar_expect_tx(mb, (G - 1) * per * 8);
            const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
            if (variant == 10 && w == 0) {
                for (int e = ln; e < (G - 1) * nch; e += 32) {
                    const int gi = e / nch, c = e - gi * nch, g = gi < me ? gi : gi + 1;
                    st_async_v2(mapa_u32(smem_u32(own + 2 * c), g), own[2 * c], own[2 * c + 1], mapa_u32(mb, g));
                }
            } else if (variant == 11 && w < G - 1) {
                const int g = w < me ? w : w + 1;
                const unsigned rb = mapa_u32(smem_u32(own), g), rm = mapa_u32(mb, g);
                for (int c = ln; c < nch; c += 32) st_async_v2(rb + 16 * c, own[2 * c], own[2 * c + 1], rm);
            }
            mbar_wait(mb, (phase >> p) & 1u);
            phase ^= 1u << p;
        } else if (variant == 12) {
            const unsigned mb = smem_u32(&mbar[p]);
            const int per = HDR + rows;
            if (tid == 0) mbar_expect_tx(mb, G * per * 8);
            if (threadIdx.x < 32) {
                double* gs = gslots + (static_cast<size_t>(p) * G + me) * slot;
                for (int i = threadIdx.x; i < per; i += 32) gs[i] = own[i];
                asm volatile("fence.proxy.async.global;" ::: "memory");
                __syncwarp();
                if (threadIdx.x == 0) bulk_mcast(smem_u32(own), gs, per * 8, mb, 0xffff);
            }
            mbar_wait(mb, (phase >> p) & 1u);
            phase ^= 1u << p;
        } else if (variant == 3) {
            if (tid < G && tid != me) {
                double* dst = cl.map_shared_rank(own, tid);
                for (int j = 0; j < HDR; ++j) dst[j] = own[j];
            }
            cl.sync();
            const int w = r % G;
            const double* src = cl.map_shared_rank(sm + (p * G + w) * slot, w);
            if (tid < rows) xb[tid] = src[HDR + tid];
            __syncthreads();
        } else if (variant == 4) {
            __syncthreads();
            const int len = HDR + rows, tot = (G - 1) * len;
            for (int e = tid; e < tot; e += T) {
                const int gi = e / len, j = e - gi * len, g = gi < me ? gi : gi + 1;
                cl.map_shared_rank(own, g)[j] = own[j];
            }
            cl.sync();
        }
        acc += sm[((p * G + (r % G)) * slot) + HDR + (tid % rows)] + xb[tid & 1023];
    }
    long long t1 = gtime();
    if (tid == 0 && me == 0) out[0] = (t1 - t0) / rounds;
    if (acc == 12345.678) out[1] = 1;
    cl.sync();
}

int main() {
    long long* out;
    cudaMalloc(&out, 16);
    double* gslots;
    cudaMalloc(&gslots, sizeof(double) * 2 * G * (HDR + 512));
    const char* names[] = {"cluster.sync only", "bulk push hdr+rows (2/peer) + mbar", "bulk push 1/peer + mbar",
                           "st.cluster hdr + cluster.sync + ld.cluster rows", "st.cluster hdr+rows + cluster.sync",
                           "bulk push hdr + mbar + ld.cluster rows", "warp0 st.cluster hdr + remote arrive",
                           "warp0 st.cluster hdr + remote arrive + ld.cluster rows", "warp0 bulk push 1/peer + mbar",
                           "15 warps x 1 bulk push + mbar", "warp0 st.async hdr+rows to all peers", "warp w st.async hdr+rows to peer w", "warp0 global slot + 1 multicast bulk copy"};
    for (int rows : {112, 272, 512}) {
        for (int v = 0; v < 13; ++v) {
            const size_t smem = sizeof(double) * 2 * G * (HDR + rows);
            cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            cudaMemset(out, 0, 16);
            probe<<<G, 512, smem>>>(v, rows, 2000, out, gslots);
            cudaError_t e = cudaGetLastError();
            long long h = -1;
            if (e == cudaSuccess) e = cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
            printf("rows %3d  %-48s %6lld ns/round  (%s)\n", rows, names[v], h, cudaGetErrorString(e));
        }
    }
    return 0;
}
